// Batched reductions and the GMRES state (part of batch.cu's translation unit).
// Included by batch.cu; not a standalone header.
// --------------------------------------------------------------------------
// Batched reductions
// --------------------------------------------------------------------------
struct Chunking {
  int chunk, nchunk;
};
Chunking chunking(const smpm_batch* b, long long len = -1) {
  if (len < 0) len = b->k;
  const long long target_ctas = 4LL * b->ctx->num_sms;
  long long per_sys = std::max(1LL, target_ctas / b->nsys);
  long long chunk = (len + per_sys - 1) / per_sys;
  chunk = std::max(128LL, std::min(2048LL, (chunk + 31) / 32 * 32));
  Chunking c;
  c.chunk = static_cast<int>(chunk);
  c.nchunk = static_cast<int>(std::max(1LL, (len + chunk - 1) / chunk));
  return c;
}

// out[s] = x_s . y_s  (device)
void batched_dot(smpm_batch* b, const double* x, const double* y, double* out, const int* act, cudaStream_t st,
                 long long len = -1) {
  if (len < 0) len = b->k;
  const Chunking c = chunking(b, len);
  b->dpart.alloc(std::max<size_t>(b->dpart.n, static_cast<size_t>(b->nsys) * c.nchunk));
  dim3 grid(c.nchunk, b->nsys);
  batched_dot_kernel<<<grid, VEC_THREADS, 0, st>>>(b->nsys, len, c.chunk, c.nchunk, act, x, y, b->dpart.p, b->dcount.p,
                                                   out);
  check_launch(b);
}

// --------------------------------------------------------------------------
// GMRES driver
// --------------------------------------------------------------------------
void ensure_gmres(smpm_batch* b, int m, int mtot) {
  const int histcap = mtot + 2;
  Chunking c;
  c.chunk = V2_CHUNK;
  c.nchunk = static_cast<int>((b->k + V2_CHUNK - 1) / V2_CHUNK);
  if (b->gm_m != m || b->gm_hist != histcap || b->G.nchunk != c.nchunk) {
    const size_t ns = static_cast<size_t>(b->nsys);
    b->dV.alloc(ns * (m + 1) * b->k);
    b->dR.alloc(ns * (m + 1) * m);
    b->dcs.alloc(ns * m);
    b->dsn.alloc(ns * m);
    b->dg.alloc(ns * (m + 1));
    b->dh1.alloc(ns * (m + 2));
    b->dh2.alloc(ns * (m + 2));
    b->dy.alloc(ns * m);
    b->dhist.alloc(ns * histcap);
    b->dgpart.alloc(ns * ((b->k + 127) / 128) * (m + 2));  // adaptive chunks down to 128 rows
    b->dscal.alloc(ns * 8);
    b->dgint.alloc(ns * 8);
    b->gm_m = m;
    b->gm_hist = histcap;
  }
  GmState_& G = b->G;
  int* ip = b->dgint.p;
  const int ns = b->nsys;
  G.jcyc = ip;
  G.iters = ip + ns;
  G.state = ip + 2 * ns;
  G.active = ip + 3 * ns;
  G.counter = ip + 4 * ns;
  G.hist_len = ip + 5 * ns;
  double* dp = b->dscal.p;
  G.bnorm = dp;
  G.target = dp + ns;
  G.hmax = dp + 2 * ns;
  G.nrm = dp + 3 * ns;
  G.R = b->dR.p;
  G.cs = b->dcs.p;
  G.sn = b->dsn.p;
  G.g = b->dg.p;
  G.h1 = b->dh1.p;
  G.h2 = b->dh2.p;
  G.y = b->dy.p;
  G.hist = b->dhist.p;
  G.part = b->dgpart.p;
  G.m = m;
  G.m_total = mtot;
  G.histcap = histcap;
  G.k = b->k;
  G.vstride = static_cast<long long>(m + 1) * b->k;
  // Arnoldi passes: fixed 512-row chunks (thread-per-row kernels, vec2.cuh)
  G.chunk = V2_CHUNK;
  G.nchunk = static_cast<int>((b->k + V2_CHUNK - 1) / V2_CHUNK);
  G.nsys = ns;
  b->dsnsq.alloc(static_cast<size_t>(ns));
  G.snsq = b->dsnsq.p;
  G.stacked = 0;
  (void)c;
  b->gm_mtot = mtot;
  CUDA_CHECK(cudaMemsetAsync(b->dgint.p, 0, sizeof(int) * ns * 8, b->ctx->stream));
}

struct SolveCfg {
  int method;
  double tol;
  int max_iter, restart, orth;
  bool fused, final_check;
  bool stacked = false;  // one GMRES over all systems (proj/src/helmholtz.cpp:187-246)
};
