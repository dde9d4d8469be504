// The C ABI of include/smpm_b200.h (part of batch.cu's translation unit).
// Included by batch.cu; not a standalone header.
// ============================================================================
// C ABI
// ============================================================================
// ---- strip solver ------------------------------------------
StripParams strip_params(const smpm_batch* b) {
  StripParams P;
  P.n = b->n;
  P.mx = b->mx;
  P.mz = b->mz;
  P.w = b->w;
  P.nmode = b->sp_nmode;
  P.npairs = b->sp_npairs;
  P.nsys = b->nsys;
  P.r = static_cast<long long>(b->mx) * b->mz * b->n * b->n;
  P.k = b->k;
  P.fac = reinterpret_cast<const double2*>(b->dsfac.p);
  P.lz = reinterpret_cast<const double2*>(b->dslz.p);
  P.mu = b->dsmu.p;
  P.tau = b->strip_tau;
  return P;
}

// out = A in for every w-long column of nsys x ncol_sys columns (system stride
// sys_stride): the resident-slice transform kernel, or a plain cuBLAS GEMM
void xf_columns(smpm_batch* b, bool inverse, const double* in, double* out, int ncol_sys, long long sys_stride,
                cudaStream_t st, int nsys_) {
  const int nsys = nsys_ < 0 ? b->nsys : nsys_;
  if (b->xf_P > 0) {
    XformArgs a;
    a.Af = inverse ? b->dTifrag.p : b->dTfrag.p;
    a.w = b->w;
    a.ncol_sys = ncol_sys;
    a.k = sys_stride;
    a.alist = nullptr;
    a.acount = nullptr;
    a.nslots = nsys;
    a.nv = 1;
    a.in[0] = in;
    a.out[0] = out;
    a.in[1] = nullptr;
    a.out[1] = nullptr;
    a.P = b->xf_P;
    const long long nch = (static_cast<long long>(nsys) * ncol_sys + 15) / 16;
    const int groups = static_cast<int>(std::max(1LL, std::min<long long>(b->ctx->num_sms / a.P, nch)));
    if (b->xp_on)
      launch_xformp(b, a, inverse, st, false);
    else
      launch_xform(b, a, groups, st, false);
    return;
  }
  if (sys_stride != static_cast<long long>(ncol_sys) * b->w) fail(SMPM_EINVAL, "strip columns must be contiguous");
  smpm_ctx* ctx = b->ctx;
  if (!ctx->blas && cublasCreate(&ctx->blas) != CUBLAS_STATUS_SUCCESS) fail(SMPM_ECUDA, "cublasCreate failed");
  if (cublasSetStream(ctx->blas, st) != CUBLAS_STATUS_SUCCESS) fail(SMPM_ECUDA, "cublasSetStream failed");
  const double one = 1.0, zero = 0.0;
  const int w = b->w;
  const long long ncols = static_cast<long long>(nsys) * ncol_sys;
  if (ncols > INT_MAX) fail(SMPM_EINVAL, "too many strip columns");
  if (cublasDgemm(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_N, w, static_cast<int>(ncols), w, &one,
                  inverse ? b->dTi.p : b->dT.p, w, in, w, &zero, out, w) != CUBLAS_STATUS_SUCCESS)
    fail(SMPM_ECUDA, "cublasDgemm failed");
}

template <bool TRACES>
void strip_modes(smpm_batch* b, const double* Xh, double* out, cudaStream_t st) {
  const StripParams P = strip_params(b);
  const dim3 grid((P.nmode + 127) / 128, P.mx, P.nsys);
  switch (P.n) {
#define SMPM_STRIP_CASE(N) \
  case N: strip_modes_kernel<N, TRACES><<<grid, 128, 0, st>>>(P, Xh, out); break;
    SMPM_STRIP_CASE(4) SMPM_STRIP_CASE(5) SMPM_STRIP_CASE(6) SMPM_STRIP_CASE(7) SMPM_STRIP_CASE(8)
    SMPM_STRIP_CASE(9) SMPM_STRIP_CASE(10) SMPM_STRIP_CASE(11) SMPM_STRIP_CASE(12) SMPM_STRIP_CASE(13)
    SMPM_STRIP_CASE(14) SMPM_STRIP_CASE(15) SMPM_STRIP_CASE(16) SMPM_STRIP_CASE(17)
#undef SMPM_STRIP_CASE
    default: fail(SMPM_EINVAL, "strip solver: n must be in [4, 17]");
  }
  check_launch(b);
}

void strip_scratch(smpm_batch* b) {
  const size_t r = static_cast<size_t>(b->mx) * b->mz * b->n * b->n;
  if (b->dsx1.n < b->nsys * r) {
    b->dsx1.alloc(b->nsys * r);
    b->dsx2.alloc(b->nsys * r);
  }
  if (b->dsbh.n < static_cast<size_t>(b->nsys) * b->k) b->dsbh.alloc(static_cast<size_t>(b->nsys) * b->k);
}

void need_strip(smpm_batch* b) {
  need_final(b);
  if (!b->strip_ok) fail(SMPM_EINVAL, "strip factors not set (smpm_batch_set_strip_factors)");
  strip_scratch(b);
}

// ---- transverse Fourier transforms (fourier.cuh) ----------------------------
// twiddle tables exp(sign 2 pi i k / m), k < m / 2, per (device, m, sign), kept for the process
int g_fy_tile = 0;  // transverse FFT rows per CTA override (smpm_batch_set_tuning(NULL, "fy_tile", v))

const double2* fy_twiddles(int m, int sign) {
  static std::vector<std::pair<long long, double*>> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  const long long key = (static_cast<long long>(dev) << 32) | (static_cast<long long>(m) << 1) | (sign > 0 ? 1 : 0);
  for (auto& e : cache)
    if (e.first == key) return reinterpret_cast<const double2*>(e.second);
  std::vector<double> h(static_cast<size_t>(m));
  for (int k = 0; k < m / 2; ++k) {
    const double ang = sign * 2.0 * M_PI * k / m;
    h[2 * k] = std::cos(ang);
    h[2 * k + 1] = std::sin(ang);
  }
  double* d = nullptr;
  CUDA_CHECK(cudaMalloc(&d, sizeof(double) * h.size()));
  CUDA_CHECK(cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  cache.emplace_back(key, d);
  return reinterpret_cast<const double2*>(d);
}

void fourier_launch(long long r, int m_y, const double* in, double* out, int sign, cudaStream_t st) {
  if (r < 1 || m_y < 2 || m_y > 4096 || (m_y & (m_y - 1)) != 0)
    fail(SMPM_EINVAL, "fourier_y: m_y must be a power of two in [2, 4096] and r >= 1");
  if (!in || !out) fail(SMPM_EINVAL, "null vector");
  FourierArgs a;
  a.r = r;
  a.m_y = m_y;
  // nodes per CTA: 16 (128-byte coalesced runs per plane) while the padded complex
  // tile stays <= 66 KB (3 CTAs per SM), fewer for long transforms
  a.tile = std::max(1, std::min(16, 4224 / (m_y + 1)));
  if (g_fy_tile > 0) a.tile = std::max(1, std::min(64, g_fy_tile));
  a.tw = fy_twiddles(m_y, sign);
  const size_t smem = sizeof(double2) * static_cast<size_t>(a.tile) * (m_y + 1);
  const unsigned grid = static_cast<unsigned>((r + a.tile - 1) / a.tile);
  auto go = [&](auto kfwd, auto kinv) {
    auto k = sign < 0 ? kfwd : kinv;
    CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k<<<grid, FY_THREADS, smem, st>>>(a, in, out);
  };
  switch (m_y) {  // register FFT for 64 <= m_y <= 512 (R = m_y / 32 per lane)
    case 64: go(fourier_y_kernel<2>, inverse_fourier_y_kernel<2>); break;
    case 128: go(fourier_y_kernel<4>, inverse_fourier_y_kernel<4>); break;
    case 256: go(fourier_y_kernel<8>, inverse_fourier_y_kernel<8>); break;
    case 512: go(fourier_y_kernel<16>, inverse_fourier_y_kernel<16>); break;
    default: go(fourier_y_kernel<0>, inverse_fourier_y_kernel<0>); break;
  }
  CUDA_CHECK(cudaGetLastError());
}

extern "C" {

const char* smpm_last_error(void) { return g_last_error.c_str(); }

const char* smpm_version(void) { return "smpm_b200 0.1 (sm_100a, fp64)"; }

int smpm_ctx_create(int device, smpm_ctx** out) {
  return guard([&] {
    if (!out) fail(SMPM_EINVAL, "null out");
    int ndev = 0;
    CUDA_CHECK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(SMPM_ECUDA, "no such CUDA device");
    CUDA_CHECK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) fail(SMPM_ECUDA, "smpm_b200 kernels are built for sm_100a; device is sm_" +
                                              std::to_string(prop.major) + std::to_string(prop.minor));
    auto ctx = std::make_unique<smpm_ctx>();
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    // blocking stream: orders with the legacy default stream torch uses for handle 0
    CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault));
    CUSOLVER_CHECK(cusolverDnCreate(&ctx->solver));
    CUSOLVER_CHECK(cusolverDnSetStream(ctx->solver, ctx->stream));
    CUDA_CHECK(cudaFuncSetAttribute(gemm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, G2_SMEM));
    *out = ctx.release();
  });
}

int smpm_ctx_destroy(smpm_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    if (ctx->solver) cusolverDnDestroy(ctx->solver);
    if (ctx->blas) cublasDestroy(ctx->blas);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

void* smpm_ctx_stream(smpm_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int smpm_batch_create(smpm_ctx* ctx, int n, int m_x, int m_z, int nsys, smpm_batch** out) {
  return guard([&] {
    if (!ctx || !out) fail(SMPM_EINVAL, "null argument");
    if (n < 2 || m_x < 2 || m_z < 1 || nsys < 1) fail(SMPM_EINVAL, "smpm_batch_create: need n>=2, m_x>=2, m_z>=1, nsys>=1");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    auto b = std::make_unique<smpm_batch>();
    b->ctx = ctx;
    b->n = n;
    b->mx = m_x;
    b->mz = m_z;
    b->nsys = nsys;
    b->w = n * m_z;
    b->d = m_x - 1;
    b->k = 2LL * b->w * b->d;
    b->nbf = b->d / 2;
    b->single = (b->d % 2) == 1;
    b->have.assign(static_cast<size_t>(nsys), 0);
    b->huS.assign(static_cast<size_t>(nsys), {});
    *out = b.release();
  });
}

int smpm_batch_destroy(smpm_batch* b) {
  return guard([&] { delete b; });
}

int smpm_batch_dims(const smpm_batch* b, long long* k, int* d, int* w) {
  return guard([&] {
    if (!b) fail(SMPM_EINVAL, "null batch");
    if (k) *k = b->k;
    if (d) *d = b->d;
    if (w) *w = b->w;
  });
}

int smpm_batch_set_couplings(smpm_batch* b, int sys, const double* G_W, const double* G_I, const double* G_E) {
  return guard([&] {
    if (!b || sys < 0 || sys >= b->nsys) fail(SMPM_EINVAL, "bad system index");
    if (b->finalized) fail(SMPM_EINVAL, "batch already finalized");
    if (!G_W || !G_E || (b->mx >= 3 && !G_I)) fail(SMPM_EINVAL, "null coupling matrix");
    const long long ww = 1LL * b->w * b->w;
    if (b->hG.empty()) b->hG.assign(static_cast<size_t>(b->nsys) * 6 * ww, 0.0);  // host staging, on first use
    double* dst = b->hG.data() + sys * 6 * ww;
    std::memcpy(dst, G_W, sizeof(double) * ww);
    if (G_I) std::memcpy(dst + ww, G_I, sizeof(double) * 4 * ww);
    std::memcpy(dst + 5 * ww, G_E, sizeof(double) * ww);
    b->have[sys] = 1;
  });
}

int smpm_batch_set_spectral(smpm_batch* b, int npairs, const double* T, const double* T_inv, const double* gamma) {
  return guard([&] {
    if (!b) fail(SMPM_EINVAL, "null batch");
    if (b->finalized) fail(SMPM_EINVAL, "batch already finalized");
    if (!T || !T_inv || !gamma) fail(SMPM_EINVAL, "null spectral factor");
    if (npairs < 0 || 2 * npairs > b->w) fail(SMPM_EINVAL, "bad number of complex pairs");
    const size_t ww = static_cast<size_t>(b->w) * b->w;
    b->sp_npairs = npairs;
    b->sp_nmode = b->w - npairs;
    b->hT.assign(T, T + ww);
    b->hTi.assign(T_inv, T_inv + ww);
    const size_t ng = static_cast<size_t>(b->nsys) * SK_NUM * b->sp_nmode * 2;
    b->hgam.assign(gamma, gamma + ng);
    b->spectral = true;
  });
}

int smpm_batch_load_schur_blocks(smpm_batch* b, int sys, const char* path) {
  return guard([&] {
    if (!b || !path) fail(SMPM_EINVAL, "null argument");
    std::FILE* fp = std::fopen(path, "rb");
    if (!fp) fail(SMPM_EINVAL, std::string("load_schur_blocks: cannot open ") + path);
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard_fp(fp, std::fclose);
    auto get = [&]() {
      std::int64_t v = 0;
      if (std::fread(&v, sizeof v, 1, fp) != 1) fail(SMPM_EINVAL, "load_schur_blocks: truncated file");
      return static_cast<long long>(v);
    };
    const long long n = get(), mx = get(), mz = get(), k = get();
    if (n != b->n || mx != b->mx || mz != b->mz || k != b->k)
      fail(SMPM_EINVAL, "load_schur_blocks: file geometry differs from the batch");
    const int d = b->d;
    std::vector<std::vector<double>> ent(d);
    std::vector<std::vector<long long>> st(d), ln(d);
    std::vector<long long> rows(d);
    std::vector<int> nseg(d);
    for (int i = 0; i < d; ++i) {
      rows[i] = get();
      const long long cols = get(), ns = get();
      if (cols != 2LL * b->w || rows[i] <= 0 || rows[i] > 4LL * b->w || ns < 1 || ns > 4)
        fail(SMPM_EINVAL, "load_schur_blocks: unexpected block shape");
      nseg[i] = static_cast<int>(ns);
      for (long long q = 0; q < ns; ++q) {
        st[i].push_back(get());
        ln[i].push_back(get());
      }
      ent[i].resize(static_cast<size_t>(rows[i] * cols));
      if (std::fread(ent[i].data(), sizeof(double), ent[i].size(), fp) != ent[i].size())
        fail(SMPM_EINVAL, "load_schur_blocks: truncated file");
    }
    std::vector<const double*> ep(d);
    std::vector<const long long*> sp(d), lp(d);
    for (int i = 0; i < d; ++i) {
      ep[i] = ent[i].data();
      sp[i] = st[i].data();
      lp[i] = ln[i].data();
    }
    const int rc = smpm_batch_set_interface_blocks(b, sys, ep.data(), rows.data(), sp.data(), lp.data(), nseg.data());
    if (rc != SMPM_OK) fail(rc, smpm_last_error());
  });
}

int smpm_batch_set_interface_blocks(smpm_batch* b, int sys, const double* const* entries, const long long* rows,
                                    const long long* const* seg_start, const long long* const* seg_len,
                                    const int* nseg) {
  return guard([&] {
    if (!b || sys < 0 || sys >= b->nsys) fail(SMPM_EINVAL, "bad system index");
    const int w = b->w, d = b->d;
    const long long w2 = 2LL * w, ww = 1LL * w * w;
    std::vector<double> GW(ww), GI(4 * ww, 0.0), GE(ww);
    std::vector<char> seenI(4, 0);
    // copy-and-verify helper: dst (ld) <- entries rows [r0,r0+w) x cols [c0,c0+w)
    auto take = [&](const double* e, long long nrows, long long r0, long long c0, double* dst, long long ld,
                    bool verify) {
      for (long long c = 0; c < w; ++c)
        for (long long r = 0; r < w; ++r) {
          const double v = e[(c0 + c) * nrows + r0 + r];
          double& t = dst[c * ld + r];
          if (verify && t != v) fail(SMPM_EINVAL, "interface blocks are not copies of strip-kind couplings");
          t = v;
        }
    };
    for (int i = 0; i < d; ++i) {
      const bool has_a = i >= 1, has_d = i <= d - 2;
      const int want = 2 + (has_a ? 1 : 0) + (has_d ? 1 : 0);
      if (nseg[i] != want || rows[i] != static_cast<long long>(want) * w)
        fail(SMPM_EINVAL, "interface block " + std::to_string(i) + " has an unexpected segment layout");
      long long off = 0;
      const double* e = entries[i];
      const long long nr = rows[i];
      int q = 0;
      if (has_a) {  // rows: W-readers of strip i, cols: E-own of strip i (interior)
        if (seg_start[i][q] != (i - 1) * w2) fail(SMPM_EINVAL, "segment start mismatch");
        take(e, nr, off, 0, GI.data() + w * w2, w2, seenI[1]);
        seenI[1] = 1;
        off += w;
        ++q;
      }
      // seg b: W-readers of strip i+1 x W-own of strip i+1 (cols w..2w)
      if (i + 1 == d) {
        take(e, nr, off, w, GE.data(), w, false);
      } else {
        take(e, nr, off, w, GI.data(), w2, seenI[0]);
        seenI[0] = 1;
      }
      off += w;
      // seg c: E-readers of strip i x E-own of strip i (cols 0..w)
      if (i == 0) {
        take(e, nr, off, 0, GW.data(), w, false);
      } else {
        take(e, nr, off, 0, GI.data() + w * w2 + w, w2, seenI[3]);
        seenI[3] = 1;
      }
      off += w;
      if (has_d) {  // E-readers of strip i+1 x W-own of strip i+1
        take(e, nr, off, w, GI.data() + w, w2, seenI[2]);
        seenI[2] = 1;
      }
      (void)seg_len;
    }
    const long long ww2 = ww;
    if (b->hG.empty()) b->hG.assign(static_cast<size_t>(b->nsys) * 6 * ww, 0.0);
    double* dst = b->hG.data() + sys * 6 * ww2;
    std::memcpy(dst, GW.data(), sizeof(double) * ww);
    std::memcpy(dst + ww, GI.data(), sizeof(double) * 4 * ww);
    std::memcpy(dst + 5 * ww, GE.data(), sizeof(double) * ww);
    b->have[sys] = 1;
  });
}

int smpm_batch_set_nullspace(smpm_batch* b, int sys, const double* u_S) {
  return guard([&] {
    if (!b || sys < 0 || sys >= b->nsys) fail(SMPM_EINVAL, "bad system index");
    if (b->finalized) fail(SMPM_EINVAL, "batch already finalized");
    if (!u_S) {
      b->huS[sys].clear();
      return;
    }
    b->huS[sys].assign(u_S, u_S + b->k);
  });
}

int smpm_batch_finalize(smpm_batch* b) {
  return guard([&] {
    if (!b) fail(SMPM_EINVAL, "null batch");
    CUDA_CHECK(cudaSetDevice(b->ctx->device));
    finalize(b);
  });
}

int smpm_batch_coarse_info(smpm_batch* b, double* C, int* tridiagonal, int* singular) {
  return guard([&] {
    need_final(b);
    if (C) std::copy(b->hC.begin(), b->hC.end(), C);
    if (tridiagonal) std::copy(b->htri.begin(), b->htri.end(), tridiagonal);
    if (singular) std::copy(b->hsing.begin(), b->hsing.end(), singular);
  });
}

#define OP_ENTRY(name, body)                                                         \
  int name(smpm_batch* b, const double* v, double* y, void* stream) {                \
    return guard([&] {                                                               \
      need_final(b);                                                                 \
      if (!v || !y) fail(SMPM_EINVAL, "null vector");                                \
      cudaStream_t st = b->st(stream);                                               \
      body;                                                                          \
    });                                                                              \
  }
OP_ENTRY(smpm_apply_S, op_S(b, v, y, all_systems(b), st))
OP_ENTRY(smpm_apply_St, op_St(b, v, y, all_systems(b), st))
OP_ENTRY(smpm_apply_block_jacobi_inv, op_BJ(b, v, y, all_systems(b), st))
OP_ENTRY(smpm_apply_Q, op_Q(b, v, y, all_systems(b), st))
OP_ENTRY(smpm_apply_Zt, launch_zt(b, v, y, st))
OP_ENTRY(smpm_apply_Z, launch_z(b, v, y, st))
OP_ENTRY(smpm_coarse_solve, run_deflate(b, DEFL_COARSE_DIRECT, v, nullptr, nullptr, y, all_systems(b), st))
#undef OP_ENTRY

int smpm_apply_P(smpm_batch* b, const double* v, double* y, int fused, void* stream) {
  return guard([&] {
    need_final(b);
    op_P(b, v, y, fused != 0, all_systems(b), b->st(stream));
  });
}

void store_strip_factors(smpm_batch* b, const smpm_strip_factors* f);

int smpm_batch_set_strip_factors(smpm_batch* b, const smpm_strip_factors* f) {
  return guard([&] {
    if (!b || !f) fail(SMPM_EINVAL, "null argument");
    if (!b->spectral || b->hT.empty()) fail(SMPM_EINVAL, "strip factors need the spectral basis (smpm_batch_set_spectral)");
    store_strip_factors(b, f);
  });
}

int smpm_batch_set_fdm(smpm_batch* b, int npairs, const double* T, const double* T_inv, const smpm_strip_factors* f) {
  return guard([&] {
    if (!b || !f) fail(SMPM_EINVAL, "null argument");
    if (b->finalized) fail(SMPM_EINVAL, "batch already finalized");
    if (!T || !T_inv) fail(SMPM_EINVAL, "null spectral basis");
    if (npairs < 0 || 2 * npairs > b->w) fail(SMPM_EINVAL, "bad number of complex pairs");
    if (b->w % 16 != 0) fail(SMPM_EINVAL, "smpm_batch_set_fdm needs w % 16 == 0 (use smpm_batch_set_couplings)");
    const int n = b->n, w = b->w;
    const size_t ww = static_cast<size_t>(w) * w;
    b->sp_npairs = npairs;
    b->sp_nmode = w - npairs;
    b->hT.assign(T, T + ww);
    b->hTi.assign(T_inv, T_inv + ww);
    b->spectral = true;
    if (b->mx >= 3) store_strip_factors(b, f);
    for (int kd = 0; kd < 3; ++kd)
      if (!f->Vx[kd] || !f->Vx_inv[kd] || !f->lx[kd]) fail(SMPM_EINVAL, "null x factor");
    if (!f->lz || !f->tW || !f->tE || !f->mu) fail(SMPM_EINVAL, "null strip factor");
    // a_kind[p] = (t_X . Vx[:, p]) Vx^{-1}[p, y_Y] for the six couplings (readers X, owner Y):
    // W_EE (west-boundary strip), I_WW, I_WE, I_EW, I_EE (interior strip), E_WW (east-boundary strip)
    const int strip_of[SK_NUM] = {0, 1, 1, 1, 1, 2};
    const int X_of[SK_NUM] = {1, 0, 0, 1, 1, 0}, Y_of[SK_NUM] = {1, 0, 1, 0, 1, 0};  // 0 = W, 1 = E
    b->fdm_a.assign(static_cast<size_t>(SK_NUM) * n * 2, 0.0);
    b->fdm_lx.assign(static_cast<size_t>(SK_NUM) * n * 2, 0.0);
    for (int kd = 0; kd < SK_NUM; ++kd) {
      const int sk = strip_of[kd];
      const double* tX = X_of[kd] ? f->tE : f->tW;
      const int y = Y_of[kd] ? n - 1 : 0;
      for (int p = 0; p < n; ++p) {
        double tr = 0.0, ti = 0.0;
        for (int ix = 0; ix < n; ++ix) {
          tr += tX[ix] * f->Vx[sk][2 * (ix + p * n)];
          ti += tX[ix] * f->Vx[sk][2 * (ix + p * n) + 1];
        }
        const double yr = f->Vx_inv[sk][2 * (p + y * n)], yi = f->Vx_inv[sk][2 * (p + y * n) + 1];
        b->fdm_a[2 * (kd * n + p)] = tr * yr - ti * yi;
        b->fdm_a[2 * (kd * n + p) + 1] = tr * yi + ti * yr;
        b->fdm_lx[2 * (kd * n + p)] = f->lx[sk][2 * p];
        b->fdm_lx[2 * (kd * n + p) + 1] = f->lx[sk][2 * p + 1];
      }
    }
    b->fdm_lz.assign(f->lz, f->lz + 2 * static_cast<size_t>(b->sp_nmode));
    b->fdm_mu.assign(f->mu, f->mu + b->nsys);
    b->fdm_tau = f->tau;
    b->from_fdm = true;
    std::fill(b->have.begin(), b->have.end(), 1);
  });
}

void store_strip_factors(smpm_batch* b, const smpm_strip_factors* f) {
  {
    if (b->mx < 3) fail(SMPM_EINVAL, "strip solver needs m_x >= 3");
    const int n = b->n;
    for (int kd = 0; kd < 3; ++kd)
      if (!f->Vx[kd] || !f->Vx_inv[kd] || !f->lx[kd]) fail(SMPM_EINVAL, "null x factor");
    if (!f->lz || !f->tW || !f->tE || !f->mu) fail(SMPM_EINVAL, "null strip factor");
    const int L = strip_fac_len(n);
    std::vector<double> fac(static_cast<size_t>(3) * L * 2);
    for (int kd = 0; kd < 3; ++kd) {
      double* o = fac.data() + static_cast<size_t>(kd) * L * 2;
      std::copy(f->Vx[kd], f->Vx[kd] + 2 * n * n, o);
      std::copy(f->Vx_inv[kd], f->Vx_inv[kd] + 2 * n * n, o + 2 * n * n);
      std::copy(f->lx[kd], f->lx[kd] + 2 * n, o + 4 * n * n);
      // tW Vx, tE Vx (row vector times the complex eigenvector matrix)
      for (int p = 0; p < n; ++p) {
        double wr = 0, wi = 0, er = 0, ei = 0;
        for (int ix = 0; ix < n; ++ix) {
          const double vr = f->Vx[kd][2 * (ix + p * n)], vi = f->Vx[kd][2 * (ix + p * n) + 1];
          wr += f->tW[ix] * vr;
          wi += f->tW[ix] * vi;
          er += f->tE[ix] * vr;
          ei += f->tE[ix] * vi;
        }
        o[4 * n * n + 2 * n + 2 * p] = wr;
        o[4 * n * n + 2 * n + 2 * p + 1] = wi;
        o[4 * n * n + 4 * n + 2 * p] = er;
        o[4 * n * n + 4 * n + 2 * p + 1] = ei;
      }
    }
    cudaStream_t st = b->ctx->stream;
    b->dsfac.upload(fac, st);
    b->dslz.upload(std::vector<double>(f->lz, f->lz + 2 * static_cast<size_t>(b->sp_nmode)), st);
    b->dsmu.upload(std::vector<double>(f->mu, f->mu + b->nsys), st);
    b->strip_tau = f->tau;
    CUDA_CHECK(cudaStreamSynchronize(st));
    b->strip_ok = true;
  }
}

int smpm_schur_rhs(smpm_batch* b, const double* f, double* b_S, void* stream) {
  return guard([&] {
    need_strip(b);
    if (!f || !b_S) fail(SMPM_EINVAL, "null vector");
    cudaStream_t st = b->st(stream);
    const StripParams P = strip_params(b);
    const long long tot = static_cast<long long>(b->nsys) * P.r;
    strip_gather_kernel<<<grid_for(tot), 256, 0, st>>>(P, f, nullptr, b->dsx1.p);
    check_launch(b);
    xf_columns(b, true, b->dsx1.p, b->dsx2.p, b->mx * b->n, P.r, st);
    strip_modes<true>(b, b->dsx2.p, b->dsbh.p, st);
    xf_columns(b, false, b->dsbh.p, b_S, 2 * b->d, b->k, st);
  });
}

int smpm_recover_solution(smpm_batch* b, const double* f, const double* x_S, double* u, void* stream) {
  return guard([&] {
    need_strip(b);
    if (!f || !x_S || !u) fail(SMPM_EINVAL, "null vector");
    cudaStream_t st = b->st(stream);
    const StripParams P = strip_params(b);
    const long long tot = static_cast<long long>(b->nsys) * P.r;
    strip_gather_kernel<<<grid_for(tot), 256, 0, st>>>(P, f, x_S, b->dsx1.p);
    check_launch(b);
    xf_columns(b, true, b->dsx1.p, b->dsx2.p, b->mx * b->n, P.r, st);
    strip_modes<false>(b, b->dsx2.p, b->dsx1.p, st);
    xf_columns(b, false, b->dsx1.p, b->dsx2.p, b->mx * b->n, P.r, st);
    strip_scatter_kernel<<<grid_for(tot), 256, 0, st>>>(P, b->dsx2.p, u);
    check_launch(b);
  });
}

int smpm_fourier_y(long long r, int m_y, const double* field, double* coeff, void* stream) {
  return guard([&] { fourier_launch(r, m_y, field, coeff, -1, static_cast<cudaStream_t>(stream)); });
}

int smpm_inverse_fourier_y(long long r, int m_y, const double* coeff, double* field, void* stream) {
  return guard([&] { fourier_launch(r, m_y, coeff, field, +1, static_cast<cudaStream_t>(stream)); });
}

int smpm_project_out(smpm_batch* b, long long len, const double* v, const double* dir, double* out, void* stream) {
  return guard([&] {
    need_final(b);
    // any per-system length: interface vectors (u_S on b_S, len = k) or node
    // vectors (u_L on f, len = r; proj/src/solver.cpp:46, proj/src/helmholtz.cpp:159-160)
    if (len < 1) fail(SMPM_EINVAL, "smpm_project_out: len must be >= 1");
    if (!v || !dir || !out) fail(SMPM_EINVAL, "null vector");
    cudaStream_t st = b->st(stream);
    double* dots = b->dsmall.p;
    batched_dot(b, dir, v, dots, nullptr, st, len);
    project_kernel<<<grid_for(b->nsys * len), 256, 0, st>>>(b->nsys, len, dots, v, dir, out);
    check_launch(b);
  });
}

int smpm_solve(smpm_batch* b, int method, const double* b_S, double* x_S, const smpm_solve_options* opt,
               smpm_report* reports, double* history, void* stream) {
  return guard([&] {
    need_final(b);
    if (!b_S || !x_S) fail(SMPM_EINVAL, "null vector");
    solve(b, cfg_from(method, opt), b_S, x_S, reports, history, b->st(stream));
  });
}

int smpm_deflated_solve(smpm_batch* b, const double* b_S, double* x_S, const smpm_solve_options* opt,
                        smpm_report* reports, double* history, void* stream) {
  return smpm_solve(b, SMPM_DBJ, b_S, x_S, opt, reports, history, stream);
}

int smpm_two_level_schwarz_solve(smpm_batch* b, const double* b_S, double* x_S, const smpm_solve_options* opt,
                                 smpm_report* reports, double* history, void* stream) {
  return smpm_solve(b, SMPM_2LAS, b_S, x_S, opt, reports, history, stream);
}

int smpm_solve_stacked(smpm_batch* b, int method, const double* b_S, double* x_S, const smpm_solve_options* opt,
                       smpm_report* report, double* history, void* stream) {
  return guard([&] {
    need_final(b);
    if (!b_S || !x_S) fail(SMPM_EINVAL, "null vector");
    if (method != SMPM_DBJ && method != SMPM_2LAS) fail(SMPM_EINVAL, "stacked solve: dbj or 2las");
    SolveCfg c = cfg_from(method, opt);
    c.stacked = true;
    // every system carries the same (global) report and history: keep one
    std::vector<smpm_report> reps(static_cast<size_t>(b->nsys));
    const int cap = static_cast<int>(std::min<long long>(c.max_iter, b->k)) + 2;  // solve's history stride
    std::vector<double> hist(history ? static_cast<size_t>(b->nsys) * cap : 0);
    solve(b, c, b_S, x_S, reps.data(), history ? hist.data() : nullptr, b->st(stream));
    if (report) *report = reps[0];
    if (history) std::copy(hist.begin(), hist.begin() + cap, history);
  });
}

int smpm_solve_host(smpm_batch* b, int method, const double* b_S_host, double* x_S_host,
                    const smpm_solve_options* opt, smpm_report* reports, double* history) {
  return guard([&] {
    need_final(b);
    cudaStream_t st = b->ctx->stream;
    const size_t bytes = sizeof(double) * b->nsys * static_cast<size_t>(b->k);
    double* din = b->vbuf[10].p;
    double* dout = b->vbuf[11].p;
    // an upload started ahead by smpm_prefetch_rhs for this host buffer: wait for it instead of copying
    // (the older of two outstanding uploads of the same buffer first: slot pf_next is the next to be refilled)
    int hit = -1;
    for (int i = 0; i < 2 && hit < 0; ++i) {
      const int q = (b->pf_next + i) & 1;
      if (b_S_host && b->pf_host[q] == b_S_host) hit = q;
    }
    if (hit >= 0) {
      CUDA_CHECK(cudaStreamWaitEvent(st, b->pfev[hit], 0));
      din = b->dpf[hit].p;
      b->pf_host[hit] = nullptr;
    } else {
      CUDA_CHECK(cudaMemcpyAsync(din, b_S_host, bytes, cudaMemcpyHostToDevice, st));
    }
    solve(b, cfg_from(method, opt), din, dout, reports, history, st, x_S_host);
    CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int smpm_prefetch_rhs(smpm_batch* b, const double* b_S_host) {
  return guard([&] {
    need_final(b);
    if (!b_S_host) fail(SMPM_EINVAL, "null right-hand side");
    const size_t n = static_cast<size_t>(b->nsys) * static_cast<size_t>(b->k);
    if (!b->st3) {
      CUDA_CHECK(cudaStreamCreateWithFlags(&b->st3, cudaStreamNonBlocking));
      for (auto& e : b->pfev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int q = b->pf_next;
    b->pf_next ^= 1;
    b->dpf[q].alloc(n);
    CUDA_CHECK(cudaMemcpyAsync(b->dpf[q].p, b_S_host, sizeof(double) * n, cudaMemcpyHostToDevice, b->st3));
    CUDA_CHECK(cudaEventRecord(b->pfev[q], b->st3));
    b->pf_host[q] = b_S_host;
  });
}

long long smpm_batch_launch_count(const smpm_batch* b) { return b ? b->launches : 0; }

int smpm_batch_set_tuning(smpm_batch* b, const char* key, long long value) {
  return guard([&] {
    if (!key) fail(SMPM_EINVAL, "null tuning key");
    const std::string k(key);
    if (!b) {
      if (k == "fy_tile") {
        g_fy_tile = static_cast<int>(value);
        return;
      }
      fail(SMPM_EINVAL, "null batch");
    }
    Tuning& t = b->tune;
    const int v = static_cast<int>(value);
    struct Knob {
      const char* name;
      int* field;
    };
    if (k == "tail_rows") {
      t.tail_rows = value;
      return;
    }
    const Knob knobs[] = {{"segb", &t.segb}, {"spec_v2", &t.spec_v2}, {"xform", &t.xform}, {"xform_parity", &t.xform_parity}, {"xform_ws", &t.xform_ws}, {"xform_ares", &t.xform_ares},
                          {"sp_stage", &t.sp_stage},
                          {"spectral", &t.spectral}, {"spec_2las", &t.spec_2las}, {"p2fuse", &t.p2fuse}, {"cgs_defer", &t.cgs_defer}, {"cgs_lanes", &t.cgs_lanes},
                          {"gt_vblock", &t.gt_vblock}, {"grid_per_sm", &t.grid_per_sm}, {"gt_ctas", &t.gt_ctas}, {"coarse_fork", &t.coarse_fork},
                          {"grid_nocoop", &t.grid_nocoop}, {"pdl", &t.pdl}, {"pythag", &t.pythag},
                          {"grid", &t.grid}, {"grid_max", &t.grid_max}, {"post_fuse", &t.post_fuse},
                          {"early", &t.early}};
    for (const Knob& kb : knobs)
      if (k == kb.name) {
        *kb.field = v;
        // grid geometry and transform plans depend on some knobs: recompute lazily
        if (k == "gt_vblock" || k == "grid_per_sm" || k == "gt_ctas") b->gt_blocks = 0;
        if ((k == "xform" || k == "xform_parity" || k == "xform_ares") && b->finalized && b->spectral) setup_xform(b);
        return;
      }
    fail(SMPM_EINVAL, "unknown tuning key '" + k + "'");
  });
}

int smpm_batch_set_allreduce(smpm_batch* b, smpm_allreduce_fn fn, void* user) {
  return guard([&] {
    if (!b) fail(SMPM_EINVAL, "null batch");
    b->ar_fn = fn;
    b->ar_user = user;
    if (fn) b->dstack.alloc(static_cast<size_t>(V2_MAXCOL + 2));
  });
}

int smpm_batch_query(const smpm_batch* b, const char* key, long long* value) {
  return guard([&] {
    if (!b || !key || !value) fail(SMPM_EINVAL, "null argument");
    const std::string k(key);
    if (k == "xform_kernel")
      *value = !b->spectral || b->xf_P == 0 ? 0 : b->xp_on ? 3 : b->xf_stream ? 2 : 1;
    else if (k == "xform_parity")
      *value = b->spectral && b->xp_on ? 1 : 0;
    else if (k == "cgs_defer")
      *value = b->tune.cgs_defer && b->tune.pythag ? 1 : 0;
    else if (k == "spectral")
      *value = b->spectral && b->tune.spectral ? 1 : 0;
    else
      fail(SMPM_EINVAL, "unknown query key '" + k + "'");
  });
}

int smpm_batch_set_trace(smpm_batch* b, int which, const char* path) {
  return guard([&] {
    if (!b) fail(SMPM_EINVAL, "null batch");
    if (which == 0)
      b->tune.gt_trace = path ? path : "";
    else if (which == 1)
      b->tune.gt_trace2 = path ? path : "";
    else
      fail(SMPM_EINVAL, "trace: which must be 0 (per-step phases) or 1 (per-CTA)");
  });
}

int smpm_batch_profile(smpm_batch* b, int enable, double* ms, long long* counts, int nclass) {
  return guard([&] {
    if (!b) fail(SMPM_EINVAL, "null batch");
    CUDA_CHECK(cudaStreamSynchronize(b->ctx->stream));
    prof_collect(b);
    if (ms)
      for (int i = 0; i < std::min(nclass, 10); ++i) ms[i] = b->prof_ms[i];
    if (counts)
      for (int i = 0; i < std::min(nclass, 10); ++i) counts[i] = b->prof_n[i];
    if (enable >= 0) {
      b->profiling = enable != 0;
      for (int i = 0; i < 10; ++i) {
        b->prof_ms[i] = 0.0;
        b->prof_n[i] = 0;
      }
    }
  });
}

}  // extern "C"
