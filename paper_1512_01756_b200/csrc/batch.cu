// Host side of the B200 Schur-GMRES library: batch setup (uploads, the
// structured block-Jacobi inverses, coarse spaces), the precomputed GEMM job
// plans of every operator, the batched GMRES driver and the C ABI declared in
// include/smpm_b200.h.
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/smpm_b200.h"
#include "common.cuh"
#include "gemm.cuh"
#include "gemm2.cuh"
#include "vec.cuh"
#include "vec2.cuh"
#include "vec3.cuh"
#include "vec4.cuh"
#include "grid.cuh"
#include "spectral.cuh"
#include "spectral3.cuh"
#include "xform.cuh"
#include "xformk.cuh"
#include "xformp.cuh"
#include "xformq.cuh"
#include "strip.cuh"
#include "fourier.cuh"

using namespace smpm;

namespace {

thread_local std::string g_last_error;

struct SmpmError : std::runtime_error {
  int code;
  SmpmError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& m) { throw SmpmError(code, m); }

#define CUDA_CHECK(x)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(SMPM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define CUSOLVER_CHECK(x)                                                        \
  do {                                                                           \
    cusolverStatus_t s_ = (x);                                                   \
    if (s_ != CUSOLVER_STATUS_SUCCESS) fail(SMPM_ECUDA, std::string(#x) + " failed"); \
  } while (0)

template <class F>
int guard(F&& f) {
  try {
    f();
    return SMPM_OK;
  } catch (const SmpmError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SMPM_ERUNTIME;
  }
}

template <class T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray() = default;
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  ~DevArray() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void upload(const std::vector<T>& h, cudaStream_t st) {
    alloc(h.size());
    if (!h.empty()) CUDA_CHECK(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  }
};

View view(int buf, long long off, long long cs = 0, int split = INT_MAX, long long soff = 0) {
  View v;
  v.buf = buf;
  v.off = off;
  v.cs = cs;
  v.split = split;
  v.soff = soff;
  return v;
}
const View kNoView = view(BUF_NONE, 0);

// One GEMM launch worth of jobs (+ split-K reduction items).
struct Plan {
  std::vector<GemmJob> jobs;
  DevArray<GemmJob> djobs;
  DevArray<GemmTile> dtiles;
  DevArray<SplitItem> ditems;
  int ntiles = 0, nitems = 0, ngemm = 0;
  long long ws_tiles = 0;
  DevArray<Tile2> dgv;  // GEMV jobs as GT_GVR-row cluster items (grid tail solver)
  int ngv = 0;
  bool v2 = false;  // hot-path kernel (DMMA tiles + GEMV tiles)
  bool shared_a = false;  // every system uses the same matrices (no per-system stride)
  DevArray<Tile2> dtiles2;

  // v2 plan: N >= 2 jobs as 64x32 DMMA tiles (split-K when the plan has too
  // few tiles for the GPU), N == 1 jobs as 32-row GEMV tiles
  std::unique_ptr<Plan> tail;  // split-K variant for the few-systems tail (v2 only)

  void build2(int num_sms, cudaStream_t st, int force_split = 0) {
    long long tiles = 0;
    for (const auto& j : jobs)
      if (j.N >= 2) tiles += static_cast<long long>((j.M + G2_BM - 1) / G2_BM) * ((j.N + G2_BN - 1) / G2_BN);
    int split = 1;
    if (tiles > 0 && tiles < 2LL * num_sms) split = static_cast<int>((2LL * num_sms + tiles - 1) / tiles);
    if (force_split > 0) split = std::max(split, force_split);
    std::vector<Tile2> ht;
    std::vector<SplitItem> hi;
    ws_tiles = 0;
    for (size_t ji = 0; ji < jobs.size(); ++ji) {
      GemmJob& j = jobs[ji];
      j.splitk = 1;
      j.ws_off = 0;
      if (j.N == 1) {
        for (int m0 = 0; m0 < j.M; m0 += GV_ROWS) ht.push_back(Tile2{static_cast<int>(ji), m0, 0, -1});
        continue;
      }
      const int mt = (j.M + G2_BM - 1) / G2_BM, nt = (j.N + G2_BN - 1) / G2_BN;
      j.splitk = std::max(1, std::min(split, j.K / (4 * G2_BK)));
      if (j.splitk > 1) {
        j.ws_off = static_cast<int>(ws_tiles);
        ws_tiles += static_cast<long long>(mt) * nt * j.splitk;
      }
      for (int a = 0; a < mt; ++a)
        for (int b = 0; b < nt; ++b) {
          for (int ks = 0; ks < j.splitk; ++ks) ht.push_back(Tile2{static_cast<int>(ji), a * G2_BM, b * G2_BN, ks});
          if (j.splitk > 1) hi.push_back(SplitItem{static_cast<int>(ji), a * G2_BM, b * G2_BN});
        }
    }
    // GEMM tiles first (long), GEMV tiles last
    std::stable_sort(ht.begin(), ht.end(), [](const Tile2& x, const Tile2& y) { return (x.ks < 0) < (y.ks < 0); });
    ntiles = static_cast<int>(ht.size());
    ngemm = static_cast<int>(std::count_if(ht.begin(), ht.end(), [](const Tile2& x) { return x.ks >= 0; }));
    nitems = static_cast<int>(hi.size());
    v2 = true;
    djobs.upload(jobs, st);
    dtiles2.upload(ht, st);
    ditems.upload(hi, st);
  }

  // the v2 kernel needs 16-byte aligned operands and unsplit B views
  bool v2_ok() const {
    for (const auto& j : jobs) {
      if ((reinterpret_cast<uintptr_t>(j.A) & 15) || (j.lda & 1) || j.transA) return false;
      if (j.b.split != INT_MAX || (j.b.off & 1) || (j.b.cs & 1)) return false;
    }
    return true;
  }

  void add(const double* A, long long lda, bool transA, int M, int N, int K, int sys, View b, View out, View addv,
           double alpha, double beta) {
    if (M <= 0 || N <= 0 || K <= 0) return;
    GemmJob j{};
    j.A = A;
    j.lda = lda;
    j.transA = transA ? 1 : 0;
    j.M = M;
    j.N = N;
    j.K = K;
    j.sys = sys;
    j.splitk = 1;
    j.b = b;
    j.out = out;
    j.add = addv;
    j.alpha = alpha;
    j.beta = beta;
    jobs.push_back(j);
  }

  // split-K when the plan has too few output tiles to fill the GPU
  void build(int num_sms, cudaStream_t st) {
    long long tiles = 0;
    for (const auto& j : jobs)
      tiles += static_cast<long long>((j.M + GEMM_BM - 1) / GEMM_BM) * ((j.N + GEMM_BN - 1) / GEMM_BN);
    int split = 1;
    if (tiles > 0 && tiles < 2LL * num_sms) split = static_cast<int>((2LL * num_sms + tiles - 1) / tiles);
    std::vector<GemmTile> ht;
    std::vector<SplitItem> hi;
    ws_tiles = 0;
    for (size_t ji = 0; ji < jobs.size(); ++ji) {
      GemmJob& j = jobs[ji];
      const int mt = (j.M + GEMM_BM - 1) / GEMM_BM, nt = (j.N + GEMM_BN - 1) / GEMM_BN;
      j.splitk = std::max(1, std::min(split, j.K / (4 * GEMM_BK)));
      j.ws_off = 0;
      if (j.splitk > 1) {
        j.ws_off = static_cast<int>(ws_tiles);
        ws_tiles += static_cast<long long>(mt) * nt * j.splitk;
      }
      for (int a = 0; a < mt; ++a)
        for (int b = 0; b < nt; ++b) {
          for (int ks = 0; ks < j.splitk; ++ks) ht.push_back(GemmTile{static_cast<int>(ji), a * GEMM_BM, b * GEMM_BN, ks});
          if (j.splitk > 1) hi.push_back(SplitItem{static_cast<int>(ji), a * GEMM_BM, b * GEMM_BN});
        }
    }
    ntiles = static_cast<int>(ht.size());
    nitems = static_cast<int>(hi.size());
    djobs.upload(jobs, st);
    dtiles.upload(ht, st);
    ditems.upload(hi, st);
  }
};

}  // namespace

struct smpm_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cublasHandle_t blas = nullptr;  // plain library GEMMs of the strip solver when the transform kernel does not apply
};

// Performance knobs and diagnostics of one batch (smpm_batch_set_tuning). The
// defaults are the measured-best settings; nothing here changes results except
// the switches documented as evaluation-order changes (pythag, p2fuse).
struct Tuning {
  int segb = 0;          // per-mode pass: blocks per warp item (0: SP_SEGB)
  int xform = 1;         // resident-slice transform kernel (xform.cuh) where it applies
  int xform_ws = 2;      // parity transforms: 0 CTA barrier per stage (xformp.cuh); 2 / 3 producer warp + mbarrier ring
                         // with that many consumer warpgroups (xformq.cuh; 2 measured best)
  int xform_ares = 1;    // parity transforms keep the slice's matrix resident in shared memory when it fits (small w)
  int xform_parity = 1;  // parity-split transforms (xformp.cuh) when T is parity-pure: 0 off, 1 where the
                         // K-streamed kernel would run (w > 176), 2 wherever w % 16 == 0
  int sp_stage = 1;      // per-mode pass stages slot rows in shared memory (spec_v2 = 0)
  int spec_v2 = 2;       // pipelined per-mode pass: 2 spec_op3_kernel (16 bytes per lane), 1 spec_op2_kernel, 0 staged
  int spectral = 1;      // spectral operator when its factors are set
  int spec_2las = 1;     // spectral operator for 2LAS
  int p2fuse = 1;        // CGS2 pass 2 single-read fusion
  int cgs_lanes = 1;     // CGS2 passes beyond 16 columns: eight lanes per row in registers (vec4.cuh) instead of
                         // shared-memory row tiles
  int cgs_defer = 1;     // CGS2 reorthogonalisation update deferred into the next pass 1 (vec4.cuh): 2 reads of V
  int gt_vblock = 2;     // grid tail V-row block: 0 off, 1 ring size, 2 as large as 2 CTAs/SM allow
  int grid_per_sm = 2;   // grid tail CTAs per SM (cap)
  int gt_ctas = 0;       // grid tail CTA cap (0: none)
  int coarse_fork = 1;   // per-stage steps: coarse solve on a side stream beside the T transform
  int grid_nocoop = 0;   // opt-in: plain (non-cooperative) cluster launch of the tail, for profilers only
  int pdl = -1;          // programmatic dependent launch of the step chain: 1 on, 0 off, -1 auto (on for k <= 100,000)
  int pythag = 1;        // norm from the second CGS2 reduction
  int grid = 1;          // grid-persistent tail
  int grid_max = 8;      // live systems at which the tail takes over
  long long tail_rows = 200000;  // ... and at most this many live interface rows (0: no cap)
  int post_fuse = 1;     // one-pass dbj epilogue
  int early = 1;         // early epilogue + x_S copy during the tail (solve_host)
  std::string gt_trace, gt_trace2;  // phase-trace dump files of the grid tail
};

struct smpm_batch {
  smpm_ctx* ctx = nullptr;
  Tuning tune;
  int n = 0, mx = 0, mz = 0, nsys = 0, w = 0, d = 0;
  long long k = 0;
  int nbf = 0;       // block-Jacobi blocks covering two interfaces
  bool single = false;  // trailing one-interface block (d odd)
  bool finalized = false;

  // host staging, per system: GW (w*w) | GI (4w*w) | GE (w*w)
  std::vector<double> hG;
  std::vector<char> have;
  std::vector<std::vector<double>> huS;

  // device matrix pool, per system: GW GI GE | K variants (inverses)
  DevArray<double> dmat;
  long long mstride = 0;
  long long oGW = 0, oGI = 0, oGE = 0, oK[4] = {0, 0, 0, 0}, oKs = 0;  // K: [first][last] flags -> index
  bool kneeded[4] = {false, false, false, false};

  // coarse space
  DevArray<double> dcinv, duc, dthomas, drowsum;
  DevArray<int> dcmode, dsingular;
  std::vector<double> hC;
  std::vector<int> htri, hsing;

  // operator plans
  Plan pS, pSt, pBJ1, pBJ2, pBJ3;
  // spectral form (spectral.cuh): T^{-1} / T transforms and per-mode factors
  bool spectral = false;
  int sp_npairs = 0, sp_nmode = 0;
  std::vector<double> hT, hTi, hgam;
  DevArray<double> dT, dTi, domega, dnu, dgam, dzpart, dvh, dvh2, dth, dkinv;
  Plan pF, pB;
  DevArray<double> dTfrag, dTifrag;    // T, T^{-1} in the xform fragment order
  int xf_P = 0, xf_MB = 0;
  bool xf_stream = false;  // K-streamed transform kernel (xformk.cuh) instead of the resident slice
  // parity-split transforms (xformp.cuh): forward = T^{-1}, backward = T
  bool xp_on = false;
  int xp_h = 0, xp_ks = 0, xp_seg_start[2][2] = {{0, 0}, {0, 0}}, xp_seg_len0[2] = {0, 0};
  // slicing variants per direction ([0] forward = T^{-1}, [1] backward = T): more, thinner row slices
  // for launches with few columns (the slow-mode tail), so every SM still gets a full 64-column chunk
  struct XpVariant {
    int P = 0, MB = 0;  // row slices (forward: both parities), m-blocks per slice
    size_t ares_smem = 0;  // > 0: the slice's matrix fits in shared memory next to a ring of column slabs
    DevArray<double> img;
  };
  std::vector<std::unique_ptr<XpVariant>> xp_var[2];
  long long cgs3_res = 0;  // resident CTAs of the CGS2 pass kernels (device)
  long long cgs3_kres[3] = {0, 0, 0};  // per kernel: pass 1, pass 2', pass 3' (norm-from-h2 path)
  long long p2t_res[V2_MAXCOL + 1] = {};  // resident CTAs of the tiled pass 2' per column capacity
  bool p2t_attr = false;
  int jhost = 0;  // Arnoldi index of the next step (all live systems of a cycle share it)
  // device-side fast-diagonalisation setup (smpm_batch_set_fdm): couplings, block inverses
  // and row sums are built on the device from the spectral data at finalize
  bool from_fdm = false;
  std::vector<double> fdm_a, fdm_lx, fdm_lz, fdm_mu;  // 6 x n, 6 x n, nmode (complex), nsys
  double fdm_tau = 0.0;
  // stacked solve across ranks: the caller's all-reduce (NCCL over NVLink) and its buffer
  smpm_allreduce_fn ar_fn = nullptr;
  void* ar_user = nullptr;
  DevArray<double> dstack;
  bool pending = false;  // deferred CGS2: the newest basis vector is still the pending pair (w', h2) (vec4.cuh)
  bool p1bt_attr = false;
  long long p1b_res = 0, p1bt_res[V2_MAXCOL + 1] = {};  // resident CTAs of the pass 1B kernels
  long long p2l_res[2] = {0, 0}, p1bl_res[2] = {0, 0};  // ... of the lane-shared-row kernels ([1]: > 64 columns)
  bool pythag = true;  // norm from the second CGS2 reduction (cgs3_pass2n / cgs3_pass3s); tuning pythag
  bool pdl = true;  // programmatic dependent launch for the Arnoldi step chain (tuning pdl)
  size_t xf_smem = 0;
  Plan pc[6];          // unsplit per-system templates (BJ1, BJ2, BJ3, S; spectral F, B) for the persistent solvers
  bool tmpl_ok = false;  // unsplit per-system templates of the hot stages exist (grid tail)
  DevArray<double> dws;  // split-K workspace
  // grid-persistent tail solver (grid.cuh)
  bool grid_ok = false;
  int gt_blocks = 0;
  bool sp_smem_set = false;
  size_t gt_smem = 0;  // tail dynamic shared memory (tile ring / V-row block region + vectors)
  int gt_vcap = 0;     // doubles of the ring / V-row block region
  DevArray<unsigned> dgbar;   // grid barrier counter
  bool gbar_clean = false;    // zeroed by the solve prologue (gm_v0_kernel), no tail launched since
  DevArray<double> dgtpart, dgtzsum, dgtzp, dgtcg;

  // vectors (nsys x k each)
  DevArray<double> vbuf[12];
  DevArray<double> dsmall;  // nsys x (d + misc) scalars
  DevArray<double> dcoarse;  // Z^T sums and coarse solutions, 2 x nsys x d
  DevArray<double> dczb;     // nsys x d: C^{-1} Z^T b_S of the current solve (dbj)
  DevArray<double> dsnsq;    // nsys: per-system ||w||^2 of the stacked solve's norm pass
  // strip solver (strip.cuh): x-factor per strip kind, z eigenvalues, shifts; scratch strip rows
  bool strip_ok = false;
  double strip_tau = 0.0;
  DevArray<double> dsfac, dslz, dsmu, dsx1, dsx2, dsbh;
  DevArray<double> dpost;    // nsys x 64: post-loop partial sums
  DevArray<int> dones, dcount, dsel, dcnt;
  DevArray<int> dalist;  // two compacted live lists + counts: [alist, acount, alist2, acount2]
  int* hcnt = nullptr;      // pinned + mapped, 4 ints (two in-flight step counters)
  int* hcnt_dev = nullptr;  // device alias of hcnt: compact_kernel writes the counters straight to the host
  void* hrep = nullptr;  // pinned + mapped report staging (written by report_pack_kernel)
  void* hrep_dev = nullptr;  // its device alias
  size_t hrep_bytes = 0;
  cudaEvent_t sev[4] = {nullptr, nullptr, nullptr, nullptr};  // solve events (timing x2, step polling x2)
  // early epilogue: the systems already stopped when the grid tail starts are finished
  // (x' = V y, M^{-1}, residual, x_S) on a side stream while the tail runs
  cudaStream_t st2 = nullptr;
  cudaStream_t st4 = nullptr;              // coarse solves beside the T transform (spec_SMinv)
  cudaEvent_t cfev[2] = {nullptr, nullptr};
  DevArray<double> dzsum;                  // nsys x d coarse right-hand sides for that kernel
  cudaEvent_t eev[3] = {nullptr, nullptr, nullptr};  // early list ready, early epilogue done, host copy done
  // right-hand sides uploaded ahead of their solve (smpm_prefetch_rhs): two device buffers in turn
  DevArray<double> dpf[2];
  cudaStream_t st3 = nullptr;
  cudaEvent_t pfev[2] = {nullptr, nullptr};
  const double* pf_host[2] = {nullptr, nullptr};
  int pf_next = 0;
  int* hearly = nullptr;      // pinned + mapped: nsys flags of the early set (read by solve_host)
  int* hearly_dev = nullptr;
  DevArray<int> dearly;       // [early flags, early list, count, late flags, late list, count]
  ~smpm_batch() {
    for (auto e : sev)
      if (e) cudaEventDestroy(e);
    for (auto e : eev)
      if (e) cudaEventDestroy(e);
    if (st2) cudaStreamDestroy(st2);
    if (st4) cudaStreamDestroy(st4);
    for (auto e : cfev)
      if (e) cudaEventDestroy(e);
    if (hearly) cudaFreeHost(hearly);
    if (hcnt) cudaFreeHost(hcnt);
    if (hrep) cudaFreeHost(hrep);
    for (auto e : ev_pool) cudaEventDestroy(e);
  }
  DevArray<double> dpart;

  // GMRES workspace
  int gm_m = -1, gm_hist = 0, gm_mtot = 0;
  DevArray<double> dV, dR, dcs, dsn, dg, dh1, dh2, dy, dhist, dgpart, dscal;
  DevArray<int> dgint;
  GmState_ G{};

  long long launches = 0;

  // optional per-class device timing (CUDA events on the launching stream)
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Span {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Span> spans;
  double prof_ms[10] = {};  // per kernel class (see PROFILE_CLASSES in _lib.py)
  long long prof_n[10] = {};

  cudaStream_t st(void* s) const { return s ? static_cast<cudaStream_t>(s) : ctx->stream; }
  double* GW(int s) const { return dmat.p + s * mstride + oGW; }
  double* GI(int s) const { return dmat.p + s * mstride + oGI; }
  double* GE(int s) const { return dmat.p + s * mstride + oGE; }
  double* Kinv(int s, int v) const { return dmat.p + s * mstride + oK[v]; }
  double* Ksingle(int s) const { return dmat.p + s * mstride + oKs; }
};

// out = A in for every w-long column of nsys x ncol_sys columns (defined with the strip solver below)
void xf_columns(smpm_batch* b, bool inverse, const double* in, double* out, int ncol_sys, long long sys_stride,
                cudaStream_t st, int nsys_ = -1);

namespace {

void check_launch(smpm_batch* b) {
  ++b->launches;
  CUDA_CHECK(cudaGetLastError());
}

// launch `kern` with programmatic stream serialization (common.cuh pdl_wait /
// pdl_launch): used for the kernel chain of an Arnoldi step
template <typename... KArgs, typename... Args>
void launch_pdl(smpm_batch* b, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = b->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
  check_launch(b);
}

// kernel classes for the optional timing
enum ProfClass : int { PC_SCHUR = 0, PC_BJ = 1, PC_DEFL = 2, PC_ORTH = 3, PC_OTHER = 4 };

cudaEvent_t prof_event(smpm_batch* b) {
  if (b->ev_used == b->ev_pool.size()) {
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreate(&e));
    b->ev_pool.push_back(e);
  }
  return b->ev_pool[b->ev_used++];
}

struct ProfScope {
  smpm_batch* b;
  int cls;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(smpm_batch* b_, int c, cudaStream_t s) : b(b_), cls(c), st(s) {
    if (b->profiling) {
      a = prof_event(b);
      CUDA_CHECK(cudaEventRecord(a, st));
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t e = prof_event(b);
      cudaEventRecord(e, st);
      b->spans.push_back({cls, a, e});
    }
  }
};

// resolve recorded spans (call after the stream is synchronized)
void prof_collect(smpm_batch* b) {
  for (const auto& s : b->spans) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, s.a, s.b) == cudaSuccess) {
      b->prof_ms[s.cls] += ms;
      b->prof_n[s.cls] += 1;
    }
  }
  b->spans.clear();
  b->ev_used = 0;
}

// The systems an operator application runs on: a device-compacted list of
// live systems (alist/acount, grids sized by an upper bound nslots), or all
// systems (alist == nullptr).  `active` is the matching per-system mask for
// the kernels that take masks.
void setup_xform(smpm_batch* b);

struct Live {
  const int* alist = nullptr;
  const int* acount = nullptr;
  int nslots = 0;
  const int* active = nullptr;
};
Live all_systems(const smpm_batch* b) {
  Live l;
  l.nslots = b->nsys;
  return l;
}

constexpr int kTailSystems = 8;

void run_plan(smpm_batch* b, Plan& p0, const double* in, double* out, double* tmp, const Live& lv, cudaStream_t st) {
  Plan& p = (p0.v2 && p0.tail && lv.nslots <= kTailSystems && lv.alist) ? *p0.tail : p0;
  if (p.ntiles == 0 || lv.nslots == 0) return;
  BufTable t;
  t.p[BUF_IN] = const_cast<double*>(in);
  t.p[BUF_OUT] = out;
  t.p[BUF_TMP] = tmp;
  t.p[BUF_TMP2] = nullptr;
  if (p.v2) {
    // per-system templates: launch only the tiles of the (bounded) live systems
    SysMap sm;
    sm.alist = lv.alist;
    sm.acount = lv.acount;
    sm.tiles_per_sys = p.ntiles;
    sm.a_stride = p0.shared_a ? 0 : b->mstride;
    sm.v_stride = b->k;
    sm.ws_stride = p.ws_tiles;
    gemm2_kernel<<<p.ntiles * lv.nslots, G2_THREADS, G2_SMEM, st>>>(p.djobs.p, p.dtiles2.p, t, sm, b->dws.p);
    check_launch(b);
    if (p.nitems > 0) {
      gemm2_splitk_reduce_kernel<<<p.nitems * lv.nslots * G2_RED_PARTS, 256, 0, st>>>(p.djobs.p, p.ditems.p, p.nitems, t, sm,
                                                                       b->dws.p);
      check_launch(b);
    }
    return;
  }
  gemm_jobs_kernel<<<p.ntiles, 128, 0, st>>>(p.djobs.p, p.dtiles.p, t, lv.active, b->dws.p);
  check_launch(b);
  if (p.nitems > 0) {
    gemm_splitk_reduce_kernel<<<p.nitems, 256, 0, st>>>(p.djobs.p, p.ditems.p, t, lv.active, b->dws.p);
    check_launch(b);
  }
}

DeflateParams deflate_params(smpm_batch* b, const int* active) {
  DeflateParams P;
  P.nsys = b->nsys;
  P.d = b->d;
  P.w = b->w;
  P.k = b->k;
  P.active = active;
  P.cmode = b->dcmode.p;
  P.cinv = b->dcinv.p;
  P.uc = b->duc.p;
  P.singular = b->dsingular.p;
  P.thomas = b->dthomas.p;
  P.rowsum = b->drowsum.p;
  P.mx = b->mx;
  P.alist = nullptr;
  P.acount = nullptr;
  return P;
}

void run_deflate(smpm_batch* b, int mode, const double* zin, const double* v, double* y, double* cout,
                 const Live& lv, cudaStream_t st) {
  ProfScope ps(b, PC_DEFL, st);
  if (lv.nslots == 0) return;
  DeflateParams P = deflate_params(b, lv.active);
  P.alist = lv.alist;
  P.acount = lv.acount;
  const size_t shm = sizeof(double) * 2 * static_cast<size_t>(b->d);
  const int d = b->d, ns = lv.nslots;
  double* sums = b->dcoarse.p;
  double* cbuf = b->dcoarse.p + static_cast<size_t>(ns) * d;
  if (mode == DEFL_COARSE_DIRECT) {
    zt_coarse_kernel<<<dim3(1, ns), V2_THREADS, shm, st>>>(P, zin, sums, cout, b->dcount.p, 1);
    check_launch(b);
    return;
  }
  if (mode != DEFL_SUB_T) {
    // Z^T + coarse solve: warp per interface, last CTA of each system solves
    launch_pdl(b, zt_coarse_kernel, dim3((d + DZ_IFACES - 1) / DZ_IFACES, ns), dim3(V2_THREADS), shm, st, P, zin, sums,
               mode == DEFL_COARSE ? cout : cbuf, b->dcount.p, 0);
    if (mode == DEFL_COARSE) return;
  }
  const int gx = static_cast<int>(std::min<long long>((b->k + V2_THREADS * 4 - 1) / (V2_THREADS * 4), 256));
  launch_pdl(b, defl_update_kernel, dim3(gx, ns), dim3(V2_THREADS), 0, st, P, mode, static_cast<const double*>(cbuf),
             zin, v, y);
}

int grid_for(long long elems) {
  return static_cast<int>(std::min<long long>((elems + 255) / 256, 148LL * 8));
}

#include "batch_ops.inl"
#include "batch_setup.inl"
#include "batch_gmres.inl"
#include "batch_spectral.inl"
#include "batch_solve.inl"

}  // namespace

#include "batch_abi.inl"
