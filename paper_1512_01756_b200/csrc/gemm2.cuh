// Hot-path fp64 contraction kernel, v2 (sm_100a).
//
// One launch serves a list of GemmJobs (all systems of a batch, one operator
// stage).  Jobs with N >= 2 run as 64x32 output tiles on the fp64 tensor
// pipe (mma.sync.m8n8k4.f64 — tcgen05 has no f64 kind), operands streamed
// with cp.async 16-byte copies through a 3-stage shared-memory ring whose
// padded layouts make every fragment load a minimal-wavefront LDS.64.
// Jobs with N == 1 (the boundary-strip blocks and the first/last
// block-Jacobi blocks) run as warp-coalesced GEMV tiles instead of wasting a
// 32-wide output tile.  Each job's per-element summation order is fixed by
// its plan (tiling, K split), so results are run-to-run deterministic.
#pragma once

#include "common.cuh"

namespace smpm {

#ifndef G2_STAGES_DEF
#define G2_STAGES_DEF 4
#endif
constexpr int G2_BM = 64, G2_BN = 32, G2_BK = 16, G2_STAGES = G2_STAGES_DEF;
constexpr int G2_APAD = 8;  // As row stride 72 doubles: 4 k-rows of 8 m's -> 2 wavefronts
constexpr int G2_BPAD = 4;  // Bs row stride 20 doubles: 8 n-rows of 4 k's -> conflict-free
constexpr int G2_THREADS = 128;
constexpr int G2_SMEM =
    G2_STAGES * (G2_BK * (G2_BM + G2_APAD) + G2_BN * (G2_BK + G2_BPAD)) * static_cast<int>(sizeof(double));
constexpr int GV_ROWS = 16;  // GEMV tile rows (8 k-groups of 16 threads)
constexpr int GV_KG = G2_THREADS / GV_ROWS;
constexpr int G2_RED_PARTS = (G2_BM * G2_BN) / 256;  // reduce CTAs (256 threads) per split tile

struct Tile2 {
  int job;
  int m0, n0;
  int ks;  // K split index (GEMM tiles) ; -1 marks a GEMV tile
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void store_out(const GemmJob& jb, const BufTable& bufs, int m, int n, double acc) {
  double* out = bufs.p[jb.out.buf];
  double v = jb.alpha * acc;
  if (jb.add.buf != BUF_NONE) v = fma(jb.beta, __ldcg(bufs.p[jb.add.buf] + jb.add.at(m, n)), v);
  out[jb.out.at(m, n)] = v;
}

// Per-system templates: jobs/tiles describe system 0; CTA blockIdx.x serves
// tile (blockIdx.x % tiles_per_sys) of the system in active-list slot
// (blockIdx.x / tiles_per_sys), so a launch sized for the live systems only
// schedules their tiles.  Matrix pointers advance by a_stride, vector views
// by v_stride and split-K workspace slots by ws_stride per system.
struct SysMap {
  const int* alist;   // compacted active systems (nullptr: slot == system)
  const int* acount;  // number of valid slots (nullptr: all)
  int tiles_per_sys;
  long long a_stride, v_stride, ws_stride;
};

__device__ __forceinline__ bool map_system(const SysMap& sm, int slot, int& s) {
  if (sm.acount && slot >= *sm.acount) return false;
  s = sm.alist ? sm.alist[slot] : slot;
  return true;
}

__device__ __forceinline__ void shift_job(GemmJob& jb, const SysMap& sm, int s) {
  jb.A += s * sm.a_stride;
  const long long vo = s * sm.v_stride;
  jb.b.off += vo;
  jb.out.off += vo;
  jb.add.off += vo;
  jb.ws_off += static_cast<int>(s * sm.ws_stride);
  jb.sys = s;
}

// GEMV tile (N == 1): 16 rows x K, 8 interleaved k-groups, UNR independent
// loads in flight per thread per round.
template <int UNR = 8>
__device__ __forceinline__ void g2_gemv_tile(const GemmJob& jb, const Tile2& tile, const BufTable& bufs) {
  const int t = threadIdx.x;
  const int r = t % GV_ROWS, kg = t / GV_ROWS;
  const int m = tile.m0 + r;
  const double* x = bufs.p[jb.b.buf] + jb.b.off;
  double acc[UNR];
#pragma unroll
  for (int u = 0; u < UNR; ++u) acc[u] = 0.0;
  if (m < jb.M) {
    const double* __restrict__ a = jb.A + m;
    const long long lda = jb.lda;
    int k = kg;
    for (; k + (UNR - 1) * GV_KG < jb.K; k += UNR * GV_KG) {
      double av[UNR], xv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        av[u] = __ldg(a + static_cast<long long>(k + u * GV_KG) * lda);
        xv[u] = __ldcg(x + k + u * GV_KG);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc[u] = fma(av[u], xv[u], acc[u]);
    }
    // remainder: still independent loads (predicated), same accumulators
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int kk = k + u * GV_KG;
      if (kk < jb.K) acc[u] = fma(__ldg(a + static_cast<long long>(kk) * lda), __ldcg(x + kk), acc[u]);
    }
  }
  __shared__ double red[GV_KG][GV_ROWS];
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < UNR; ++u) v += acc[u];
  red[kg][r] = v;
  __syncthreads();
  if (kg == 0 && m < jb.M) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < GV_KG; ++q) s += red[q][r];
    store_out(jb, bufs, m, 0, s);
  }
}

// K range [kb, ke) of split `ks` of a job
__device__ __forceinline__ void g2_krange(const GemmJob& jb, int ks, int& kb, int& ke) {
  kb = 0;
  ke = jb.K;
  if (jb.splitk > 1) {
    const int kc = ((jb.K + jb.splitk * G2_BK - 1) / (jb.splitk * G2_BK)) * G2_BK;
    kb = ks * kc;
    ke = min(jb.K, kb + kc);
  }
}

// GEMM tile main loop (DMMA m8n8k4) over this split's K range; STAGES-deep
// cp.async ring in `smem`.  acc(i, j, e) holds row wm*32+i*8+lane/4 and
// column wn*16+j*8+(lane%4)*2+e of the 64x32 tile (warp = 2*wm + wn).
template <int STAGES>
__device__ __forceinline__ void g2_mainloop(const GemmJob& jb, const Tile2& tile, const BufTable& bufs, double* smem,
                                            double (&acc)[4][2][2]) {
  auto As = reinterpret_cast<double(*)[G2_BK][G2_BM + G2_APAD]>(smem);
  auto Bs = reinterpret_cast<double(*)[G2_BN][G2_BK + G2_BPAD]>(smem + STAGES * G2_BK * (G2_BM + G2_APAD));
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int M = jb.M, N = jb.N;
  const int m0 = tile.m0, n0 = tile.n0;
  int kb, ke;
  g2_krange(jb, tile.ks, kb, ke);
  const double* __restrict__ A = jb.A;
  const long long lda = jb.lda;
  const double* B = bufs.p[jb.b.buf] + jb.b.off;
  const long long ldb = jb.b.cs;

  auto load_stage = [&](int s, int k0) {
    // A: 16 k-rows x 64 m = 512 chunks of 2 doubles, 4 per thread
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = t + q * G2_THREADS;
      const int kk = c >> 5, m2 = (c & 31) << 1;
      const int k = k0 + kk, m = m0 + m2;
      const bool ok = (k < ke) && (m < M);
      const double* src = ok ? A + static_cast<long long>(k) * lda + m : A;
      cp_async16(&As[s][kk][m2], src, ok);
    }
    // B: 32 n-cols x 16 k = 256 chunks, 2 per thread
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = t + q * G2_THREADS;
      const int n = c >> 3, k2 = (c & 7) << 1;
      const int k = k0 + k2, nn = n0 + n;
      const bool ok = (k < ke) && (nn < N);
      const double* src = ok ? B + static_cast<long long>(nn) * ldb + k : B;
      cp_async16(&Bs[s][n][k2], src, ok);
    }
  };

#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int wm = warp >> 1, wn = warp & 1;
  const int nk = (ke - kb + G2_BK - 1) / G2_BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kb + s * G2_BK);
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int s = it % STAGES;
    // prefetch the stage STAGES-1 ahead into the slot freed last iteration
    const int nx = it + STAGES - 1;
    if (nx < nk) load_stage(nx % STAGES, kb + nx * G2_BK);
    cp_async_commit();
#pragma unroll
    for (int kq = 0; kq < G2_BK / 4; ++kq) {
      const int kr = kq * 4 + (lane & 3);
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[s][kr][wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bs[s][wn * 16 + j * 8 + (lane >> 2)][kr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
}

// workspace slot of split `ks` of a tile (64x32 doubles each)
__device__ __forceinline__ long long g2_ws_slot(const GemmJob& jb, const Tile2& tile, int ks) {
  const int ntn = (jb.N + G2_BN - 1) / G2_BN;
  return static_cast<long long>(jb.ws_off) + (static_cast<long long>(tile.m0 / G2_BM) * ntn + tile.n0 / G2_BN) * jb.splitk +
         ks;
}

__device__ __forceinline__ void g2_store_ws(const GemmJob& jb, const Tile2& tile, double* ws, const double (&acc)[4][2][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wm = warp >> 1, wn = warp & 1;
  double* w = ws + g2_ws_slot(jb, tile, tile.ks) * (G2_BM * G2_BN);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = wm * 32 + i * 8 + (lane >> 2), c = wn * 16 + j * 8 + (lane & 3) * 2 + e;
        w[r * G2_BN + c] = acc[i][j][e];
      }
}

__device__ __forceinline__ void g2_store_tile(const GemmJob& jb, const Tile2& tile, const BufTable& bufs,
                                              const double (&acc)[4][2][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wm = warp >> 1, wn = warp & 1;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = tile.m0 + wm * 32 + i * 8 + (lane >> 2);
        const int n = tile.n0 + wn * 16 + j * 8 + (lane & 3) * 2 + e;
        if (m < jb.M && n < jb.N) store_out(jb, bufs, m, n, acc[i][j][e]);
      }
}

// One output tile of one (system-shifted) job, computed by the calling CTA's
// first G2_THREADS threads with G2_SMEM bytes of shared memory at `smem`.
// Shared by the per-stage launches and the cluster-persistent solver.
__device__ __forceinline__ void g2_run_tile(const GemmJob& jb, const Tile2& tile, const BufTable& bufs,
                                            double* __restrict__ ws, double* smem) {
  __syncthreads();  // shared memory may still be read by this CTA's previous tile
  if (tile.ks < 0) {
    g2_gemv_tile(jb, tile, bufs);
    return;
  }
  double acc[4][2][2];
  g2_mainloop<G2_STAGES>(jb, tile, bufs, smem, acc);
  if (jb.splitk > 1)
    g2_store_ws(jb, tile, ws, acc);
  else
    g2_store_tile(jb, tile, bufs, acc);
}

__global__ void __launch_bounds__(G2_THREADS, 4)
gemm2_kernel(const GemmJob* __restrict__ jobs, const Tile2* __restrict__ tiles, BufTable bufs, SysMap smap,
             double* __restrict__ ws) {
  // dynamic shared memory (G2_SMEM bytes): As[STAGES][BK][BM+APAD], Bs[STAGES][BN][BK+BPAD]
  extern __shared__ __align__(16) double g2_smem[];
  int sysid;
  if (!map_system(smap, blockIdx.x / smap.tiles_per_sys, sysid)) return;
  const Tile2 tile = tiles[blockIdx.x % smap.tiles_per_sys];
  GemmJob jb = jobs[tile.job];
  shift_job(jb, smap, sysid);
  g2_run_tile(jb, tile, bufs, ws, g2_smem);
}

// split-K reduction in fixed K order + epilogue (64x32 tiles)
__global__ void __launch_bounds__(256)
gemm2_splitk_reduce_kernel(const GemmJob* __restrict__ jobs, const SplitItem* __restrict__ items, int items_per_sys,
                           BufTable bufs, SysMap smap, const double* __restrict__ ws) {
  // G2_RED_PARTS CTAs per tile, one output element per thread (a single
  // round of independent loads instead of a latency-bound loop)
  int sysid;
  const int tile_id = blockIdx.x / G2_RED_PARTS;
  if (!map_system(smap, tile_id / items_per_sys, sysid)) return;
  const SplitItem it = items[tile_id % items_per_sys];
  GemmJob jb = jobs[it.job];
  shift_job(jb, smap, sysid);
  const int ntn = (jb.N + G2_BN - 1) / G2_BN;
  const long long slot0 =
      static_cast<long long>(jb.ws_off) + (static_cast<long long>(it.m0 / G2_BM) * ntn + it.n0 / G2_BN) * jb.splitk;
  const int e = (blockIdx.x % G2_RED_PARTS) * blockDim.x + threadIdx.x;
  const int r = e / G2_BN, c = e % G2_BN;
  const int m = it.m0 + r, n = it.n0 + c;
  if (m >= jb.M || n >= jb.N) return;
  double s = 0.0;
  for (int ks = 0; ks < jb.splitk; ++ks) s += ws[(slot0 + ks) * (G2_BM * G2_BN) + e];
  store_out(jb, bufs, m, n, s);
}

}  // namespace smpm
