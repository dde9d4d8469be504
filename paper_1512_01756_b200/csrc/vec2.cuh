// Bandwidth/latency-oriented vector kernels, v2 (sm_100a).
//
// Arnoldi orthogonalization: one thread per row (R rows per thread), looping
// over the basis columns so each thread keeps many independent coalesced
// loads in flight; per-column sums reduce by warp shuffles, then across the
// CTA's warps in shared memory, then across CTAs by the deterministic
// "last CTA reduces in chunk order" pattern.
//
// Deflation: Z^T segmented sums by many CTAs (warp per interface), the
// coarse solve by the last CTA of each system, and the O(k) update on a 2D
// (chunk, system) grid with 32-bit in-system indexing.
#pragma once

#include "common.cuh"
#include "vec.cuh"

namespace smpm {

constexpr int V2_THREADS = 256;
constexpr int V2_ROWS = 2;  // rows per thread -> chunk = 512 rows
constexpr int V2_CHUNK = V2_THREADS * V2_ROWS;
constexpr int V2_MAXCOL = 128;

// part[c] = sum over this CTA's rows of V[:, c] * x  (c < ncols); x from smem
__device__ __forceinline__ void cta_col_dots(const double* __restrict__ Vs, long long k, int ncols, const double* xs,
                                             int r0, int r1, double* __restrict__ part, double (*red)[V2_MAXCOL + 1]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = V2_THREADS >> 5;
  int rows[V2_ROWS];
  double xv[V2_ROWS];
#pragma unroll
  for (int q = 0; q < V2_ROWS; ++q) {
    rows[q] = r0 + t + q * V2_THREADS;
    xv[q] = rows[q] < r1 ? xs[rows[q] - r0] : 0.0;
  }
  constexpr int GRP = 16;  // columns per group: GRP * V2_ROWS independent loads in flight
  for (int c0 = 0; c0 < ncols; c0 += GRP) {
    double acc[GRP];
#pragma unroll
    for (int u = 0; u < GRP; ++u) {
      acc[u] = 0.0;
      const int c = c0 + u;
      if (c < ncols) {
        const double* col = Vs + static_cast<long long>(c) * k;
#pragma unroll
        for (int q = 0; q < V2_ROWS; ++q)
          if (rows[q] < r1) acc[u] = fma(col[rows[q]], xv[q], acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < GRP; ++u) {
      const double v = warp_sum(acc[u]);
      if (lane == 0 && c0 + u < ncols) red[warp][c0 + u] = v;
    }
  }
  __syncthreads();
  for (int c = t; c < ncols; c += V2_THREADS) {
    double s = 0.0;
    for (int q = 0; q < nw; ++q) s += red[q][c];
    part[c] = s;
  }
}

// ---- CGS2 pass 1: h1 = V^T w ----------------------------------------------
// tdefl != nullptr: the fused deflation P of the dbj operator is applied on
// the fly, w = t - Z c - (S - I) Z c with c = C^{-1} Z^T t precomputed per
// system in cbuf (strip row-sum identity), and w is stored.
__global__ void __launch_bounds__(V2_THREADS) cgs2_dot_kernel(GmState_ G, const double* __restrict__ V,
                                                              double* __restrict__ w, const double* __restrict__ tdefl,
                                                              DeflateParams P, const double* __restrict__ cbuf) {
  __shared__ double xs[V2_CHUNK];
  __shared__ double red[V2_THREADS / 32][V2_MAXCOL + 1];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int ncols = G.jcyc[s] + 1;
  const int ch = blockIdx.x;
  const int r0 = ch * G.chunk, r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  double* ws = w + s * G.k;
  if (tdefl) {
    const int wd = P.w, w2 = 2 * wd, mx = P.mx;
    const double* c = cbuf + static_cast<long long>(s) * P.d;
    const double* rs = P.rowsum + static_cast<long long>(s) * 6 * wd;
    const double *rWI = rs, *rEI = rs + w2, *rEW = rs + 2 * w2, *rWE = rEW + wd;
    const double* ts = tdefl + s * G.k;
    for (int e = r0 + threadIdx.x; e < r1; e += V2_THREADS) {
      const int blk = e / wd, r = e - blk * wd, i = blk >> 1;
      double sz;
      if ((blk & 1) == 0)
        sz = (i + 1 == mx - 1) ? c[i] * rWE[r] : c[i] * rWI[r] + c[i + 1] * rEI[r];
      else
        sz = (i == 0) ? c[i] * rEW[r] : c[i - 1] * rWI[wd + r] + c[i] * rEI[wd + r];
      const double v = ts[e] - (c[i] + sz);
      ws[e] = v;
      xs[e - r0] = v;
    }
  } else {
    for (int r = r0 + threadIdx.x; r < r1; r += V2_THREADS) xs[r - r0] = ws[r];
  }
  __syncthreads();
  const int stride = G.m + 2;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  cta_col_dots(V + s * G.vstride, G.k, ncols, xs, r0, r1, part, red);
  if (last_cta(G.counter + s, G.nchunk))
    reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols,
                 G.h1 + static_cast<long long>(s) * stride);
}

// ---- CGS2 pass 2 (h2 = V^T w after w -= V h1) / pass 3 (||w|| + Givens) ----
template <bool NORM>
__global__ void __launch_bounds__(V2_THREADS) cgs2_update_kernel(GmState_ G, const double* __restrict__ V,
                                                                 double* __restrict__ w, int do_update) {
  __shared__ double xs[V2_CHUNK];
  __shared__ double hs[V2_MAXCOL];
  __shared__ double red[V2_THREADS / 32][V2_MAXCOL + 1];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int j = G.jcyc[s];
  const int ncols = j + 1;
  const int stride = G.m + 2;
  const double* hin = (NORM ? G.h2 : G.h1) + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < ncols; i += V2_THREADS) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = ch * G.chunk, r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  double sq = 0.0;
#pragma unroll
  for (int q = 0; q < V2_ROWS; ++q) {
    const int r = r0 + threadIdx.x + q * V2_THREADS;
    if (r >= r1) continue;
    double acc = ws[r];
    if (do_update) {
      // 16 independent column loads per round: the update is latency-bound
      // when few systems are live, so the number of load rounds is what counts
      double a1 = 0.0, a2 = 0.0;
      for (int i0 = 0; i0 < ncols; i0 += 16) {
        double vv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) vv[u] = i0 + u < ncols ? Vs[static_cast<long long>(i0 + u) * G.k + r] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          a1 = fma(vv[u], i0 + u < ncols ? hs[i0 + u] : 0.0, a1);
          a2 = fma(vv[u + 1], i0 + u + 1 < ncols ? hs[i0 + u + 1] : 0.0, a2);
        }
      }
      acc -= a1 + a2;
      ws[r] = acc;
    }
    xs[r - r0] = acc;
    sq = fma(acc, acc, sq);
  }
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  if (!NORM) {
    __syncthreads();
    cta_col_dots(Vs, G.k, ncols, xs, r0, r1, part, red);
    if (last_cta(G.counter + s, G.nchunk))
      reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols,
                   G.h2 + static_cast<long long>(s) * stride);
    return;
  }
  sq = warp_sum(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tsum = 0.0;
    for (int q = 0; q < V2_THREADS / 32; ++q) tsum += red[q][0];
    part[0] = tsum;
  }
  if (!last_cta(G.counter + s, G.nchunk)) return;
  if (threadIdx.x >= 32) return;
  const double nsq = warp_reduce_strided(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride);
  givens_step(G, s, j, sqrt(nsq));
}

// ---------------------------------------------------------------------------
// Deflation v2
// ---------------------------------------------------------------------------
constexpr int DZ_IFACES = 8;  // interfaces per CTA in the Z^T pass (warp each)

// Z^T sums of zin (nsys x k) -> sums (nsys x d); last CTA per system solves
// the coarse system and writes c (nsys x d). mode DEFL_COARSE_DIRECT takes
// the coarse right-hand side from zin (nsys x d) directly.
__global__ void __launch_bounds__(V2_THREADS) zt_coarse_kernel(DeflateParams P, const double* __restrict__ zin,
                                                               double* __restrict__ sums, double* __restrict__ cout,
                                                               int* counter, int direct) {
  pdl_wait();
  pdl_launch();
  extern __shared__ double sm[];
  int s;
  if (!defl_slot(P, blockIdx.y, s)) return;
  const int d = P.d, w2 = 2 * P.w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ss = sums + static_cast<long long>(s) * d;
  if (!direct) {
    const double* zs = zin + static_cast<long long>(s) * P.k;
    const int i = blockIdx.x * DZ_IFACES + warp;
    if (warp < DZ_IFACES && i < d) {
      const double* seg = zs + static_cast<long long>(i) * w2;
      double a0 = 0.0, a1 = 0.0;
      int e = lane;
      for (; e + 32 < w2; e += 64) {
        a0 += seg[e];
        a1 += seg[e + 32];
      }
      if (e < w2) a0 += seg[e];
      const double v = warp_sum(a0 + a1);
      if (lane == 0) ss[i] = v;
    }
    if (!last_cta(counter + s, gridDim.x)) return;
  }
  double* bsh = sm;
  double* csh = sm + d;
  const double* src = direct ? zin + static_cast<long long>(s) * d : ss;
  for (int i = threadIdx.x; i < d; i += blockDim.x) bsh[i] = src[i];
  __syncthreads();
  coarse_solve_block(P, s, bsh, csh);
  for (int i = threadIdx.x; i < d; i += blockDim.x) cout[static_cast<long long>(s) * d + i] = csh[i];
}

// elementwise deflation updates on a (chunk, system) grid
__global__ void __launch_bounds__(V2_THREADS) defl_update_kernel(DeflateParams P, int mode, const double* __restrict__ c,
                                                                 const double* __restrict__ zin,
                                                                 const double* __restrict__ v, double* __restrict__ y) {
  pdl_wait();
  pdl_launch();
  int s;
  if (!defl_slot(P, blockIdx.y, s)) return;
  const int w = P.w, w2 = 2 * w, mx = P.mx;
  const int k = static_cast<int>(P.k);
  const double* cs = c + static_cast<long long>(s) * P.d;
  const long long base = static_cast<long long>(s) * P.k;
  const double* vs = v + base;
  double* ys = y + base;
  const double* rs = P.rowsum + static_cast<long long>(s) * 6 * w;
  const double* rWI = rs;
  const double* rEI = rs + w2;
  const double* rEW = rs + 2 * w2;
  const double* rWE = rEW + w;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x) {
    const int blk = e / w;
    const int r = e - blk * w;
    const int i = blk >> 1;
    if (mode == DEFL_SUB_T) {
      ys[e] = vs[e] - zin[base + e];
    } else if (mode == DEFL_Q_TAIL) {
      ys[e] = vs[e] - cs[i];
    } else if (mode == DEFL_ADD_ZC) {
      ys[e] = vs[e] + cs[i];
    } else {  // DEFL_P_FUSED: y = v - Z c - (S - I) Z c via strip row sums
      double sz;
      if ((blk & 1) == 0)
        sz = (i + 1 == mx - 1) ? cs[i] * rWE[r] : cs[i] * rWI[r] + cs[i + 1] * rEI[r];
      else
        sz = (i == 0) ? cs[i] * rEW[r] : cs[i - 1] * rWI[w + r] + cs[i] * rEI[w + r];
      ys[e] = vs[e] - (cs[i] + sz);
    }
  }
}

// dbj epilogue in one pass over the batch (spectral fused path):
//   final residual (proj/src/gmres.cpp:129-136): r = rhs - P t with t = S M^{-1} x',
//     P t = t - Z c - (S - I) Z c, c = C^{-1} Z^T t (from the per-mode pass); ||r||^2 -> nrf
//   solution (proj/src/deflation.cpp:118-120): x_S = Q u + Z c_b with u = M^{-1} x',
//     Q u = u - Z C^{-1} Z^T S u = u - Z c (S u = t: the same coarse solution), c_b = C^{-1} Z^T b_S
// Per-system ||r||^2: CTA partials summed by the last CTA in chunk order (deterministic).
__global__ void __launch_bounds__(V2_THREADS)
post_dbj_kernel(DeflateParams P, const double* __restrict__ t, const double* __restrict__ u,
                const double* __restrict__ rhs, const double* __restrict__ ct, const double* __restrict__ cb,
                double* __restrict__ xS, double* __restrict__ part, int* counter, double* __restrict__ nrf, int check) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[V2_THREADS / 32];
  int s;
  if (!defl_slot(P, blockIdx.y, s)) return;
  const int w = P.w, w2 = 2 * w, mx = P.mx;
  const int k = static_cast<int>(P.k);
  const double* c = ct + static_cast<long long>(s) * P.d;
  const double* c2 = cb + static_cast<long long>(s) * P.d;
  const long long base = static_cast<long long>(s) * P.k;
  const double* rs = P.rowsum + static_cast<long long>(s) * 6 * w;
  const double *rWI = rs, *rEI = rs + w2, *rEW = rs + 2 * w2, *rWE = rEW + w;
  double sq = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x) {
    const int blk = e / w, r = e - blk * w, i = blk >> 1;
    xS[base + e] = (u[base + e] - c[i]) + c2[i];
    if (check) {
      double sz;
      if ((blk & 1) == 0)
        sz = (i + 1 == mx - 1) ? c[i] * rWE[r] : c[i] * rWI[r] + c[i + 1] * rEI[r];
      else
        sz = (i == 0) ? c[i] * rEW[r] : c[i - 1] * rWI[w + r] + c[i] * rEI[w + r];
      const double rr = rhs[base + e] - (t[base + e] - (c[i] + sz));
      sq = fma(rr, rr, sq);
    }
  }
  if (!check) return;
  sq = warp_sum(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int q = 0; q < V2_THREADS / 32; ++q) a += red[q];
    part[static_cast<long long>(s) * gridDim.x + blockIdx.x] = a;
  }
  if (!last_cta(counter + s, gridDim.x)) return;
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int q = 0; q < static_cast<int>(gridDim.x); ++q) a += __ldcg(part + static_cast<long long>(s) * gridDim.x + q);
    nrf[s] = a;
  }
}

}  // namespace smpm
