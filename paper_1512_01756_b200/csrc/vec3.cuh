// CGS2 Arnoldi passes with long row chunks (sm_100a).
//
// Same arithmetic as the vec2.cuh passes (classical Gram-Schmidt with one
// reorthogonalisation, fused deflation P in pass 1, Givens update after the
// norm pass), but each CTA owns thousands of rows of one system so a batch
// of live systems is one wave of CTAs: per-system partial sums are few, the
// last-CTA reductions are short, and every thread keeps two rows x eight
// columns of independent loads in flight.  Chunk length is chosen on the
// host so (live systems x chunks) ~ the resident CTA count.
#pragma once

#include "vec.cuh"
#include "vec2.cuh"

namespace smpm {

constexpr int V3_THREADS = 256;
constexpr int V3_GRP = 8;  // columns per register group

constexpr int V3_NR = 2;   // rows per thread per round (stride V3_THREADS)

// partial dots over rows [r0, r1) of V_s[:, 0..ncols) with x -> out[0..ncols).
// Thread t accumulates rows r0 + t, r0 + t + 256, ... in that order, V3_NR rows
// per round with every load of the round independent; columns past ncols are
// not loaded.
__device__ __forceinline__ void cta_dots_long(const double* __restrict__ Vs, long long k, int ncols,
                                              const double* x, int r0, int r1, double* __restrict__ out,
                                              double (*red)[V3_GRP]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int c0 = 0; c0 < ncols; c0 += V3_GRP) {
    const int nc = min(V3_GRP, ncols - c0);
    double acc[V3_GRP];
#pragma unroll
    for (int u = 0; u < V3_GRP; ++u) acc[u] = 0.0;
    for (int r = r0 + t; r < r1; r += V3_NR * V3_THREADS) {
      double xv[V3_NR], v[V3_NR][V3_GRP];
#pragma unroll
      for (int q = 0; q < V3_NR; ++q) {
        const int rq = r + q * V3_THREADS;
        const bool ok = rq < r1;
        xv[q] = ok ? __ldcg(x + rq) : 0.0;
#pragma unroll
        for (int u = 0; u < V3_GRP; ++u)
          v[q][u] = (ok && u < nc) ? __ldcg(Vs + static_cast<long long>(c0 + u) * k + rq) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < V3_NR; ++q)
#pragma unroll
        for (int u = 0; u < V3_GRP; ++u) acc[u] = fma(v[q][u], xv[q], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < V3_GRP; ++u) {
      const double v = warp_sum(acc[u]);
      if (lane == 0) red[warp][u] = v;
    }
    __syncthreads();
    if (t < V3_GRP && c0 + t < ncols) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < V3_THREADS / 32; ++q) s += red[q][t];
      out[c0 + t] = s;
    }
    __syncthreads();
  }
}

// w[r] -= sum_c V[r, c] h[c] over rows [r0, r1); returns sum of squares of the new rows
// (two rows per thread and round; per row, even / odd columns accumulate
// separately in column order; columns past ncols are not loaded)
__device__ __forceinline__ double rows_update_long(const double* __restrict__ Vs, long long k, int ncols,
                                                   const double* h, double* ws, int r0, int r1) {
  double sq = 0.0;
  for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += 2 * V3_THREADS) {
    const int r2 = r + V3_THREADS;
    const bool two = r2 < r1;
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    for (int c0 = 0; c0 < ncols; c0 += V3_GRP) {
      const int nc = min(V3_GRP, ncols - c0);
      double v0[V3_GRP], v1[V3_GRP];
#pragma unroll
      for (int u = 0; u < V3_GRP; ++u) {
        const double* col = Vs + static_cast<long long>(c0 + u) * k;
        v0[u] = u < nc ? __ldcg(col + r) : 0.0;
        v1[u] = (two && u < nc) ? __ldcg(col + r2) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < V3_GRP; u += 2) {
        const double h0 = u < nc ? h[c0 + u] : 0.0, h1 = u + 1 < nc ? h[c0 + u + 1] : 0.0;
        a0 = fma(v0[u], h0, a0);
        a1 = fma(v0[u + 1], h1, a1);
        b0 = fma(v1[u], h0, b0);
        b1 = fma(v1[u + 1], h1, b1);
      }
    }
    const double n0 = __ldcg(ws + r) - (a0 + a1);
    ws[r] = n0;
    sq = fma(n0, n0, sq);
    if (two) {
      const double n1 = __ldcg(ws + r2) - (b0 + b1);
      ws[r2] = n1;
      sq = fma(n1, n1, sq);
    }
  }
  return sq;
}

// ---- pass 1: h1 = V^T w (with the fused deflation P when tdefl != nullptr) ----
__global__ void __launch_bounds__(V3_THREADS) cgs3_dot_kernel(GmState_ G, const double* __restrict__ V, double* w,
                                                              const double* __restrict__ tdefl, DeflateParams P,
                                                              const double* __restrict__ cbuf) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[V3_THREADS / 32][V3_GRP];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int ncols = G.jcyc[s] + 1;
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  double* ws = w + s * G.k;
  if (tdefl) {
    // w = t - Z c - (S - I) Z c (strip row-sum identity)
    const int wd = P.w, w2 = 2 * wd, mx = P.mx;
    const double* c = cbuf + static_cast<long long>(s) * P.d;
    const double* rs = P.rowsum + static_cast<long long>(s) * 6 * wd;
    const double *rWI = rs, *rEI = rs + w2, *rEW = rs + 2 * w2, *rWE = rEW + wd;
    const double* ts = tdefl + s * G.k;
    for (int e = r0 + threadIdx.x; e < r1; e += V3_THREADS) {
      const int blk = e / wd, r = e - blk * wd, i = blk >> 1;
      double sz;
      if ((blk & 1) == 0)
        sz = (i + 1 == mx - 1) ? c[i] * rWE[r] : c[i] * rWI[r] + c[i + 1] * rEI[r];
      else
        sz = (i == 0) ? c[i] * rEW[r] : c[i - 1] * rWI[wd + r] + c[i] * rEI[wd + r];
      ws[e] = ts[e] - (c[i] + sz);
    }
    __syncthreads();
  }
  const int stride = G.m + 2;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  cta_dots_long(V + s * G.vstride, G.k, ncols, ws, r0, r1, part, red);
  if (last_cta(G.counter + s, G.nchunk))
    reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols,
                 G.h1 + static_cast<long long>(s) * stride);
}

// ---- pass 2 (w -= V h1 ; h2 = V^T w) / pass 3 (w -= V h2 ; ||w|| + Givens) ----
template <bool NORM>
__global__ void __launch_bounds__(V3_THREADS) cgs3_update_kernel(GmState_ G, const double* __restrict__ V, double* w) {
  pdl_wait();
  pdl_launch();
  __shared__ double hs[V2_MAXCOL];
  __shared__ double red[V3_THREADS / 32][V3_GRP];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int j = G.jcyc[s];
  const int ncols = j + 1;
  const int stride = G.m + 2;
  const double* hin = (NORM ? G.h2 : G.h1) + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < ncols; i += V3_THREADS) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  double sq = rows_update_long(Vs, G.k, ncols, hs, ws, r0, r1);
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  if (!NORM) {
    __syncthreads();
    cta_dots_long(Vs, G.k, ncols, ws, r0, r1, part, red);
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
    for (int q = 0; q < V3_THREADS / 32; ++q) tsum += red[q][0];
    part[0] = tsum;
  }
  if (!last_cta(G.counter + s, G.nchunk)) return;
  if (threadIdx.x >= 32) return;
  const double nsq = warp_reduce_strided(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride);
  givens_step(G, s, j, sqrt(nsq));
}

}  // namespace smpm
