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
#ifndef CGS3_MINB
#define CGS3_MINB 2  // minimum resident CTAs per SM requested for pass 2'
#endif

// Row-major work of one thread: rows r0 + t, r0 + t + 256, ... in that order.
// NR rows per round and NG columns per register group, all loads of a round
// independent; few columns (early Arnoldi steps) take more rows per round so
// the memory-level parallelism stays ~16-20 loads per thread.  The per-column
// (dots) and per-row (update) accumulation sequences do not depend on NR / NG,
// so every instance gives bit-identical results.

// x[r] read from memory (the default source of dots_rows)
struct XLoad {
  const double* x;
  __device__ __forceinline__ double operator()(int r) const { return __ldcg(x + r); }
  __device__ __forceinline__ bool first() const { return false; }
};

// pass 1's fused deflation: x[r] = t[r] - (Z c)[r] - ((S - I) Z c)[r] (strip
// row-sum identity), stored to w[r] as it is produced
struct XDeflate {
  const double *c, *rWI, *rEI, *rEW, *rWE, *ts;
  double* ws;
  int wd, mx;
  __device__ __forceinline__ bool first() const { return true; }
  __device__ __forceinline__ double operator()(int e) const {
    const int blk = e / wd, r = e - blk * wd, i = blk >> 1;
    double sz;
    if ((blk & 1) == 0)
      sz = (i + 1 == mx - 1) ? c[i] * rWE[r] : c[i] * rWI[r] + c[i + 1] * rEI[r];
    else
      sz = (i == 0) ? c[i] * rEW[r] : c[i - 1] * rWI[wd + r] + c[i] * rEI[wd + r];
    const double v = ts[e] - (c[i] + sz);
    ws[e] = v;
    return v;
  }
};

// acc[u] += sum over this thread's rows of V[r, c0 + u] x[r], u < nc <= NG
// (x[r] = xs(r); a thread visits rows r0 + t + i * 256, the same rows every pass
// owns, so a source that computes and stores x[r] needs no barrier)
template <int NR, int NG, class XS = XLoad>
__device__ __forceinline__ void dots_rows(const double* __restrict__ Vs, long long k, int c0, int nc,
                                          XS xs, int r0, int r1, double (&acc)[V3_GRP]) {
  for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += NR * V3_THREADS) {
    double xv[NR], v[NR][NG];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int rq = r + q * V3_THREADS;
      const bool ok = rq < r1;
      xv[q] = ok ? xs(rq) : 0.0;
#pragma unroll
      for (int u = 0; u < NG; ++u)
        v[q][u] = (ok && u < nc) ? __ldcg(Vs + static_cast<long long>(c0 + u) * k + rq) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int u = 0; u < NG; ++u) acc[u] = fma(v[q][u], xv[q], acc[u]);
  }
}

template <class XS>
__device__ __forceinline__ void dots_rows_any(const double* __restrict__ Vs, long long k, int c0, int nc, XS xs,
                                              int r0, int r1, double (&acc)[V3_GRP]) {
  if (nc <= 1)
    dots_rows<8, 1>(Vs, k, c0, nc, xs, r0, r1, acc);
  else if (nc <= 2)
    dots_rows<8, 2>(Vs, k, c0, nc, xs, r0, r1, acc);
  else if (nc <= 4)
    dots_rows<4, 4>(Vs, k, c0, nc, xs, r0, r1, acc);
  else
    dots_rows<2, V3_GRP>(Vs, k, c0, nc, xs, r0, r1, acc);
}

// partial dots over rows [r0, r1) of V_s[:, 0..ncols) with x -> out[0..ncols);
// the first column group takes x from xs0 (which may compute and store x), the
// rest re-read the stored x
template <class XS = XLoad>
__device__ __forceinline__ void cta_dots_long(const double* __restrict__ Vs, long long k, int ncols,
                                              const double* x, int r0, int r1, double* __restrict__ out,
                                              double (*red)[V3_GRP], XS xs0 = XS{}) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int c0 = 0; c0 < ncols; c0 += V3_GRP) {
    const int nc = min(V3_GRP, ncols - c0);
    double acc[V3_GRP];
#pragma unroll
    for (int u = 0; u < V3_GRP; ++u) acc[u] = 0.0;
    if (c0 == 0 && xs0.first())
      dots_rows_any(Vs, k, c0, nc, xs0, r0, r1, acc);
    else
      dots_rows_any(Vs, k, c0, nc, XLoad{x}, r0, r1, acc);
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

// w[r] -= sum_c V[r, c] h[c] for this thread's rows, NR rows per round; per row
// the even / odd columns (within each group of 8) accumulate separately in column
// order; returns the sum of squares of the new rows (in row order)
// SCALE: also v = w_new * inv into col and vs (pass 3', the same rows this thread
// owns, so the new basis vector comes from registers instead of a re-read of w)
template <int NR, int NG, bool SCALE = false>
__device__ __forceinline__ double rows_update_nr(const double* __restrict__ Vs, long long k, int ncols,
                                                 const double* h, double* ws, int r0, int r1,
                                                 double inv = 0.0, double* col = nullptr, double* vs = nullptr) {
  double sq = 0.0;
  for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += NR * V3_THREADS) {
    double a[NR][2];
#pragma unroll
    for (int q = 0; q < NR; ++q) a[q][0] = a[q][1] = 0.0;
    for (int c0 = 0; c0 < ncols; c0 += NG) {
      const int nc = min(NG, ncols - c0);
      double v[NR][NG];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int rq = r + q * V3_THREADS;
#pragma unroll
        for (int u = 0; u < NG; ++u)
          v[q][u] = (rq < r1 && u < nc) ? __ldcg(Vs + static_cast<long long>(c0 + u) * k + rq) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NG; u += 2) {
        const double h0 = u < nc ? h[c0 + u] : 0.0, h1 = u + 1 < nc ? h[c0 + u + 1] : 0.0;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          a[q][0] = fma(v[q][u], h0, a[q][0]);
          if (u + 1 < NG) a[q][1] = fma(v[q][u + 1], h1, a[q][1]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int rq = r + q * V3_THREADS;
      if (rq < r1) {
        const double nv = __ldcg(ws + rq) - (a[q][0] + a[q][1]);
        if (SCALE) {
          // pass 3': only the new basis vector and the operator input are live
          // (the next pass 1 rewrites w)
          const double v = nv * inv;
          col[rq] = v;
          vs[rq] = v;
        } else {
          ws[rq] = nv;
          sq = fma(nv, nv, sq);
        }
      }
    }
  }
  return sq;
}

__device__ __forceinline__ double rows_update_long(const double* __restrict__ Vs, long long k, int ncols,
                                                   const double* h, double* ws, int r0, int r1) {
  if (ncols <= 2) return rows_update_nr<8, 2>(Vs, k, ncols, h, ws, r0, r1);
  if (ncols <= 4) return rows_update_nr<4, 4>(Vs, k, ncols, h, ws, r0, r1);
  return rows_update_nr<2, V3_GRP>(Vs, k, ncols, h, ws, r0, r1);
}

// Pass 2 for ncols <= 8 in one traversal of V: each round's V values stay in
// registers for both the update w -= V h and the reorthogonalisation dots
// acc[u] += V[r, u] w_new[r]; same accumulation orders as rows_update_nr and
// dots_rows (bit-identical), one read of V instead of two. Returns ||w_new||^2
// of this thread's rows.
template <int NR, int NG>
__device__ __forceinline__ double pass2_fused_rows(const double* __restrict__ Vs, long long k, int ncols,
                                                   const double* h, double* ws, int r0, int r1,
                                                   double (&acc)[2 * V3_GRP]) {
  double sq = 0.0;
  for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += NR * V3_THREADS) {
    double v[NR][NG], wv[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int rq = r + q * V3_THREADS;
      const bool ok = rq < r1;
      wv[q] = ok ? __ldcg(ws + rq) : 0.0;
#pragma unroll
      for (int u = 0; u < NG; ++u) v[q][u] = (ok && u < ncols) ? __ldcg(Vs + static_cast<long long>(u) * k + rq) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int rq = r + q * V3_THREADS;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int u = 0; u < NG; u += 2) {  // groups of 8 in order: the same sequence as rows_update_nr<2, 8>
        const double h0 = u < ncols ? h[u] : 0.0, h1 = u + 1 < ncols ? h[u + 1] : 0.0;
        a0 = fma(v[q][u], h0, a0);
        a1 = fma(v[q][u + 1], h1, a1);
      }
      const double nv = rq < r1 ? wv[q] - (a0 + a1) : 0.0;
      if (rq < r1) {
        ws[rq] = nv;
        sq = fma(nv, nv, sq);
      }
#pragma unroll
      for (int u = 0; u < NG; ++u) acc[u] = fma(v[q][u], nv, acc[u]);
    }
  }
  return sq;
}

// ---- pass 1: h1 = V^T w (with the fused deflation P when tdefl != nullptr) ----
__global__ void __launch_bounds__(V3_THREADS, 3) cgs3_dot_kernel(GmState_ G, const double* __restrict__ V, double* w,
                                                              const double* __restrict__ tdefl, DeflateParams P,
                                                              const double* __restrict__ cbuf) {
  pdl_wait();
  __shared__ double red[V3_THREADS / 32][V3_GRP];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int ncols = G.jcyc[s] + 1;
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  double* ws = w + s * G.k;
  const int stride = G.m + 2;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  if (tdefl) {
    // w = t - Z c - (S - I) Z c computed row by row inside the first column
    // group's dots (the thread's own rows: no barrier, no re-read of w)
    const int wd = P.w, w2 = 2 * wd;
    const double* rs = P.rowsum + static_cast<long long>(s) * 6 * wd;
    XDeflate xd{cbuf + static_cast<long long>(s) * P.d, rs, rs + w2, rs + 2 * w2, rs + 2 * w2 + wd,
                tdefl + s * G.k, ws, wd, P.mx};
    cta_dots_long(V + s * G.vstride, G.k, ncols, ws, r0, r1, part, red, xd);
  } else {
    cta_dots_long(V + s * G.vstride, G.k, ncols, ws, r0, r1, part, red);
  }
  pdl_launch();  // the row work is done: dependents may start launching
  if (last_cta(G.counter + s, G.nchunk))
    reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols,
                 G.h1 + static_cast<long long>(s) * stride);
}

// ---- pass 2 (w -= V h1 ; h2 = V^T w) / pass 3 (w -= V h2 ; ||w|| + Givens) ----
template <bool NORM>
__global__ void __launch_bounds__(V3_THREADS) cgs3_update_kernel(GmState_ G, const double* __restrict__ V, double* w) {
  pdl_wait();
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
    pdl_launch();  // the row work is done: dependents may start launching
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
  if (G.stacked) {
    if (threadIdx.x == 0) G.snsq[s] = nsq;  // stack_givens_kernel sums over the systems
    return;
  }
  givens_step(G, s, j, sqrt(nsq));
}

// ---- default CGS2 passes 2/3 (SMPM_NO_PYTHAG=1 restores cgs3_update<true> + scale) ----
// pass 2': w -= V h1; h2 = V^T w and ||w||^2 in one reduction; the last CTA takes
// ||w - V h2||^2 = ||w||^2 - ||h2||^2 (h2 is the O(eps) reorthogonalisation
// correction, so the difference is accurate) and runs the Givens step
__global__ void __launch_bounds__(V3_THREADS, CGS3_MINB) cgs3_pass2n_kernel(GmState_ G, const double* __restrict__ V, double* w,
                                                                 int fuse) {
  pdl_wait();
  __shared__ double hs[V2_MAXCOL];
  __shared__ double red[V3_THREADS / 32][V3_GRP];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int j = G.jcyc[s];
  const int ncols = j + 1;
  const int stride = G.m + 2;
  const double* hin = G.h1 + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < ncols; i += V3_THREADS) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  double sq;
  if (fuse && ncols <= 2 * V3_GRP) {
    double acc[2 * V3_GRP];
#pragma unroll
    for (int u = 0; u < 2 * V3_GRP; ++u) acc[u] = 0.0;
    if (ncols <= 2)
      sq = pass2_fused_rows<8, 2>(Vs, G.k, ncols, hs, ws, r0, r1, acc);
    else if (ncols <= 4)
      sq = pass2_fused_rows<4, 4>(Vs, G.k, ncols, hs, ws, r0, r1, acc);
    else if (ncols <= V3_GRP)
      sq = pass2_fused_rows<2, V3_GRP>(Vs, G.k, ncols, hs, ws, r0, r1, acc);
    else
      sq = pass2_fused_rows<1, 2 * V3_GRP>(Vs, G.k, ncols, hs, ws, r0, r1, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      if (g * V3_GRP >= ncols) break;
#pragma unroll
      for (int u = 0; u < V3_GRP; ++u) {
        const double v = warp_sum(acc[g * V3_GRP + u]);
        if (lane == 0) red[warp][u] = v;
      }
      __syncthreads();
      if (threadIdx.x < V3_GRP && g * V3_GRP + static_cast<int>(threadIdx.x) < ncols) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < V3_THREADS / 32; ++q) a += red[q][threadIdx.x];
        part[g * V3_GRP + threadIdx.x] = a;
      }
      __syncthreads();
    }
  } else {
    sq = rows_update_long(Vs, G.k, ncols, hs, ws, r0, r1);
    __syncthreads();
    cta_dots_long(Vs, G.k, ncols, ws, r0, r1, part, red);
  }
  sq = warp_sum(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tsum = 0.0;
    for (int q = 0; q < V3_THREADS / 32; ++q) tsum += red[q][0];
    part[ncols] = tsum;
  }
  pdl_launch();  // the row work is done: dependents may start launching
  if (!last_cta(G.counter + s, G.nchunk)) return;
  double* h2 = G.h2 + static_cast<long long>(s) * stride;
  reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols + 1, h2);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  double hh = 0.0;
  for (int i = threadIdx.x; i < ncols; i += 32) hh = fma(h2[i], h2[i], hh);
  hh = warp_sum(hh);
  const double nsq = h2[ncols];
  __syncwarp();
  if (threadIdx.x == 0) h2[ncols] = 0.0;
  __syncwarp();
  givens_step(G, s, j, sqrt(fmax(nsq - hh, 0.0)));
}

// ---- pass 2' beyond 16 columns: one read of V through shared-memory row tiles ----
// The CTA walks its rows in tiles of TR rows (double-buffered cp.async, 16-byte
// copies: a tile is ncols contiguous column segments of TR doubles).  From the
// staged tile it first forms w1 = w - V h1 for the tile's rows (thread t: row
// t % 64 (+64, ...) over column quarter t / 64, quarters combined in fixed
// order), then accumulates h2 += V^T w1 (warp q owns columns q, q + 8, ...,
// lane l rows l, l + 32, ... of the tile).  Same reduction tree for every
// launch and batch: deterministic.  Returns this thread's ||w1||^2 part.
constexpr int P2T_MAXC = 16;  // columns per warp in the dots phase (ncols <= 8 * 16)
// Tile rows and ring depth: a tile is ~25 KB, and NS - 1 tiles per CTA are in
// flight while one is consumed (2 CTAs/SM: ~150 KB in flight per SM; the measured
// loaded HBM latency of ~2 us needs ~100 KB per SM for full bandwidth — the
// two-deep ring of round 1 had 40 KB in flight and ran at 0.45 of HBM).
// (ring <= ~100 KB so that two CTAs fit an SM)
__host__ __device__ __forceinline__ int p2t_rows(int ncols) { return ncols <= 23 ? 128 : ncols <= 46 ? 64 : 32; }
__host__ __device__ __forceinline__ int p2t_stages(int ncols) { return ncols <= 93 ? 4 : 3; }
__host__ __device__ __forceinline__ size_t p2t_smem_doubles(int cap) {
  const int tr = p2t_rows(cap), ns = p2t_stages(cap);
  return static_cast<size_t>(ns) * tr * cap + static_cast<size_t>(ns) * tr + 4 * tr + tr;
}

template <int NS>
__device__ __forceinline__ double pass2_tiled(const double* __restrict__ Vs, long long k, int ncols,
                                              const double* hs, double* ws, int r0, int r1, double* sm,
                                              double (&acc)[P2T_MAXC]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int TR = p2t_rows(ncols);
  double* tile = sm;                                               // [NS][ncols][TR]
  double* wt = tile + static_cast<size_t>(NS) * TR * ncols;        // [NS][TR]
  double* qp = wt + NS * TR;                                       // [4][TR]
  double* nvs = qp + 4 * TR;                                       // [TR]
  const int ntile = (r1 - r0 + TR - 1) / TR;
  const int pieces = TR / 2;  // 16-byte pieces per column segment
  auto issue = [&](int it) {
    const int a = r0 + it * TR;
    double* tb = tile + static_cast<size_t>(it % NS) * TR * ncols;
    for (int p = t; p < ncols * pieces; p += V3_THREADS) {
      const int c = p / pieces, q = p - c * pieces;
      const int r = a + 2 * q;
      cp_async16(tb + c * TR + 2 * q, Vs + static_cast<long long>(c) * k + (r < r1 ? r : r0), r < r1);
    }
    for (int q = t; q < pieces; q += V3_THREADS) {
      const int r = a + 2 * q;
      cp_async16(wt + (it % NS) * TR + 2 * q, ws + (r < r1 ? r : r0), r < r1);
    }
  };
  double sq = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < NS - 1; ++s0) {
    if (s0 < ntile) issue(s0);
    cp_async_commit();
  }
  const int quarter = t >> 6, qrow = t & 63;
  const int qc = (ncols + 3) >> 2;  // columns per quarter (contiguous ranges)
  const int c0q = quarter * qc, c1q = min(ncols, c0q + qc);
  for (int it = 0; it < ntile; ++it) {
    if (it + NS - 1 < ntile) issue(it + NS - 1);  // into the slot consumed in iteration it - 1
    cp_async_commit();
    cp_async_wait<NS - 1>();
    __syncthreads();
    const double* tb = tile + static_cast<size_t>(it % NS) * TR * ncols;
    const double* wb = wt + (it % NS) * TR;
    // update partials: quarter sums of V[r][c] h[c], c ascending
    for (int r = qrow; r < TR; r += 64) {
      double a0 = 0.0, a1 = 0.0;
      int c = c0q;
      for (; c + 1 < c1q; c += 2) {
        a0 = fma(tb[c * TR + r], hs[c], a0);
        a1 = fma(tb[(c + 1) * TR + r], hs[c + 1], a1);
      }
      if (c < c1q) a0 = fma(tb[c * TR + r], hs[c], a0);
      qp[quarter * TR + r] = a0 + a1;
    }
    __syncthreads();
    const int a = r0 + it * TR;
    for (int r = t; r < TR; r += V3_THREADS) {
      const double nv = (a + r < r1) ? wb[r] - ((qp[r] + qp[TR + r]) + (qp[2 * TR + r] + qp[3 * TR + r])) : 0.0;
      nvs[r] = nv;
      if (a + r < r1) {
        ws[a + r] = nv;
        sq = fma(nv, nv, sq);
      }
    }
    __syncthreads();
    // reorthogonalisation dots from the same tile
#pragma unroll
    for (int i = 0; i < P2T_MAXC; ++i) {
      const int c = warp + 8 * i;
      if (c < ncols) {
        const double* col = tb + c * TR;
        for (int r = lane; r < TR; r += 32) acc[i] = fma(col[r], nvs[r], acc[i]);
      }
    }
    __syncthreads();  // the tile slot, qp and nvs are reused next
  }
  cp_async_wait<0>();
  return sq;
}

// pass 2' for ncols > 16 (tiled single read); ncols > cap (not expected: the host
// sizes cap from the step index) falls back to the two-read form
__global__ void __launch_bounds__(V3_THREADS, 2) cgs3_pass2t_kernel(GmState_ G, const double* __restrict__ V, double* w,
                                                                 int cap) {
  pdl_wait();
  extern __shared__ __align__(16) double p2t_sm[];
  __shared__ double hs[V2_MAXCOL];
  __shared__ double red[V3_THREADS / 32][V3_GRP];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int j = G.jcyc[s];
  const int ncols = j + 1;
  const int stride = G.m + 2;
  const double* hin = G.h1 + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < ncols; i += V3_THREADS) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  double sq;
  if (ncols <= cap && ncols <= 8 * P2T_MAXC) {
    double acc[P2T_MAXC];
#pragma unroll
    for (int i = 0; i < P2T_MAXC; ++i) acc[i] = 0.0;
    sq = p2t_stages(ncols) == 4 ? pass2_tiled<4>(Vs, G.k, ncols, hs, ws, r0, r1, p2t_sm, acc)
                                : pass2_tiled<3>(Vs, G.k, ncols, hs, ws, r0, r1, p2t_sm, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < P2T_MAXC; ++i) {
      const int c = warp + 8 * i;
      const double v = warp_sum(acc[i]);
      if (lane == 0 && c < ncols) part[c] = v;
    }
  } else {
    sq = rows_update_long(Vs, G.k, ncols, hs, ws, r0, r1);
    __syncthreads();
    cta_dots_long(Vs, G.k, ncols, ws, r0, r1, part, red);
  }
  sq = warp_sum(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tsum = 0.0;
    for (int q = 0; q < V3_THREADS / 32; ++q) tsum += red[q][0];
    part[ncols] = tsum;
  }
  pdl_launch();  // the row work is done: dependents may start launching
  if (!last_cta(G.counter + s, G.nchunk)) return;
  double* h2 = G.h2 + static_cast<long long>(s) * stride;
  reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols + 1, h2);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  double hh = 0.0;
  for (int i = threadIdx.x; i < ncols; i += 32) hh = fma(h2[i], h2[i], hh);
  hh = warp_sum(hh);
  const double nsq = h2[ncols];
  __syncwarp();
  if (threadIdx.x == 0) h2[ncols] = 0.0;
  __syncwarp();
  givens_step(G, s, j, sqrt(fmax(nsq - hh, 0.0)));
}

// pass 3': w -= V h2 and v_{j+1} = w / ||w|| into the basis and the operator input
// (the scale kernel folded in; runs after the Givens step, so stopped systems skip it)
__global__ void __launch_bounds__(V3_THREADS) cgs3_pass3s_kernel(GmState_ G, double* __restrict__ V, double* w,
                                                                 double* __restrict__ vin) {
  pdl_wait();
  __shared__ double hs[V2_MAXCOL];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int jn = G.jcyc[s];  // already advanced by the Givens step: the new column
  const int ncols = jn;
  const int stride = G.m + 2;
  const double* hin = G.h2 + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < ncols; i += V3_THREADS) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  const double inv = 1.0 / G.nrm[s];
  double* col = Vs + static_cast<long long>(jn) * G.k;
  double* vs = vin + s * G.k;
  if (ncols <= 2)
    rows_update_nr<8, 2, true>(Vs, G.k, ncols, hs, ws, r0, r1, inv, col, vs);
  else if (ncols <= 4)
    rows_update_nr<4, 4, true>(Vs, G.k, ncols, hs, ws, r0, r1, inv, col, vs);
  else
    rows_update_nr<2, V3_GRP, true>(Vs, G.k, ncols, hs, ws, r0, r1, inv, col, vs);
  pdl_launch();
}

}  // namespace smpm
