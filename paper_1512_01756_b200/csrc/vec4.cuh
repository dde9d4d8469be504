// CGS2 with the reorthogonalisation update deferred into the next step's first
// pass: two reads of the Krylov basis per Arnoldi step instead of three (sm_100a).
//
// vec3.cuh runs, per step j (basis V_{j+1} = [v_0 .. v_j]):
//   pass 1 : h1 = V^T t,  t = P S M^{-1} v_j                      (read V)
//   pass 2': w' = t - V h1, h2 = V^T w', ||w'||^2, Givens          (read V)
//   pass 3': v_{j+1} = (w' - V h2) / nrm                           (read V)
// Pass 3' only applies the O(eps) correction h2.  The operator is linear, so it
// can run on the pending vector u = w' itself, and v_{j+1} can be formed while
// the next step's first pass streams the same columns anyway:
//   operator: a = S M^{-1} u   (u unnormalised, uncorrected)
//   pass 1B : v_{j+1} = (u - V h2) / nrm  -> V[:, j+1]             (read V once)
//             x = (P a) / nrm             -> w
//             h1 = [V, v_{j+1}]^T x
//   pass 2' : unchanged
// With A V_{j+1} = V_{j+2} Hbar (Arnoldi relation) the exact operator image of
// v_{j+1} is x - V_{j+2} q, q = Hbar h2 / nrm; the update w' = x - V h1 is the
// same either way (the q terms cancel) and the recorded Hessenberg column
// differs by q = O(eps ||H||) — the size of the rounding error of the dots
// themselves — which is dropped.  v_{j+1} itself is computed with the same
// arithmetic (and summation order) as pass 3'.
//
// Two kernels, as for pass 2': up to 16 old columns in registers
// (cgs4_pass1b_kernel), more through shared-memory row tiles
// (cgs4_pass1bt_kernel).  Deterministic: fixed reduction trees.
#pragma once

#include <type_traits>

#include "vec3.cuh"

namespace smpm {

// operator output -> x (unscaled): plain, or with the fused deflation
// x[e] = t[e] - (Z c)[e] - ((S - I) Z c)[e] (strip row-sum identity, as XDeflate)
struct XVal {
  __device__ __forceinline__ double from(int, double tv) const { return tv; }
};
struct XDeflVal {
  const double *c, *rWI, *rEI, *rEW, *rWE;
  int wd, mx;
  __device__ __forceinline__ double from(int e, double tv) const {
    const int blk = e / wd, r = e - blk * wd, i = blk >> 1;
    double sz;
    if ((blk & 1) == 0)
      sz = (i + 1 == mx - 1) ? c[i] * rWE[r] : c[i] * rWI[r] + c[i + 1] * rEI[r];
    else
      sz = (i == 0) ? c[i] * rEW[r] : c[i - 1] * rWI[wd + r] + c[i] * rEI[wd + r];
    return tv - (c[i] + sz);
  }
};

// one traversal of the old columns for this thread's rows: v_new and x stored,
// acc[u] += V[r, u] x[r], returns sum v_new[r] x[r]
template <int NR, int NG, class XS>
__device__ __forceinline__ double pass1b_rows(const double* __restrict__ Vs, long long k, int nold, const double* h2s,
                                              double* ws, const double* __restrict__ ts, XS xs, double inv,
                                              double* col, int r0, int r1, double (&acc)[2 * V3_GRP]) {
  double accn = 0.0;
  for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += NR * V3_THREADS) {
    double v[NR][NG], uv[NR], tv[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int rq = r + q * V3_THREADS;
      const bool ok = rq < r1;
      uv[q] = ok ? __ldcg(ws + rq) : 0.0;
      tv[q] = ok ? __ldcg(ts + rq) : 0.0;
#pragma unroll
      for (int u = 0; u < NG; ++u) v[q][u] = (ok && u < nold) ? __ldcg(Vs + static_cast<long long>(u) * k + rq) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int rq = r + q * V3_THREADS;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int u = 0; u < NG; u += 2) {  // the accumulation sequence of rows_update_nr (pass 3')
        const double h0 = u < nold ? h2s[u] : 0.0, h1 = u + 1 < nold ? h2s[u + 1] : 0.0;
        a0 = fma(v[q][u], h0, a0);
        a1 = fma(v[q][u + 1], h1, a1);
      }
      if (rq < r1) {
        const double vj = (uv[q] - (a0 + a1)) * inv;
        const double x = xs.from(rq, tv[q]) * inv;
        col[rq] = vj;
        ws[rq] = x;
        accn = fma(vj, x, accn);
#pragma unroll
        for (int u = 0; u < NG; ++u) acc[u] = fma(v[q][u], x, acc[u]);
      }
    }
  }
  return accn;
}

template <class XS>
__device__ __forceinline__ void pass1b_body(const GmState_& G, double* __restrict__ V, double* w,
                                            const double* __restrict__ t, XS xs, int s, double* hs,
                                            double (*red)[V3_GRP]) {
  const int nold = G.jcyc[s];  // columns 0 .. nold-1 exist; column nold is formed here
  const int stride = G.m + 2;
  const double* hin = G.h2 + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < nold; i += V3_THREADS) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  const double* ts = t + s * G.k;
  double* col = Vs + static_cast<long long>(nold) * G.k;
  const double inv = 1.0 / G.nrm[s];
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  double acc[2 * V3_GRP];
#pragma unroll
  for (int u = 0; u < 2 * V3_GRP; ++u) acc[u] = 0.0;
  double accn;
  if (nold <= 2)
    accn = pass1b_rows<8, 2>(Vs, G.k, nold, hs, ws, ts, xs, inv, col, r0, r1, acc);
  else if (nold <= 4)
    accn = pass1b_rows<4, 4>(Vs, G.k, nold, hs, ws, ts, xs, inv, col, r0, r1, acc);
  else if (nold <= V3_GRP)
    accn = pass1b_rows<2, V3_GRP>(Vs, G.k, nold, hs, ws, ts, xs, inv, col, r0, r1, acc);
  else
    accn = pass1b_rows<1, 2 * V3_GRP>(Vs, G.k, nold, hs, ws, ts, xs, inv, col, r0, r1, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    if (g * V3_GRP >= nold) break;
#pragma unroll
    for (int u = 0; u < V3_GRP; ++u) {
      const double v = warp_sum(acc[g * V3_GRP + u]);
      if (lane == 0) red[warp][u] = v;
    }
    __syncthreads();
    if (threadIdx.x < V3_GRP && g * V3_GRP + static_cast<int>(threadIdx.x) < nold) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < V3_THREADS / 32; ++q) a += red[q][threadIdx.x];
      part[g * V3_GRP + threadIdx.x] = a;
    }
    __syncthreads();
  }
  accn = warp_sum(accn);
  if (lane == 0) red[warp][0] = accn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tsum = 0.0;
    for (int q = 0; q < V3_THREADS / 32; ++q) tsum += red[q][0];
    part[nold] = tsum;
  }
  if (last_cta(G.counter + s, G.nchunk))
    reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, nold + 1,
                 G.h1 + static_cast<long long>(s) * stride);
}

// ---- pass 1B, up to 16 old columns (registers) ----
__global__ void __launch_bounds__(V3_THREADS, CGS3_MINB) cgs4_pass1b_kernel(GmState_ G, double* __restrict__ V, double* w,
                                                                            const double* __restrict__ t, int defl,
                                                                            DeflateParams P,
                                                                            const double* __restrict__ cbuf) {
  pdl_wait();
  __shared__ double hs[2 * V3_GRP];
  __shared__ double red[V3_THREADS / 32][V3_GRP];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  if (defl) {
    const int wd = P.w, w2 = 2 * wd;
    const double* rs = P.rowsum + static_cast<long long>(s) * 6 * wd;
    const XDeflVal xd{cbuf + static_cast<long long>(s) * P.d, rs, rs + w2, rs + 2 * w2, rs + 2 * w2 + wd, wd, P.mx};
    pass1b_body(G, V, w, t, xd, s, hs, red);
  } else {
    pass1b_body(G, V, w, t, XVal{}, s, hs, red);
  }
  pdl_launch();
}

// ---- pass 1B beyond 16 old columns: shared-memory row tiles (as pass2_tiled) ----
__host__ __device__ __forceinline__ size_t p1bt_smem_doubles(int cap) {
  return p2t_smem_doubles(cap) + static_cast<size_t>(p2t_stages(cap)) * p2t_rows(cap);
}

template <int NS, class XS>
__device__ __forceinline__ double pass1b_tiled(const double* __restrict__ Vs, long long k, int nold, const double* hs,
                                               double* ws, const double* __restrict__ ts, XS xs, double inv,
                                               double* col, int r0, int r1, double* sm, double (&acc)[P2T_MAXC]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int TR = p2t_rows(nold);
  double* tile = sm;                                         // [NS][nold][TR]
  double* wt = tile + static_cast<size_t>(NS) * TR * nold;   // [NS][TR]  pending vector u
  double* at = wt + NS * TR;                                 // [NS][TR]  operator output
  double* qp = at + NS * TR;                                 // [4][TR]
  double* nvs = qp + 4 * TR;                                 // [TR]      x of the tile
  const int ntile = (r1 - r0 + TR - 1) / TR;
  const int pieces = TR / 2;
  auto issue = [&](int it) {
    const int a = r0 + it * TR;
    double* tb = tile + static_cast<size_t>(it % NS) * TR * nold;
    for (int p = t; p < nold * pieces; p += V3_THREADS) {
      const int c = p / pieces, q = p - c * pieces;
      const int r = a + 2 * q;
      cp_async16(tb + c * TR + 2 * q, Vs + static_cast<long long>(c) * k + (r < r1 ? r : r0), r < r1);
    }
    for (int q = t; q < 2 * pieces; q += V3_THREADS) {
      const int which = q >= pieces ? 1 : 0, qq = q - which * pieces;
      const int r = a + 2 * qq;
      const double* src = which ? ts : ws;
      double* dst = (which ? at : wt) + (it % NS) * TR + 2 * qq;
      cp_async16(dst, src + (r < r1 ? r : r0), r < r1);
    }
  };
  double accn = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < NS - 1; ++s0) {
    if (s0 < ntile) issue(s0);
    cp_async_commit();
  }
  const int quarter = t >> 6, qrow = t & 63;
  const int qc = (nold + 3) >> 2;
  const int c0q = quarter * qc, c1q = min(nold, c0q + qc);
  for (int it = 0; it < ntile; ++it) {
    if (it + NS - 1 < ntile) issue(it + NS - 1);  // into the slot consumed in iteration it - 1
    cp_async_commit();
    cp_async_wait<NS - 1>();
    __syncthreads();
    const double* tb = tile + static_cast<size_t>(it % NS) * TR * nold;
    const double* wb = wt + (it % NS) * TR;
    const double* ab = at + (it % NS) * TR;
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
      double x = 0.0;
      if (a + r < r1) {
        const double vj = (wb[r] - ((qp[r] + qp[TR + r]) + (qp[2 * TR + r] + qp[3 * TR + r]))) * inv;
        x = xs.from(a + r, ab[r]) * inv;
        col[a + r] = vj;
        ws[a + r] = x;
        accn = fma(vj, x, accn);
      }
      nvs[r] = x;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < P2T_MAXC; ++i) {
      const int c = warp + 8 * i;
      if (c < nold) {
        const double* cc = tb + c * TR;
        for (int r = lane; r < TR; r += 32) acc[i] = fma(cc[r], nvs[r], acc[i]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  return accn;
}

template <class XS>
__device__ __forceinline__ void pass1bt_body(const GmState_& G, double* __restrict__ V, double* w,
                                             const double* __restrict__ t, XS xs, int s, double* hs, double* red,
                                             double* sm) {
  const int nold = G.jcyc[s];
  const int stride = G.m + 2;
  const double* hin = G.h2 + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < nold; i += V3_THREADS) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  const double* ts = t + s * G.k;
  double* col = Vs + static_cast<long long>(nold) * G.k;
  const double inv = 1.0 / G.nrm[s];
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  double acc[P2T_MAXC];
#pragma unroll
  for (int i = 0; i < P2T_MAXC; ++i) acc[i] = 0.0;
  double accn = p2t_stages(nold) == 4 ? pass1b_tiled<4>(Vs, G.k, nold, hs, ws, ts, xs, inv, col, r0, r1, sm, acc)
                                      : pass1b_tiled<3>(Vs, G.k, nold, hs, ws, ts, xs, inv, col, r0, r1, sm, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < P2T_MAXC; ++i) {
    const int c = warp + 8 * i;
    const double v = warp_sum(acc[i]);
    if (lane == 0 && c < nold) part[c] = v;
  }
  accn = warp_sum(accn);
  if (lane == 0) red[warp] = accn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tsum = 0.0;
    for (int q = 0; q < V3_THREADS / 32; ++q) tsum += red[q];
    part[nold] = tsum;
  }
  if (last_cta(G.counter + s, G.nchunk))
    reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, nold + 1,
                 G.h1 + static_cast<long long>(s) * stride);
}

__global__ void __launch_bounds__(V3_THREADS, 2) cgs4_pass1bt_kernel(GmState_ G, double* __restrict__ V, double* w,
                                                                     const double* __restrict__ t, int defl,
                                                                     DeflateParams P, const double* __restrict__ cbuf) {
  pdl_wait();
  extern __shared__ __align__(16) double p1bt_sm[];
  __shared__ double hs[V2_MAXCOL];
  __shared__ double red[V3_THREADS / 32];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  if (defl) {
    const int wd = P.w, w2 = 2 * wd;
    const double* rs = P.rowsum + static_cast<long long>(s) * 6 * wd;
    const XDeflVal xd{cbuf + static_cast<long long>(s) * P.d, rs, rs + w2, rs + 2 * w2, rs + 2 * w2 + wd, wd, P.mx};
    pass1bt_body(G, V, w, t, xd, s, hs, red, p1bt_sm);
  } else {
    pass1bt_body(G, V, w, t, XVal{}, s, hs, red, p1bt_sm);
  }
  pdl_launch();
}

// ---------------------------------------------------------------------------
// More than 16 columns without shared-memory tiles: G lanes share a row pair.
//
// Lane (rho, g) of a warp (g = lane % G, rho = lane / G) owns two consecutive
// rows (one 16-byte load per column) and the columns g, g + G, g + 2 G, ...
// (CPT of them).  A row's update sum is the butterfly sum of its G lanes'
// partial sums (the same value in all G lanes: fp addition is commutative and
// the tree is symmetric); the updated entries are then multiplied into each
// lane's column accumulators, which stay in registers for the whole row chunk.
// No barrier and no shared-memory staging inside the row loop; every load is
// independent (CPT x NR 16-byte loads per thread in flight), and one warp load
// covers G columns x (32 / G) row pairs: 128 contiguous bytes per column for
// G = 4 (up to 64 columns), 64 for G = 8 (up to 128 columns).  Measured on the
// way here (profiles/r02): 8-byte loads with 32 contiguous bytes per column
// stall on the L1 (2.6-3.3 TB/s); the two-deep shared-memory tiles were
// instruction- and barrier-bound (85 warp instructions per KB, 2.9 TB/s).
// Used by pass 2' (update + reorthogonalisation dots) and pass 1B beyond 16
// columns; fixed summation orders: deterministic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 ldcg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }

template <int G, int CPT, int NR, bool P1B, class XS>
__device__ __forceinline__ double lanes_rows(const double* __restrict__ Vs, long long k, int ncols, const double* hsm,
                                             double* ws, const double* __restrict__ ts, XS xs, double inv, double* col,
                                             int r0, int r1, double (&acc)[CPT]) {
  constexpr int LR = 32 / G;  // lane rows (row pairs) per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane % G, rho = lane / G;
  const double* vbase = Vs + static_cast<long long>(g) * k;
  const long long kG = static_cast<long long>(G) * k;
  double sq = 0.0;  // pass 2': ||w_new||^2 part; pass 1B: v_new . x part (lane g == 0 only)
  constexpr int RPI = (V3_THREADS / 32) * 2 * LR * NR;  // rows per CTA iteration
  for (int rb = r0; rb < r1; rb += RPI) {
    double2 v[NR][CPT], wv[NR], tv[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = rb + ((warp * NR + q) * LR + rho) * 2;  // even: r0 and the chunk are multiples of 256
      const bool ok = r < r1;                              // r1 is even (k = 2 w d), so r + 1 < r1 as well
      wv[q] = ok ? ldcg2(ws + r) : make_double2(0.0, 0.0);
      if (P1B) tv[q] = (ok && g == 0) ? ldcg2(ts + r) : make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < CPT; ++i)
        v[q][i] = (ok && g + G * i < ncols) ? ldcg2(vbase + i * kG + r) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = rb + ((warp * NR + q) * LR + rho) * 2;
      const bool ok = r < r1;
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const double h = hsm[g + G * i];
        p0 = fma(v[q][i].x, h, p0);
        p1 = fma(v[q][i].y, h, p1);
      }
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        p1 += __shfl_xor_sync(0xffffffffu, p1, o);
      }
      double y0, y1;  // the vector the dots are taken with
      if (P1B) {
        double x0 = 0.0, x1 = 0.0;
        if (ok && g == 0) {
          const double vj0 = (wv[q].x - p0) * inv, vj1 = (wv[q].y - p1) * inv;
          x0 = xs.from(r, tv[q].x) * inv;
          x1 = xs.from(r + 1, tv[q].y) * inv;
          *reinterpret_cast<double2*>(col + r) = make_double2(vj0, vj1);
          *reinterpret_cast<double2*>(ws + r) = make_double2(x0, x1);
          sq = fma(vj0, x0, sq);
          sq = fma(vj1, x1, sq);
        }
        y0 = __shfl_sync(0xffffffffu, x0, lane - g);
        y1 = __shfl_sync(0xffffffffu, x1, lane - g);
      } else {
        y0 = ok ? wv[q].x - p0 : 0.0;
        y1 = ok ? wv[q].y - p1 : 0.0;
        if (ok && g == 0) {
          *reinterpret_cast<double2*>(ws + r) = make_double2(y0, y1);
          sq = fma(y0, y0, sq);
          sq = fma(y1, y1, sq);
        }
      }
#pragma unroll
      for (int i = 0; i < CPT; ++i) acc[i] = fma(v[q][i].y, y1, fma(v[q][i].x, y0, acc[i]));
    }
  }
  return sq;
}

// column sums of the lanes' accumulators -> part[0 .. ncols), and `sq` -> part[ncols]
// red: [V3_THREADS / 32][LN_RED] doubles of shared memory
constexpr int LN_MAXCOL = 128;
constexpr int LN_RED = LN_MAXCOL + 1;
template <int G, int CPT>
__device__ __forceinline__ void lanes_reduce(double (&acc)[CPT], double sq, int ncols, double* part, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    double a = acc[i];
#pragma unroll
    for (int o = G; o < 32; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane < G) red[warp * LN_RED + lane + G * i] = a;
  }
  sq = warp_sum(sq);
  if (lane == 0) red[warp * LN_RED + LN_MAXCOL] = sq;
  __syncthreads();
  for (int c = threadIdx.x; c <= ncols; c += V3_THREADS) {
    const int idx = c < ncols ? c : LN_MAXCOL;
    double a = 0.0;
#pragma unroll
    for (int q = 0; q < V3_THREADS / 32; ++q) a += red[q * LN_RED + idx];
    part[c] = a;
  }
}

template <bool P1B, bool WIDE, class XS>
__device__ __forceinline__ void lanes_dispatch(const double* __restrict__ Vs, long long k, int ncols, const double* hsm,
                                               double* ws, const double* __restrict__ ts, XS xs, double inv, double* col,
                                               int r0, int r1, double* part, double* red) {
  auto run = [&](auto g_tag, auto cpt_tag, auto nr_tag) {
    constexpr int G = decltype(g_tag)::value, CPT = decltype(cpt_tag)::value, NR = decltype(nr_tag)::value;
    double acc[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) acc[i] = 0.0;
    const double sq = lanes_rows<G, CPT, NR, P1B>(Vs, k, ncols, hsm, ws, ts, xs, inv, col, r0, r1, acc);
    lanes_reduce<G, CPT>(acc, sq, ncols, part, red);
  };
  // G lanes x CPT columns >= ncols; CPT x NR independent 16-byte loads per thread in flight.
  // Up to 64 columns (WIDE = false): 2 CTAs per SM at 128 registers, 12-16 loads per thread
  // (100-130 KB per SM).  Beyond (WIDE = true): eight lanes per row pair leave only 64 rows per
  // CTA iteration at NR = 1, and each iteration costs a full memory latency (2.6 TB/s measured
  // with the few systems that run this deep); one CTA per SM at up to 255 registers holds NR = 2-3
  // row groups (28-36 loads per thread, 115-150 KB per SM in flight, half to a third of the iterations)
  using std::integral_constant;
#define SMPM_LANES_CASE(LIM, G_, CPT_, NR_)                                                            \
  if (ncols <= LIM) {                                                                                  \
    run(integral_constant<int, G_>{}, integral_constant<int, CPT_>{}, integral_constant<int, NR_>{}); \
    return;                                                                                            \
  }
  if (!WIDE) {
    SMPM_LANES_CASE(24, 4, 6, 2)
    SMPM_LANES_CASE(32, 4, 8, 2)
    SMPM_LANES_CASE(48, 4, 12, 1)
    SMPM_LANES_CASE(64, 4, 16, 1)
  } else {
#ifdef SMPM_WIDE_G8
    SMPM_LANES_CASE(80, 8, 10, 3)
    SMPM_LANES_CASE(96, 8, 12, (P1B ? 2 : 3))
    SMPM_LANES_CASE(112, 8, 14, 2)
    SMPM_LANES_CASE(128, 8, 16, 2)
#else
    SMPM_LANES_CASE(80, 4, 20, 1)
    SMPM_LANES_CASE(96, 4, 24, 1)
    SMPM_LANES_CASE(112, 4, 28, 1)
    SMPM_LANES_CASE(128, 4, 32, 1)
#endif
  }
#undef SMPM_LANES_CASE
}

// pass 2' for 16 < ncols <= 128 (w -= V h1; h2 = V^T w; ||w||^2; Givens in the last CTA)
template <bool WIDE>
__global__ void __launch_bounds__(V3_THREADS, WIDE ? 1 : 2) cgs5_pass2l_kernel(GmState_ G, const double* __restrict__ V,
                                                                              double* w) {
  pdl_wait();
  __shared__ double hs[V2_MAXCOL];
  __shared__ double red[(V3_THREADS / 32) * LN_RED];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int j = G.jcyc[s];
  const int ncols = j + 1;
  const int stride = G.m + 2;
  const double* hin = G.h1 + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < V2_MAXCOL; i += V3_THREADS) hs[i] = i < ncols ? hin[i] : 0.0;  // zero past ncols
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  lanes_dispatch<false, WIDE>(Vs, G.k, ncols, hs, ws, nullptr, XVal{}, 1.0, nullptr, r0, r1, part, red);
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

// pass 1B for 16 < old columns <= 128
template <bool WIDE>
__global__ void __launch_bounds__(V3_THREADS, WIDE ? 1 : 2) cgs5_pass1bl_kernel(GmState_ G, double* __restrict__ V, double* w,
                                                                     const double* __restrict__ t, int defl,
                                                                     DeflateParams P, const double* __restrict__ cbuf) {
  pdl_wait();
  __shared__ double hs[V2_MAXCOL];
  __shared__ double red[(V3_THREADS / 32) * LN_RED];
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const int nold = G.jcyc[s];
  const int stride = G.m + 2;
  const double* hin = G.h2 + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < V2_MAXCOL; i += V3_THREADS) hs[i] = i < nold ? hin[i] : 0.0;  // zero past nold
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = static_cast<int>(min(G.k, static_cast<long long>(ch) * G.chunk));
  const int r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  const double* ts = t + s * G.k;
  double* col = Vs + static_cast<long long>(nold) * G.k;
  const double inv = 1.0 / G.nrm[s];
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  if (defl) {
    const int wd = P.w, w2 = 2 * wd;
    const double* rs = P.rowsum + static_cast<long long>(s) * 6 * wd;
    const XDeflVal xd{cbuf + static_cast<long long>(s) * P.d, rs, rs + w2, rs + 2 * w2, rs + 2 * w2 + wd, wd, P.mx};
    lanes_dispatch<true, WIDE>(Vs, G.k, nold, hs, ws, ts, xd, inv, col, r0, r1, part, red);
  } else {
    lanes_dispatch<true, WIDE>(Vs, G.k, nold, hs, ws, ts, XVal{}, inv, col, r0, r1, part, red);
  }
  pdl_launch();  // the row work is done: dependents may start launching
  if (last_cta(G.counter + s, G.nchunk))
    reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, nold + 1,
                 G.h1 + static_cast<long long>(s) * stride);
}

}  // namespace smpm
