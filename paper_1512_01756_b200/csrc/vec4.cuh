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
  pdl_launch();
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
}

// ---- pass 1B beyond 16 old columns: shared-memory row tiles (as pass2_tiled) ----
__host__ __device__ __forceinline__ size_t p1bt_smem_doubles(int cap) {
  return p2t_smem_doubles(cap) + 2 * static_cast<size_t>(p2t_rows(cap));
}

template <class XS>
__device__ __forceinline__ double pass1b_tiled(const double* __restrict__ Vs, long long k, int nold, const double* hs,
                                               double* ws, const double* __restrict__ ts, XS xs, double inv,
                                               double* col, int r0, int r1, double* sm, double (&acc)[P2T_MAXC]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int TR = p2t_rows(nold);
  double* tile = sm;                                        // [2][nold][TR]
  double* wt = tile + 2 * static_cast<size_t>(TR) * nold;   // [2][TR]  pending vector u
  double* at = wt + 2 * TR;                                 // [2][TR]  operator output
  double* qp = at + 2 * TR;                                 // [4][TR]
  double* nvs = qp + 4 * TR;                                // [TR]     x of the tile
  const int ntile = (r1 - r0 + TR - 1) / TR;
  const int pieces = TR / 2;
  auto issue = [&](int it) {
    const int a = r0 + it * TR;
    double* tb = tile + static_cast<size_t>(it & 1) * TR * nold;
    for (int p = t; p < nold * pieces; p += V3_THREADS) {
      const int c = p / pieces, q = p - c * pieces;
      const int r = a + 2 * q;
      cp_async16(tb + c * TR + 2 * q, Vs + static_cast<long long>(c) * k + (r < r1 ? r : r0), r < r1);
    }
    for (int q = t; q < 2 * pieces; q += V3_THREADS) {
      const int which = q >= pieces ? 1 : 0, qq = q - which * pieces;
      const int r = a + 2 * qq;
      const double* src = which ? ts : ws;
      double* dst = (which ? at : wt) + (it & 1) * TR + 2 * qq;
      cp_async16(dst, src + (r < r1 ? r : r0), r < r1);
    }
  };
  double accn = 0.0;
  issue(0);
  cp_async_commit();
  const int quarter = t >> 6, qrow = t & 63;
  const int qc = (nold + 3) >> 2;
  const int c0q = quarter * qc, c1q = min(nold, c0q + qc);
  for (int it = 0; it < ntile; ++it) {
    if (it + 1 < ntile) issue(it + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* tb = tile + static_cast<size_t>(it & 1) * TR * nold;
    const double* wb = wt + (it & 1) * TR;
    const double* ab = at + (it & 1) * TR;
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
  double accn = pass1b_tiled(Vs, G.k, nold, hs, ws, ts, xs, inv, col, r0, r1, sm, acc);
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
  pdl_launch();
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
}

}  // namespace smpm
