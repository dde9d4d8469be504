// Parity-split shared-matrix transform kernels (sm_100a).
//
// The z factor of every strip block commutes with the reflection z -> l_z - z
// (uniform elements, symmetric GLL nodes), so each column of the spectral basis
// T — and each row of T^{-1} — is an even or an odd function of the node index
// inside a w-block (fdm.py builds them exactly parity-pure).  With h = w / 2,
// J the reversal and s_m = +-1 the parity of eigenmode m:
//
//   forward   (T^{-1} x)_m      = sum_{k<h} T^{-1}[m, k] (x[k] + s_m x[w-1-k])
//   backward  (T t)[k]          = E[k] + O[k]
//             (T t)[w-1-k]      = E[k] - O[k],    E = sum_{m even} T[k, m] t_m,
//                                                  O = sum_{m odd}  T[k, m] t_m
//
// i.e. two h x h contractions instead of one w x w: HALF the fp64 MMA work of
// xform.cuh / xformk.cuh for the same result up to rounding.  The fold
// (x[k] +- x[w-1-k]) and the unfold (E +- O) happen inside the kernels: vectors
// stay in nodal order everywhere else.
//
// Kernel shape (both directions), as xformk.cuh: grid = P row slices x G column
// groups, one persistent CTA per SM; a CTA walks its columns in chunks of 64
// (8 n-blocks) and the contraction index in stages of 16 through an NS-deep
// ring; the A slab of a stage (DMMA fragment order, one contiguous block) comes
// by ONE bulk copy (cp.async.bulk on an mbarrier, SASS UBLKCP), the columns by
// 16-byte cp.async; one CTA barrier per stage; warp (s, hh) computes n-blocks
// s, s + 4 for half hh of the slice's m-blocks with m8n8k4 f64 MMA (DMMA).
//   forward : a slice is single-parity rows (eigenmodes); a stage carries the
//             low 16 entries x[k0 .. k0+16) and the mirrored high 16 of every
//             column, folded as the B fragments are read from shared memory;
//   backward: a slice is rows k < h; the stages run over the even modes into
//             accumulator set E, then over the odd modes into set O; the
//             epilogue writes E + O to row k and E - O to row w - 1 - k.
// Mode order (fdm.real_basis): complex pairs first (even, then odd), then real
// modes (even, then odd) — so the modes of one parity are two contiguous,
// 16-byte aligned segments.  Summation order per output element is fixed.
#pragma once

#include "common.cuh"
#include "gemm2.cuh"
#include "xform.cuh"
#include "xformk.cuh"

namespace smpm {

struct XformPArgs {
  XformArgs x;      // vectors, live list, w, Af (the image of this direction), P
  int h;            // w / 2
  int ks;           // stages per parity: ceil(h / 16)
  int seg_start[2][2];  // [parity][segment]: first mode index
  int seg_len0[2];      // [parity]: length of segment 0
};

__host__ __device__ __forceinline__ int xp_mode(const int (&start)[2][2], const int (&len0)[2], int par, int kap) {
  return kap < len0[par] ? start[par][0] + kap : start[par][1] + (kap - len0[par]);
}

// Host: A image of one direction.  get(row, par, kap) is the matrix entry of
// slice-row `row` against contraction index kap of parity par (0 outside).
//   forward : slices [0, Ps) even rows, [Ps, 2 Ps) odd rows, stages = ks (own parity)
//   backward: P slices of rows k, stages = 2 ks (even modes, then odd modes)
template <class Get>
inline void xformp_image(int nslice, int nstage, int MB, Get get, std::vector<double>& F) {
  F.assign(static_cast<size_t>(nslice) * nstage * 2 * MB * 64, 0.0);
  for (int sl = 0; sl < nslice; ++sl)
    for (int q = 0; q < nstage; ++q)
      for (int g = 0; g < 2; ++g)
        for (int mb = 0; mb < MB; ++mb)
          for (int ln = 0; ln < 32; ++ln)
            for (int e = 0; e < 2; ++e) {
              const int r = mb * 8 + ln / 4, kk = 16 * q + 8 * g + 2 * (ln % 4) + e;
              F[(((((static_cast<size_t>(sl) * nstage + q) * 2 + g) * MB + mb) * 32 + ln) * 2) + e] = get(sl, r, kk);
            }
}

// forward stage: B fragments folded from the low slab and the mirrored high slab
template <int MB, int NMB, int NNB>
__device__ __forceinline__ void xp_stage_fwd(const double* Ap, const double* Blo, const double* Bhi, double sg,
                                             double (&acc)[NMB][2][2]) {
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    double2 bf[NNB], af[NMB];
#pragma unroll
    for (int jn = 0; jn < NNB; ++jn) {
      const double2 lo = lds128(Blo + jn * 32 * XK_BSTR + 8 * g);
      const double2 hi = lds128(Bhi + jn * 32 * XK_BSTR - 8 * g);
      bf[jn].x = fma(sg, hi.y, lo.x);
      bf[jn].y = fma(sg, hi.x, lo.y);
    }
#pragma unroll
    for (int i = 0; i < NMB; ++i) af[i] = lds128(Ap + (g * MB + i) * 64);
#pragma unroll
    for (int jn = 0; jn < NNB; ++jn)
#pragma unroll
      for (int i = 0; i < NMB; ++i) dmma884(acc[i][jn], af[i].x, bf[jn].x);
#pragma unroll
    for (int jn = 0; jn < NNB; ++jn)
#pragma unroll
      for (int i = 0; i < NMB; ++i) dmma884(acc[i][jn], af[i].y, bf[jn].y);
  }
}

template <int MB, int NMB, int NS, bool BWD>
__device__ __forceinline__ void xp_warp(const XformPArgs& pa, double* ring, unsigned long long* full, int c0, int c1,
                                        int slice, int mb0, int cps, const double* Aslice) {
  const XformArgs& a = pa.x;
  const int t = threadIdx.x, lane = t & 31, nb = (t >> 5) & 3;
  const int w = a.w, h = pa.h;
  const int KS = BWD ? 2 * pa.ks : pa.ks;  // stages per chunk
  const int nch = (c1 - c0 + XF_NT - 1) / XF_NT;
  const int nst = nch * KS;
  constexpr int ASTAGE = xk_astage(MB);
  constexpr int BSTAGE = BWD ? XK_BSTAGE : 2 * XK_BSTAGE;
  constexpr int STAGE = ASTAGE + BSTAGE;
  constexpr unsigned ABYTES = static_cast<unsigned>(ASTAGE * sizeof(double));
  // forward: slices [0, P/2) hold even rows, [P/2, P) odd rows
  const int Ps = BWD ? a.P : a.P / 2;
  const int par = BWD ? 0 : slice / Ps;
  const int row0 = (BWD ? slice : slice % Ps) * 8 * MB;
  const double sg = par ? -1.0 : 1.0;
  // loader: thread t moves 16-byte pieces lq and lq + 4 of column lc of a B slab
  const int lc = t >> 2, lq = t & 3;
  const double* lsrc = nullptr;
  auto issue = [&](int sidx) {
    const int ci = sidx / KS, kq = sidx - ci * KS;
    double* st = ring + static_cast<size_t>(sidx % NS) * STAGE;
    if (kq == 0) lsrc = xf_in_col(a, c0 + ci * XF_NT + lc, c1, cps);
    if (t == 0) {
      mbar_expect_tx(full + sidx % NS, ABYTES);
      bulk_g2s(st, Aslice + static_cast<size_t>(kq) * ASTAGE, ABYTES, full + sidx % NS);
    }
    double* dst = st + ASTAGE + lc * XK_BSTR;
    const bool ok = lsrc != nullptr;
    const double* src = ok ? lsrc : a.in[0];
    if constexpr (BWD) {
      // 16 consecutive modes of one parity (two aligned segments); past h: zeros
      const int pq = kq >= pa.ks ? 1 : 0;
      const int kap0 = (kq - pq * pa.ks) * XK_KS;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int kap = kap0 + 2 * (lq + 4 * u);
        const bool in = ok && kap < h;
        const int m = in ? xp_mode(pa.seg_start, pa.seg_len0, pq, kap) : 0;
        cp_async16(dst + 2 * (lq + 4 * u), src + m, in);
      }
    } else {
      // low entries x[k0, k0 + 16) and their mirrors x[w - k0 - 16, w - k0)
      const int k0 = kq * XK_KS;
      cp_async16(dst + 2 * lq, src + k0 + 2 * lq, ok);
      cp_async16(dst + 2 * lq + 8, src + k0 + 2 * lq + 8, ok);
      double* dhi = dst + XK_BSTAGE;
      const double* shi = src + (w - k0 - XK_KS);
      cp_async16(dhi + 2 * lq, shi + 2 * lq, ok);
      cp_async16(dhi + 2 * lq + 8, shi + 2 * lq + 8, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nst) issue(s);
    cp_async_commit();
  }
  constexpr int NSET = BWD ? 2 : 1;
  double acc[NSET][NMB][2][2];
  double* ocol[2][2];
  for (int sidx = 0; sidx < nst; ++sidx) {
    const int ci = sidx / KS, kq = sidx - ci * KS;
    const int cb = c0 + ci * XF_NT;
    cp_async_wait<NS - 2>();
    mbar_wait(full + sidx % NS, static_cast<unsigned>((sidx / NS) & 1));
    __syncthreads();  // stage sidx visible to all; every warp is past stage sidx - 1
    if (sidx + NS - 1 < nst) issue(sidx + NS - 1);
    cp_async_commit();
    if (kq == 0) {
#pragma unroll
      for (int z = 0; z < NSET; ++z)
#pragma unroll
        for (int i = 0; i < NMB; ++i) acc[z][i][0][0] = acc[z][i][0][1] = acc[z][i][1][0] = acc[z][i][1][1] = 0.0;
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int e = 0; e < 2; ++e) ocol[jn][e] = xf_out_col(a, cb + nb * 8 + 32 * jn + 2 * (lane & 3) + e, c1, cps);
    }
    const double* st = ring + static_cast<size_t>(sidx % NS) * STAGE;
    const double* Ap = st + (mb0 * 32 + lane) * 2;
    const double* Bp = st + ASTAGE + (nb * 8 + (lane >> 2)) * XK_BSTR + 2 * (lane & 3);
    const bool wide = cb + 32 < c1;
    if constexpr (BWD) {
      if (kq < pa.ks) {
        if (wide)
          xf_stage<MB, NMB, 2, 2>(Ap, Bp, XK_BSTR, 0, 2, acc[0]);
        else
          xf_stage<MB, NMB, 1, 2>(Ap, Bp, XK_BSTR, 0, 2, acc[0]);
      } else {
        if (wide)
          xf_stage<MB, NMB, 2, 2>(Ap, Bp, XK_BSTR, 0, 2, acc[NSET - 1]);
        else
          xf_stage<MB, NMB, 1, 2>(Ap, Bp, XK_BSTR, 0, 2, acc[NSET - 1]);
      }
    } else {
      // mirror of entry 8 g + 2 j (and + 1) of the low slab: entries 14 - 8 g - 2 j (+ 1) of the high slab
      const double* Bh = st + ASTAGE + XK_BSTAGE + (nb * 8 + (lane >> 2)) * XK_BSTR + 14 - 2 * (lane & 3);
      if (wide)
        xp_stage_fwd<MB, NMB, 2>(Ap, Bp, Bh, sg, acc[0]);
      else
        xp_stage_fwd<MB, NMB, 1>(Ap, Bp, Bh, sg, acc[0]);
    }
    if (kq == KS - 1) {
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double* o = ocol[jn][e];
          if (o) {
#pragma unroll
            for (int i = 0; i < NMB; ++i) {
              const int r = row0 + (mb0 + i) * 8 + (lane >> 2);
              if (r < h) {
                if constexpr (BWD) {
                  const double ev = acc[0][i][jn][e], od = acc[NSET - 1][i][jn][e];
                  o[r] = ev + od;
                  o[w - 1 - r] = ev - od;
                } else {
                  o[xp_mode(pa.seg_start, pa.seg_len0, par, r)] = acc[0][i][jn][e];
                }
              }
            }
          }
        }
    }
  }
  cp_async_wait<0>();
}

// smem: ring[NS][A slab | B slab(s)] | full[NS] mbarriers
template <int MB, int NS, bool BWD>
__global__ void __launch_bounds__(XF_THREADS, 1) xformp_kernel(XformPArgs pa) {
  pdl_wait();
  extern __shared__ __align__(128) double xp_smem[];
  const XformArgs& a = pa.x;
  constexpr int STAGE = xk_astage(MB) + (BWD ? XK_BSTAGE : 2 * XK_BSTAGE);
  double* ring = xp_smem;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xp_smem + static_cast<size_t>(NS) * STAGE);
  const int t = threadIdx.x, warp = t >> 5;
  const int slice = blockIdx.x % a.P, grp = blockIdx.x / a.P, ngrp = gridDim.x / a.P;
  const int L = a.acount ? min(*a.acount, a.nslots) : a.nslots;
  const int cps = L * a.ncol_sys;
  const int ncols = cps * a.nv;
  const int share = ((ncols + ngrp - 1) / ngrp + 7) & ~7;
  const int c0 = grp * share, c1 = min(ncols, c0 + share);
  if (c0 >= c1) return;
  if (t == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nstage = BWD ? 2 * pa.ks : pa.ks;
  const double* Aslice = a.Af + static_cast<size_t>(slice) * nstage * xk_astage(MB);
  constexpr int MB0 = (MB + 1) / 2;
  if (warp < 4)
    xp_warp<MB, MB0, NS, BWD>(pa, ring, full, c0, c1, slice, 0, cps, Aslice);
  else
    xp_warp<MB, MB - MB0, NS, BWD>(pa, ring, full, c0, c1, slice, MB0, cps, Aslice);
  pdl_launch();  // dependents may start launching: this CTA's main work is done
}

template <int MB, int NS, bool BWD>
constexpr size_t xformp_smem() {
  return sizeof(double) * static_cast<size_t>(NS) * (xk_astage(MB) + (BWD ? XK_BSTAGE : 2 * XK_BSTAGE)) +
         NS * sizeof(unsigned long long);
}

}  // namespace smpm
