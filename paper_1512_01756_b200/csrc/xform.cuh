// Shared-matrix transform kernel (sm_100a): Y = A X for one w x w matrix A
// (T or T^{-1} of the spectral form, spectral.cuh) applied to every w-block
// of every live system of a batch — the "A^{-1}B sweep as one dense GEMM
// over all elements" of the north star.
//
// The matrix is shared by all M = w rows x N = 2d * live-systems columns, so
// instead of streaming it per output tile (gemm2.cuh), each CTA keeps one
// row slice of A resident in shared memory for the whole launch, in DMMA
// fragment order (copied once from a pre-ordered global image), and streams
// only the columns:
//   * grid = P slices x G column groups, one CTA per SM (persistent); group g
//     owns a contiguous, 8-aligned range of the batch's columns and walks it in
//     chunks of up to 64 columns; CTA (slice, g) computes the slice's rows;
//   * each chunk streams through a two-slot cp.async ring in two K halves
//     ([column][k] layout, row stride = 64 mod 128 bytes: conflict-free
//     LDS.128), the ring running across chunk boundaries: one CTA barrier
//     pair per half chunk (w / 16 k8 groups of DMMAs);
//   * the m8n8k4 f64 MMA (DMMA, the fp64 tensor pipe; tcgen05 has no f64
//     kind) runs two k-steps per fragment load: inside each group of 8 k's a
//     lane feeds k = 2j in the first step and k = 2j + 1 in the second
//     (j = lane % 4), for A and B alike, so a step pair's fragment is one
//     16-byte load;
//   * warp (s, h) (SMSP s = warp % 4, half h = warp / 4) computes n-blocks s
//     and s + 4 of the chunk for the h-th half of the slice's m-blocks: every
//     tensor pipe gets equal work, and a chunk of <= 32 columns still spreads
//     over all four.
// Per-element summation order is fixed (k ascending): results are
// run-to-run deterministic.
#pragma once

#include "common.cuh"
#include "gemm2.cuh"

namespace smpm {

constexpr int XF_THREADS = 256;
constexpr int XF_NT = 64;      // columns per chunk (8 n-blocks)
constexpr int XF_NS = 2;       // ring depth: a stage is half of K (w / 2), one CTA barrier per half chunk

// ring row stride for a stage of ks k's (doubles): = 64 mod 128 bytes -> conflict-free LDS.128
__host__ __device__ __forceinline__ int xf_bstr(int ks) { return ks % 16 == 0 ? ks + 8 : ks + 16; }

struct XformArgs {
  const double* Af;      // P row slices of the w x w matrix in DMMA fragment order (xform_frag_order)
  int w;                 // rows = cols = w (multiple of 16)
  int ncol_sys;          // 2d columns (w-blocks) per system
  long long k;           // system stride (doubles)
  const int* alist;      // live systems (nullptr: slot == system)
  const int* acount;     // live count (nullptr: nslots)
  int nslots;
  int nv;                // 1 or 2 (in, out) pairs (columns of pair 1 follow those of pair 0)
  const double* in[2];
  double* out[2];
  int P;                 // row slices
};

// Fragment order of a w x w column-major matrix A for P slices of 8*MB rows:
// F[((slice*K8 + p)*MB + mb)*32 + ln] = (A[r][8p+2j], A[r][8p+2j+1]) as double2,
// r = slice*8*MB + mb*8 + ln/4, j = ln%4; rows past w are zero (host setup).
inline void xform_frag_order(const double* A, int w, int P, int MB, double* F) {
  const int K8 = w / 8;
  for (int sl = 0; sl < P; ++sl)
    for (int p = 0; p < K8; ++p)
      for (int mb = 0; mb < MB; ++mb)
        for (int ln = 0; ln < 32; ++ln)
          for (int e = 0; e < 2; ++e) {
            const int r = sl * 8 * MB + mb * 8 + ln / 4, kk = 8 * p + 2 * (ln % 4) + e;
            F[((((static_cast<size_t>(sl) * K8 + p) * MB + mb) * 32 + ln) * 2) + e] =
                r < w ? A[static_cast<size_t>(kk) * w + r] : 0.0;
          }
}

__device__ __forceinline__ double2 lds128(const double* p) {
  double2 v;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

// offset of column gc of the batch (pair 1's columns follow pair 0's)
__device__ __forceinline__ long long xf_col_off(const XformArgs& a, int gc, int cps, int& v) {
  v = gc >= cps ? 1 : 0;
  const int c = gc - v * cps;
  const int q = c / a.ncol_sys, cc = c - q * a.ncol_sys;
  const int s = a.alist ? a.alist[q] : q;
  return s * a.k + static_cast<long long>(cc) * a.w;
}

// one ring stage (ks / 8 k8 groups) of one warp: NMB m-blocks, n-blocks nb and
// nb + 4 (NNB = 2) or nb only (NNB = 1)
template <int MB, int NMB, int NNB, int NG>
__device__ __forceinline__ void xf_stage(const double* Ap, const double* Bp, int bstr, int p0, int ng_rt,
                                         double (&acc)[NMB][2][2]) {
  const int ng = NG > 0 ? NG : ng_rt;  // compile-time group count: fully unrolled stage
#pragma unroll(NG > 0 ? NG : 2)
  for (int g = 0; g < ng; ++g) {
    double2 bf[NNB], af[NMB];
#pragma unroll
    for (int jn = 0; jn < NNB; ++jn) bf[jn] = lds128(Bp + jn * 32 * bstr + 8 * g);
#pragma unroll
    for (int i = 0; i < NMB; ++i) af[i] = lds128(Ap + ((p0 + g) * MB + i) * 64);
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

// batch column gc -> its vector (pair v) and offset; nullptr past the range
__device__ __forceinline__ const double* xf_in_col(const XformArgs& a, int gc, int c1, int cps) {
  if (gc >= c1) return nullptr;
  int v;
  const long long off = xf_col_off(a, gc, cps, v);
  return (v ? a.in[1] : a.in[0]) + off;
}
__device__ __forceinline__ double* xf_out_col(const XformArgs& a, int gc, int c1, int cps) {
  if (gc >= c1) return nullptr;
  int v;
  const long long off = xf_col_off(a, gc, cps, v);
  return (v ? a.out[1] : a.out[0]) + off;
}

template <int MB, int NMB>
__device__ __forceinline__ void xf_warp(const XformArgs& a, const double* Af, double* ring, int c0, int c1, int row0,
                                        int mb0, int cps) {
  const int t = threadIdx.x, lane = t & 31, nb = (t >> 5) & 3;
  const int w = a.w, ks = w / 2, bstr = xf_bstr(ks), hp = ks / 2;  // 16-byte pieces per column and stage
  const int nch = (c1 - c0 + XF_NT - 1) / XF_NT;
  const int nst = nch * 2;  // ring stages of this CTA (two per chunk)
  // loader: thread t moves pieces t%4, t%4 + 4, ... of column t/4 of a stage; the
  // column addresses of a chunk are resolved one chunk ahead (no dependent loads
  // or divisions on the issue path)
  const int lc = t >> 2, lq = t & 3;
  const double* lsrc = xf_in_col(a, c0 + lc, c1, cps);                 // chunk 0
  const double* lnext = xf_in_col(a, c0 + XF_NT + lc, c1, cps);        // chunk 1
  auto load = [&](int sidx) {
    const int q = sidx & 1;
    double* dst = ring + static_cast<size_t>(sidx % XF_NS) * XF_NT * bstr + lc * bstr;
    const double* src = lsrc ? lsrc + q * ks : a.in[0];
    for (int i = lq; i < hp; i += 4) cp_async16(dst + 2 * i, src + 2 * i, lsrc != nullptr);
  };
  load(0);
  cp_async_commit();
  const double* Ap = Af + (mb0 * 32 + lane) * 2;
  double acc[NMB][2][2];
  double* ocol[2][2];
  for (int sidx = 0; sidx < nst; ++sidx) {
    const int ci = sidx >> 1, q = sidx & 1;
    const int cb = c0 + ci * XF_NT;  // first column of the chunk
    __syncthreads();  // the slot about to be refilled was consumed
    if (sidx + 1 < nst) {
      if (q == 1) {  // next stage starts chunk ci + 1; resolve chunk ci + 2 for later
        lsrc = lnext;
        lnext = xf_in_col(a, cb + 2 * XF_NT + lc, c1, cps);
      }
      load(sidx + 1);
    }
    cp_async_commit();
    if (q == 0) {
#pragma unroll
      for (int i = 0; i < NMB; ++i) acc[i][0][0] = acc[i][0][1] = acc[i][1][0] = acc[i][1][1] = 0.0;
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int e = 0; e < 2; ++e) ocol[jn][e] = xf_out_col(a, cb + nb * 8 + 32 * jn + 2 * (lane & 3) + e, c1, cps);
    }
    cp_async_wait<1>();
    __syncthreads();
    const double* Bp = ring + static_cast<size_t>(sidx % XF_NS) * XF_NT * bstr + (nb * 8 + (lane >> 2)) * bstr + 2 * (lane & 3);
    const int ng = ks / 8;
    if (cb + 32 < c1) {
      if (ng == 11)
        xf_stage<MB, NMB, 2, 11>(Ap, Bp, bstr, q * ng, ng, acc);
      else
        xf_stage<MB, NMB, 2, 0>(Ap, Bp, bstr, q * ng, ng, acc);
    } else {
      xf_stage<MB, NMB, 1, 0>(Ap, Bp, bstr, q * ng, ng, acc);
    }
    if (q == 1) {
      // epilogue: lane holds rows row0 + (mb0+i)*8 + lane/4 of columns nb*8 + 32*jn + 2*(lane%4) + e
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double* o = ocol[jn][e];
          if (o) {
#pragma unroll
            for (int i = 0; i < NMB; ++i) {
              const int r = row0 + (mb0 + i) * 8 + (lane >> 2);
              if (r < w) o[r] = acc[i][jn][e];
            }
          }
        }
    }
  }
  cp_async_wait<0>();
}

// smem: Af[w/8][MB][32] double2 (A slice, fragment order) | ring[XF_NS][XF_NT][xf_bstr(w/2)]
template <int MB>
__global__ void __launch_bounds__(XF_THREADS, 1) xform_kernel(XformArgs a) {
  pdl_wait();
  extern __shared__ __align__(16) double xf_smem[];
  const int t = threadIdx.x, warp = t >> 5;
  const int K8 = a.w >> 3;
  const int slice = blockIdx.x % a.P, grp = blockIdx.x / a.P, ngrp = gridDim.x / a.P;
  double* Af = xf_smem;
  double* ring = xf_smem + static_cast<size_t>(K8) * MB * 64;
  const int L = a.acount ? min(*a.acount, a.nslots) : a.nslots;
  const int cps = L * a.ncol_sys;  // columns per (in, out) pair
  const int ncols = cps * a.nv;
  // this group's column range: 8-aligned equal shares
  const int share = ((ncols + ngrp - 1) / ngrp + 7) & ~7;
  const int c0 = grp * share, c1 = min(ncols, c0 + share);
  if (c0 >= c1) return;
  // resident A slice: a contiguous block of the fragment-ordered image
  {
    const double* src = a.Af + static_cast<size_t>(slice) * K8 * MB * 64;
    for (int e = t; e < K8 * MB * 32; e += XF_THREADS) cp_async16(Af + 2 * e, src + 2 * e, true);
    cp_async_commit();
  }
  constexpr int MB0 = (MB + 1) / 2;
  const int row0 = slice * 8 * MB;
  if (warp < 4)
    xf_warp<MB, MB0>(a, Af, ring, c0, c1, row0, 0, cps);
  else
    xf_warp<MB, MB - MB0>(a, Af, ring, c0, c1, row0, MB0, cps);
  pdl_launch();  // dependents may start launching: this CTA's main work is done
}

}  // namespace smpm
