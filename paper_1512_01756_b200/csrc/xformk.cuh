// K-streamed shared-matrix transform kernel (sm_100a) for w x w matrices too
// large to keep a row slice resident (w > 176: C2 w = 416, C3 w = 272,
// C5 w = 544).  Same contraction as xform.cuh — Y = A X for one w x w matrix
// A (T or T^{-1}) and every w-block column of the live systems — and the same
// warp tiling, but A streams through shared memory together with the columns:
//   * grid = P row slices x G column groups, one CTA per SM (persistent); CTA
//     (slice, g) computes rows [slice*8*MB, +8*MB) of its group's columns,
//     walking them in chunks of 64 columns (8 n-blocks);
//   * the K dimension of a chunk runs in stages of 16 k's through an NS-deep
//     ring; a stage holds the A slab (8*MB rows x 16 k, already in DMMA
//     fragment order in global memory, so it is one contiguous block) and the
//     B slab (64 columns x 16 k);
//   * the A slab arrives by ONE bulk copy (cp.async.bulk, the TMA copy engine;
//     SASS UBLKCP) issued by one thread and completed on an mbarrier with a
//     byte count, the B slab by 16-byte cp.async (two per thread; columns are
//     gathered through the live-system list, so they are not one box);
//   * one CTA barrier per stage: after it every warp has finished the stage
//     whose slot is refilled next, so the refill is issued right behind it,
//     NS - 1 stages ahead of the compute;
//   * warp (s, h) computes n-blocks s and s + 4 of the chunk for half h of the
//     slice's m-blocks with m8n8k4 f64 MMA (DMMA; tcgen05 has no f64 kind), two
//     k-steps per 16-byte fragment load (xf_stage).
// The accumulation order of every output element is k ascending in steps of
// 4 (fixed): deterministic, and independent of the batch composition.
#pragma once

#include "common.cuh"
#include "gemm2.cuh"
#include "xform.cuh"

namespace smpm {

constexpr int XK_KS = 16;                   // k's per ring stage
constexpr int XK_BSTR = 24;                 // B slab row stride (doubles): 192 B = 64 mod 128 -> conflict-free LDS.128
constexpr int XK_BSTAGE = XF_NT * XK_BSTR;  // doubles of a B slab

__host__ __device__ constexpr int xk_astage(int MB) { return 2 * MB * 64; }  // doubles of an A slab (2 k8 groups)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// one contiguous global -> shared copy on the TMA engine, completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int MB, int NMB, int NS>
__device__ __forceinline__ void xk_warp(const XformArgs& a, double* ring, unsigned long long* full, int c0, int c1,
                                        int row0, int mb0, int cps, const double* Aslice) {
  const int t = threadIdx.x, lane = t & 31, nb = (t >> 5) & 3;
  const int w = a.w;
  const int KS = w / XK_KS;  // stages per chunk
  const int nch = (c1 - c0 + XF_NT - 1) / XF_NT;
  const int nst = nch * KS;
  constexpr int STAGE = xk_astage(MB) + XK_BSTAGE;
  constexpr unsigned ABYTES = static_cast<unsigned>(xk_astage(MB) * sizeof(double));
  // loader: thread t moves 16-byte pieces lq and lq + 4 of column lc of a B slab
  const int lc = t >> 2, lq = t & 3;
  const double* lsrc = nullptr;
  auto issue = [&](int sidx) {
    const int ci = sidx / KS, kq = sidx - ci * KS;
    double* st = ring + static_cast<size_t>(sidx % NS) * STAGE;
    if (kq == 0) lsrc = xf_in_col(a, c0 + ci * XF_NT + lc, c1, cps);
    if (t == 0) {
      mbar_expect_tx(full + sidx % NS, ABYTES);
      bulk_g2s(st, Aslice + static_cast<size_t>(kq) * xk_astage(MB), ABYTES, full + sidx % NS);
    }
    double* dst = st + xk_astage(MB) + lc * XK_BSTR;
    const double* src = lsrc ? lsrc + kq * XK_KS : a.in[0];
    cp_async16(dst + 2 * lq, src + 2 * lq, lsrc != nullptr);
    cp_async16(dst + 2 * lq + 8, src + 2 * lq + 8, lsrc != nullptr);
  };
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nst) issue(s);
    cp_async_commit();
  }
  double acc[NMB][2][2];
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
      for (int i = 0; i < NMB; ++i) acc[i][0][0] = acc[i][0][1] = acc[i][1][0] = acc[i][1][1] = 0.0;
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int e = 0; e < 2; ++e) ocol[jn][e] = xf_out_col(a, cb + nb * 8 + 32 * jn + 2 * (lane & 3) + e, c1, cps);
    }
    const double* st = ring + static_cast<size_t>(sidx % NS) * STAGE;
    const double* Ap = st + (mb0 * 32 + lane) * 2;
    const double* Bp = st + xk_astage(MB) + (nb * 8 + (lane >> 2)) * XK_BSTR + 2 * (lane & 3);
    if (cb + 32 < c1)
      xf_stage<MB, NMB, 2, 2>(Ap, Bp, XK_BSTR, 0, 2, acc);
    else
      xf_stage<MB, NMB, 1, 2>(Ap, Bp, XK_BSTR, 0, 2, acc);
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
              if (r < w) o[r] = acc[i][jn][e];
            }
          }
        }
    }
  }
  cp_async_wait<0>();
}

// smem: ring[NS][A slab | B slab] | full[NS] mbarriers
template <int MB, int NS>
__global__ void __launch_bounds__(XF_THREADS, 1) xformk_kernel(XformArgs a) {
  pdl_wait();
  extern __shared__ __align__(128) double xk_smem[];
  constexpr int STAGE = xk_astage(MB) + XK_BSTAGE;
  double* ring = xk_smem;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xk_smem + static_cast<size_t>(NS) * STAGE);
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
  const int K8 = a.w >> 3;
  const double* Aslice = a.Af + static_cast<size_t>(slice) * K8 * MB * 64;
  constexpr int MB0 = (MB + 1) / 2;
  const int row0 = slice * 8 * MB;
  if (warp < 4)
    xk_warp<MB, MB0, NS>(a, ring, full, c0, c1, row0, 0, cps, Aslice);
  else
    xk_warp<MB, MB - MB0, NS>(a, ring, full, c0, c1, row0, MB0, cps, Aslice);
  pdl_launch();  // dependents may start launching: this CTA's main work is done
}

template <int MB, int NS>
constexpr size_t xformk_smem() {
  return sizeof(double) * static_cast<size_t>(NS) * (xk_astage(MB) + XK_BSTAGE) + NS * sizeof(unsigned long long);
}

}  // namespace smpm
