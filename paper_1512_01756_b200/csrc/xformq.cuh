// Warp-specialised variant of the parity-split transform kernels (sm_100a).
//
// Same contraction, tiling, images and results as xformp.cuh; the stage ring is
// driven by mbarriers alone instead of one CTA barrier per stage:
//   * warp 8 is the producer (its warpgroup gives its registers to the consumers
//     with setmaxnreg): per stage it waits for the slot to be released
//     (empty[slot], one arrival per consumer warp), then issues the A slab as
//     one bulk copy (cp.async.bulk, complete_tx on full[slot]) and the column
//     slab(s) as 16-byte cp.async copies whose completion arrives on the same
//     barrier (cp.async.mbarrier.arrive.noinc);
//   * warps 0-7 are consumers: wait on full[slot], run the stage's DMMAs,
//     release the slot.  They never meet at a CTA barrier, so a warp that
//     finishes a stage early starts the next one instead of idling, and the
//     producer runs up to NS - 1 stages ahead of the slowest consumer.
#pragma once

#include "xformp.cuh"

namespace smpm {


__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrival on `bar` when all cp.async copies this thread has issued so far have landed
__device__ __forceinline__ void cp_async_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int MB, int NS, bool BWD, bool ARES>
__device__ __forceinline__ void xq_producer(const XformPArgs& pa, double* ring, unsigned long long* full,
                                            unsigned long long* empty, int c0, int c1, int cps, const double* Aslice) {
  const XformArgs& a = pa.x;
  const int lane = threadIdx.x & 31;
  const int w = a.w, h = pa.h;
  const int KS = BWD ? 2 * pa.ks : pa.ks;
  const int nch = (c1 - c0 + XF_NT - 1) / XF_NT;
  const int nst = nch * KS;
  constexpr int ASTAGE = xk_astage(MB);
  constexpr int BSTAGE = BWD ? XK_BSTAGE : 2 * XK_BSTAGE;
  constexpr int AOFF = ARES ? 0 : ASTAGE;  // resident A: the ring holds the column slabs only
  constexpr int STAGE = AOFF + BSTAGE;
  constexpr unsigned ABYTES = static_cast<unsigned>(ASTAGE * sizeof(double));
  const double* col[2] = {nullptr, nullptr};  // this lane's columns lane, lane + 32 of the chunk
  for (int sidx = 0; sidx < nst; ++sidx) {
    const int ci = sidx / KS, kq = sidx - ci * KS;
    const int slot = sidx % NS, use = sidx / NS;
    if (kq == 0) {
      col[0] = xf_in_col(a, c0 + ci * XF_NT + lane, c1, cps);
      col[1] = xf_in_col(a, c0 + ci * XF_NT + lane + 32, c1, cps);
    }
    if (use > 0) mbar_wait(empty + slot, static_cast<unsigned>((use - 1) & 1));
    double* st = ring + static_cast<size_t>(slot) * STAGE;
    if (!ARES && lane == 0) {
      mbar_expect_tx(full + slot, ABYTES);
      bulk_g2s(st, Aslice + static_cast<size_t>(kq) * ASTAGE, ABYTES, full + slot);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      double* dst = st + AOFF + (lane + 32 * u) * XK_BSTR;
      const bool ok = col[u] != nullptr;
      const double* src = ok ? col[u] : a.in[0];
      if constexpr (BWD) {
        const int pq = kq >= pa.ks ? 1 : 0;
        const int kap0 = (kq - pq * pa.ks) * XK_KS;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int kap = kap0 + 2 * q;
          const bool in = ok && kap < h;
          const int m = in ? xp_mode(pa.seg_start, pa.seg_len0, pq, kap) : 0;
          cp_async16(dst + 2 * q, src + m, in);
        }
      } else {
        const int k0 = kq * XK_KS;
        const double* shi = src + (w - k0 - XK_KS);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          cp_async16(dst + 2 * q, src + k0 + 2 * q, ok);
          cp_async16(dst + XK_BSTAGE + 2 * q, shi + 2 * q, ok);
        }
      }
    }
    cp_async_arrive_noinc(full + slot);
  }
}

template <int MB, int NMB, int NS, bool BWD, bool ARES>
__device__ __forceinline__ void xq_consumer(const XformPArgs& pa, const double* ring, unsigned long long* full,
                                            unsigned long long* empty, int c0, int c1, int slice, int mb0, int cps,
                                            const double* Ares) {
  const XformArgs& a = pa.x;
  const int t = threadIdx.x, lane = t & 31, nb = (t >> 5) & 3;
  const int w = a.w, h = pa.h;
  const int KS = BWD ? 2 * pa.ks : pa.ks;
  const int nch = (c1 - c0 + XF_NT - 1) / XF_NT;
  const int nst = nch * KS;
  constexpr int ASTAGE = xk_astage(MB);
  constexpr int BSTAGE = BWD ? XK_BSTAGE : 2 * XK_BSTAGE;
  constexpr int AOFF = ARES ? 0 : ASTAGE;
  constexpr int STAGE = AOFF + BSTAGE;
  const int Ps = BWD ? a.P : a.P / 2;
  const int par = BWD ? 0 : slice / Ps;
  const int row0 = (BWD ? slice : slice % Ps) * 8 * MB;
  const double sg = par ? -1.0 : 1.0;
  constexpr int NSET = BWD ? 2 : 1;
  double acc[NSET][NMB][2][2];
  double* ocol[2][2];
  for (int sidx = 0; sidx < nst; ++sidx) {
    const int ci = sidx / KS, kq = sidx - ci * KS;
    const int cb = c0 + ci * XF_NT;
    const int slot = sidx % NS, use = sidx / NS;
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
    mbar_wait(full + slot, static_cast<unsigned>(use & 1));
    const double* st = ring + static_cast<size_t>(slot) * STAGE;
    const double* Ap = (ARES ? Ares + static_cast<size_t>(kq) * ASTAGE : st) + (mb0 * 32 + lane) * 2;
    const double* Bp = st + AOFF + (nb * 8 + (lane >> 2)) * XK_BSTR + 2 * (lane & 3);
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
      const double* Bh = st + AOFF + XK_BSTAGE + (nb * 8 + (lane >> 2)) * XK_BSTR + 14 - 2 * (lane & 3);
      if (wide)
        xp_stage_fwd<MB, NMB, 2>(Ap, Bp, Bh, sg, acc[0]);
      else
        xp_stage_fwd<MB, NMB, 1>(Ap, Bp, Bh, sg, acc[0]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + slot);  // this warp is done reading the slot
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
}

// smem: ring[NS][A slab | B slab(s)] | full[NS] | empty[NS]
// NW consumer warpgroups split the slice's m-blocks NW ways (warp (s, hh): n-blocks s, s + 4, part hh):
// NW = 3 puts three DMMA-issuing warps on every scheduler, so one warp's fragment loads hide under
// the other two's MMAs (two left the fp64 tensor pipe idle 30 % of the time)
// ARES: the slice's whole matrix image (all K stages) is resident in shared memory after the ring
// (small w: C4's 176 x 88 per direction fits), the ring then carries the column slabs only
template <int MB, int NS, bool BWD, int NW, bool ARES = false>
__global__ void __launch_bounds__(128 * NW + 128, 1) xformq_kernel(XformPArgs pa) {
  pdl_wait();
  extern __shared__ __align__(128) double xq_smem[];
  const XformArgs& a = pa.x;
  constexpr int STAGE = (ARES ? 0 : xk_astage(MB)) + (BWD ? XK_BSTAGE : 2 * XK_BSTAGE);
  constexpr int NCW = 4 * NW;  // consumer warps
  double* ring = xq_smem;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xq_smem + static_cast<size_t>(NS) * STAGE);
  unsigned long long* empty = full + NS;
  const int t = threadIdx.x, warp = t >> 5;
  const int slice = blockIdx.x % a.P, grp = blockIdx.x / a.P, ngrp = gridDim.x / a.P;
  const int L = a.acount ? min(*a.acount, a.nslots) : a.nslots;
  const int cps = L * a.ncol_sys;
  const int ncols = cps * a.nv;
  const int share = ((ncols + ngrp - 1) / ngrp + 7) & ~7;
  const int c0 = grp * share, c1 = min(ncols, c0 + share);
  if (c0 >= c1) return;
  if (t == 0) {
    for (int s = 0; s < NS; ++s) {
      // 32 cp.async arrivals of the producer lanes (+ the bulk copy's expect_tx arrival)
      mbar_init(full + s, ARES ? 32 : 33);
      mbar_init(empty + s, NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int nstage = BWD ? 2 * pa.ks : pa.ks;
  const double* Aslice = a.Af + static_cast<size_t>(slice) * nstage * xk_astage(MB);
  double* Ares = reinterpret_cast<double*>(empty + NS);
  if (ARES) {
    const int pieces = nstage * xk_astage(MB) / 2;
    for (int e = t; e < pieces; e += blockDim.x) cp_async16(Ares + 2 * e, Aslice + 2 * e, true);
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();
  // register budget: the kernel is compiled for (128 NW + 128) threads; the producer's warpgroup
  // hands its registers to the consumers (setmaxnreg)
  if (warp >= NCW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == NCW) xq_producer<MB, NS, BWD, ARES>(pa, ring, full, empty, c0, c1, cps, Aslice);
  } else if (NW == 2) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    constexpr int MB0 = (MB + 1) / 2;
    if (warp < 4)
      xq_consumer<MB, MB0, NS, BWD, ARES>(pa, ring, full, empty, c0, c1, slice, 0, cps, Ares);
    else
      xq_consumer<MB, MB - MB0, NS, BWD, ARES>(pa, ring, full, empty, c0, c1, slice, MB0, cps, Ares);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;");
    constexpr int M0 = (MB + 2) / 3, M1 = (MB - M0 + 1) / 2, M2 = MB - M0 - M1;
    if (warp < 4)
      xq_consumer<MB, M0, NS, BWD, ARES>(pa, ring, full, empty, c0, c1, slice, 0, cps, Ares);
    else if (warp < 8)
      xq_consumer<MB, M1, NS, BWD, ARES>(pa, ring, full, empty, c0, c1, slice, M0, cps, Ares);
    else
      xq_consumer<MB, (M2 > 0 ? M2 : 1), NS, BWD, ARES>(pa, ring, full, empty, c0, c1, slice, M0 + M1, cps, Ares);
  }
  pdl_launch();
}

template <int MB, int NS, bool BWD>
constexpr size_t xformq_smem() {
  return xformp_smem<MB, NS, BWD>() + NS * sizeof(unsigned long long);
}
// resident-matrix variant: ring of column slabs, barriers, then nstage A slabs
template <int MB, int NS, bool BWD>
inline size_t xformq_ares_smem(int nstage) {
  return sizeof(double) * (static_cast<size_t>(NS) * (BWD ? XK_BSTAGE : 2 * XK_BSTAGE) +
                           static_cast<size_t>(nstage) * xk_astage(MB)) + 2 * NS * sizeof(unsigned long long);
}

}  // namespace smpm
