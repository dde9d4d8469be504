// Per-mode pass with 16 bytes per lane for every mode (sm_100a).
//
// spec_op2_kernel (spectral.cuh) gives each lane one eigenmode: a complex pair's
// two coordinates travel as one 16-byte load, but a real mode is an 8-byte load
// and drags a zero imaginary part through complex arithmetic and registers.  At
// C5 79 % of the modes are real and the pass ran at 0.21 of HBM, latency-bound
// with one block of loads in flight per warp.  Here a lane owns either one
// complex pair (as before) or TWO adjacent real modes packed in a double2 whose
// components multiply elementwise: every load and store is 16 bytes, real modes
// need half the warps, and the bytes in flight per SM double.  Same arithmetic
// per mode as spec_op2_kernel (spec_block_solve / spec_block_S): results are
// bit-identical for the pair modes; for the real modes the complex products with
// zero imaginary parts reduce to the same real products.
#pragma once

#include "spectral.cuh"

namespace smpm {

template <bool PAIR>
struct SpNum {
  static __device__ __forceinline__ double2 mul(double2 a, double2 b) {
    if (PAIR) return cmul(a, b);
    return make_double2(a.x * b.x, a.y * b.y);
  }
  static __device__ __forceinline__ double2 fma_(double2 a, double2 b, double2 c) {  // a * b + c
    if (PAIR) return cfma(a, b, c);
    return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
  }
  static __device__ __forceinline__ double2 ld(const double* p) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return PAIR ? make_double2(v.x, -v.y) : v;
  }
  static __device__ __forceinline__ void st(double* p, double2 z) {
    *reinterpret_cast<double2*>(p) = PAIR ? make_double2(z.x, -z.y) : z;
  }
  // per-mode complex coefficient array (gamma, kinv) at mode m: the pair's value, or the
  // real parts of the two real modes m, m + 1
  static __device__ __forceinline__ double2 coef(const double2* base, int m) {
    if (PAIR) return base[m];
    return make_double2(base[m].x, base[m + 1].x);
  }
  static __device__ __forceinline__ double zt(const double* om, double2 z) {  // omega . coordinates (om at e0)
    return PAIR ? fma(om[0], z.x, -om[1] * z.y) : fma(om[0], z.x, om[1] * z.y);
  }
};

template <bool PAIR>
struct Mode3 {
  long long base;  // system offset + e0
  int sys, w, e0, m;
  const double2 *gam, *kinv;  // system's arrays
  int nmode;
  double2 wee, a, b, c, e, eww;
  __device__ __forceinline__ double2 K(int idx) const { return SpNum<PAIR>::coef(kinv + static_cast<long long>(idx) * nmode, m); }
};

template <bool BJ, bool PAIR>
__device__ __forceinline__ void spec3_solve(const SpecParams& sp, const Mode3<PAIR>& M, int blk, const double2 (&y)[4],
                                            double2 (&x)[4]) {
  using N = SpNum<PAIR>;
  if (!BJ) {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = y[j];
  } else if (blk == sp.nbf) {
    const double2 h = sp.d >= 2 ? M.e : M.wee;
    x[0] = N::mul(csub(y[0], N::mul(M.eww, y[1])), M.K(16));
    x[1] = csub(y[1], N::mul(h, x[0]));
    x[2] = x[3] = make_double2(0.0, 0.0);
  } else {
    const bool first = blk == 0, last = 2 * blk + 2 > sp.mx - 2;
    const double2 ex = first ? M.wee : M.e;
    const double2 wx = last ? M.eww : M.a;
    const int kb = ((first ? 1 : 0) | (last ? 2 : 0)) * 4;
    const double2 r0 = csub(csub(y[0], N::mul(M.a, y[1])), N::mul(M.b, y[2]));
    const double2 r3 = csub(csub(y[3], N::mul(M.c, y[1])), N::mul(M.e, y[2]));
    x[0] = N::fma_(M.K(kb + 1), r3, N::mul(M.K(kb), r0));
    x[3] = N::fma_(M.K(kb + 2), r0, N::mul(M.K(kb + 3), r3));
    x[1] = csub(y[1], N::mul(ex, x[0]));
    x[2] = csub(y[2], N::mul(wx, x[3]));
  }
  if (sp.cadd) {
    // 2LAS: slot 4 blk + j of interface 2 blk + j / 2 gains c_i T^{-1} 1
    const int ns = spec_bslots(sp, blk);
    const double* c = sp.cadd + static_cast<long long>(M.sys) * sp.d;
    const double2 nu = make_double2(sp.nu[M.e0], PAIR ? -sp.nu[M.e0 + 1] : sp.nu[M.e0 + 1]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < ns) {
        const double ci = c[2 * blk + (j >> 1)];
        x[j] = make_double2(fma(ci, nu.x, x[j].x), fma(ci, nu.y, x[j].y));
      }
  }
}

template <bool PAIR>
__device__ __forceinline__ void spec3_S(const SpecParams& sp, const Mode3<PAIR>& M, int blk, const double2 (&x)[4],
                                        double2 xp3, double2 xn0, double2 (&t)[4]) {
  using N = SpNum<PAIR>;
  if (blk == sp.nbf) {
    t[0] = N::fma_(M.eww, x[1], x[0]);
    t[1] = sp.d >= 2 ? N::fma_(M.c, xp3, N::fma_(M.e, x[0], x[1])) : N::fma_(M.wee, x[0], x[1]);
    t[2] = t[3] = make_double2(0.0, 0.0);
    return;
  }
  t[0] = N::fma_(M.a, x[1], N::fma_(M.b, x[2], x[0]));
  t[1] = blk >= 1 ? N::fma_(M.c, xp3, N::fma_(M.e, x[0], x[1])) : N::fma_(M.wee, x[0], x[1]);
  t[2] = 2 * blk + 2 <= sp.mx - 2 ? N::fma_(M.a, x[3], N::fma_(M.b, xn0, x[2])) : N::fma_(M.eww, x[3], x[2]);
  t[3] = N::fma_(M.c, x[1], N::fma_(M.e, x[2], x[3]));
}

template <bool PAIR>
__device__ __forceinline__ void spec3_ld(const SpecParams& sp, const Mode3<PAIR>& M, const double* __restrict__ vh,
                                         int blk, bool ok, double2 (&y)[4]) {
  const int ns = ok ? spec_bslots(sp, blk) : 0;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    y[j] = j < ns ? SpNum<PAIR>::ld(vh + M.base + static_cast<long long>(4 * blk + j) * M.w) : make_double2(0.0, 0.0);
}

// one warp: 32 lane items (pairs, or pairs of real modes) x a segment of blocks [b0, b1);
// the pipelined walk of spec_warp_item2
template <bool BJ, bool PAIR>
__device__ __forceinline__ void spec_warp_item3(const SpecParams& sp, int s, int item0, int sg,
                                                const double* __restrict__ vh, double* __restrict__ th, double* zout,
                                                double* __restrict__ uh) {
  using N = SpNum<PAIR>;
  const int lane = threadIdx.x & 31;
  const int it = item0 + lane;
  const int nreal2 = (sp.nmode - sp.npairs) >> 1;
  const bool ok = PAIR ? it < sp.npairs : it < nreal2;
  const int nb = spec_nblocks(sp);
  const int b0 = sg * sp.segb, b1 = min(nb, b0 + sp.segb);
  Mode3<PAIR> M;
  M.sys = s;
  M.w = sp.w;
  M.m = ok ? (PAIR ? it : sp.npairs + 2 * it) : (PAIR ? 0 : sp.npairs);
  M.e0 = PAIR ? 2 * M.m : sp.npairs + M.m;
  M.base = s * sp.k + M.e0;
  M.nmode = sp.nmode;
  M.gam = sp.gam + static_cast<long long>(s) * SK_NUM * sp.nmode;
  M.kinv = sp.kinv + static_cast<long long>(s) * 20 * sp.nmode;
  M.wee = N::coef(M.gam + SK_W_EE * sp.nmode, M.m);
  M.a = N::coef(M.gam + SK_I_WW * sp.nmode, M.m);
  M.b = N::coef(M.gam + SK_I_WE * sp.nmode, M.m);
  M.c = N::coef(M.gam + SK_I_EW * sp.nmode, M.m);
  M.e = N::coef(M.gam + SK_I_EE * sp.nmode, M.m);
  M.eww = N::coef(M.gam + SK_E_WW * sp.nmode, M.m);
  double2 xp3, xc[4], xn[4], yc[4], yn[4];
  const bool halo = th && b0 > 0;
  {
    double2 y0[4], y1[4];
    spec3_ld(sp, M, vh, halo ? b0 - 1 : b0, ok, y0);
    spec3_ld(sp, M, vh, b0, ok && halo, y1);
    spec3_ld(sp, M, vh, b0 + 1, ok && b0 + 1 < nb && (th || b0 + 1 < b1), yc);
    if (halo) {
      double2 xq[4];
      spec3_solve<BJ>(sp, M, b0 - 1, y0, xq);
      xp3 = xq[3];
      spec3_solve<BJ>(sp, M, b0, y1, xc);
    } else {
      spec3_solve<BJ>(sp, M, b0, y0, xc);
      xp3 = make_double2(0.0, 0.0);
    }
  }
  for (int blk = b0; blk < b1; ++blk) {
    const int ns = spec_bslots(sp, blk);
    const bool need_next = blk + 1 < nb && (th || blk + 1 < b1);
    const bool need_nn = blk + 2 < nb && (th ? blk + 2 <= b1 : blk + 2 < b1);
    spec3_ld(sp, M, vh, blk + 2, ok && need_nn, yn);
    if (uh && ok) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < ns) N::st(uh + M.base + static_cast<long long>(4 * blk + j) * M.w, xc[j]);
    }
    if (need_next) spec3_solve<BJ>(sp, M, blk + 1, yc, xn);
    if (th) {
      double2 t[4];
      spec3_S(sp, M, blk, xc, xp3, xn[0], t);
      if (ok) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < ns) N::st(th + M.base + static_cast<long long>(4 * blk + j) * M.w, t[j]);
      }
      if (zout) {
        const double z0 = ok ? N::zt(sp.omega + M.e0, cadd(t[0], t[1])) : 0.0;
        const double z1 = ok && ns == 4 ? N::zt(sp.omega + M.e0, cadd(t[2], t[3])) : 0.0;
        const double r0 = warp_sum(z0);
        const double r1 = warp_sum(z1);
        if (lane == 0) {
          zout[2 * blk] = r0;
          if (2 * blk + 1 < sp.d) zout[2 * blk + 1] = r1;
        }
      }
    }
    xp3 = xc[3];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xc[j] = xn[j];
      yc[j] = yn[j];
    }
  }
}

// lane-item chunks of 32: pair chunks first, then real-pair chunks
__host__ __device__ __forceinline__ int spec3_pair_chunks(int npairs) { return (npairs + 31) / 32; }
__host__ __device__ __forceinline__ int spec3_chunks(int npairs, int nmode) {
  return spec3_pair_chunks(npairs) + (((nmode - npairs) >> 1) + 31) / 32;
}

// grid (chunks * ceil(nseg / SP_WARPS), live slots); zpart: nsys x chunks x d; cout: the coarse
// solutions c = C^{-1} Z^T t, or (sums_only) the coarse right-hand sides Z^T t
template <bool BJ>
__global__ void __launch_bounds__(SP_THREADS, 4) spec_op3_kernel(SpecParams sp, const double* __restrict__ vh,
                                                              double* __restrict__ th, DeflateParams P, double* zpart,
                                                              int* counter, double* cout, double* __restrict__ uh,
                                                              int sums_only) {
  pdl_wait();
  extern __shared__ double sm3[];  // 2 d doubles (coarse solve)
  int s;
  if (!defl_slot(P, blockIdx.y, s)) return;
  const int npc = spec3_pair_chunks(sp.npairs), nch = spec3_chunks(sp.npairs, sp.nmode);
  const int nsg = (sp.nseg + SP_WARPS - 1) / SP_WARPS;
  const int mc = blockIdx.x / nsg, sg = (blockIdx.x % nsg) * SP_WARPS + (threadIdx.x >> 5);
  if (sg < sp.nseg) {
    double* zo = zpart ? zpart + (static_cast<long long>(s) * nch + mc) * sp.d : nullptr;
    if (mc < npc)
      spec_warp_item3<BJ, true>(sp, s, mc * 32, sg, vh, th, zo, uh);
    else
      spec_warp_item3<BJ, false>(sp, s, (mc - npc) * 32, sg, vh, th, zo, uh);
  }
  pdl_launch();  // dependents may start launching: this CTA's main work is done
  if (!zpart) return;
  if (!last_cta(counter + s, nch * nsg)) return;
  double* sums = sm3;
  double* c = sm3 + sp.d;
  for (int i = threadIdx.x; i < sp.d; i += blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < nch; ++q) v += __ldcg(zpart + (static_cast<long long>(s) * nch + q) * sp.d + i);
    sums[i] = v;
    // sums_only: the coarse right-hand side goes out as it is; the (serial) coarse solve runs in
    // zt_coarse_kernel on a side stream beside the T transform (spec_SMinv)
    if (sums_only) cout[static_cast<long long>(s) * sp.d + i] = v;
  }
  if (sums_only) return;
  __syncthreads();
  coarse_solve_block(P, s, sums, c);
  for (int i = threadIdx.x; i < sp.d; i += blockDim.x) cout[static_cast<long long>(s) * sp.d + i] = c[i];
}

}  // namespace smpm
