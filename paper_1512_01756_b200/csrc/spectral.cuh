// Spectral form of the Schur operator and its block-Jacobi preconditioner.
//
// Every coupling block of the SMPM Schur complement is the trace of the same
// separable strip solve, so all of them share the z eigenbasis of the strip
// operator: G_kind[X,Y](mu) = Vz diag(gamma_kind,XY(mu)) Vz^{-1}
// (fast diagonalisation of (A - mu), the A^{-1}B sweep of the north star).
// The eigenpairs are real or complex-conjugate; with the real basis
//   T = [Re v_q, Im v_q (complex pairs, first) | v_q (real modes)]
// every w-block of an interface vector maps to T^{-1} v, where a pair's two
// coordinates (a, b) act as one complex number z = a - i b and each G block
// is multiplication by gamma_q.  So
//   S M^{-1} v = T [ S^ M^^{-1} ] T^{-1} v
// with T^{-1}, T two GEMMs whose matrix (w x w) is shared by every system,
// interface and mode, and S^, M^^{-1} independent per eigenmode: S^ couples
// the 2d interface slots of one mode like the dense blocks couple w-blocks
// (SURVEY App. A), and each block-Jacobi block (two interfaces, four slots;
// /root/reference/proj/src/schur.cpp:188-225) is a 4x4 per mode, solved
// through its 2x2 reduced system K = I - G' diag(Gee, Gww) in closed form.
// The Z^T interface sums of the deflation are weighted sums of the
// transformed coordinates (weights omega = T^T 1), so the coarse right-hand
// side comes out of the same pass.
#pragma once

#include "common.cuh"
#include "vec.cuh"

namespace smpm {

// gamma kinds per system and mode (complex, (re, im))
enum SpecKind : int { SK_W_EE = 0, SK_I_WW = 1, SK_I_WE = 2, SK_I_EW = 3, SK_I_EE = 4, SK_E_WW = 5, SK_NUM = 6 };

struct SpecParams {
  int w, d, mx, nbf, single;  // geometry (nbf full two-interface blocks, single trailing block)
  int npairs, nmode;           // complex-pair modes first, then real modes; nmode = w - npairs
  long long k;                 // 2 d w
  const double2* gam;          // nsys x SK_NUM x nmode
  const double* omega;         // w: column sums of T (Z^T weights)
  int nmc, nseg;               // mode chunks, block segments (grid x = nmc * nseg)
};

constexpr int SP_THREADS = 128;  // modes per CTA
constexpr int SP_SEGB = 4;       // block-Jacobi blocks per segment (8 interfaces)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = fma(b.x, b.x, b.y * b.y);
  return make_double2(fma(a.x, b.x, a.y * b.y) / den, fma(a.y, b.x, -a.x * b.y) / den);
}

// one mode's view of a system's transformed vector: slot beta lives at
// base + beta*w + e0 (and e0 + 1 for the second coordinate of a pair)
struct ModeRef {
  long long base;
  int w, e0;
  bool pair;
  __device__ __forceinline__ double2 ld(const double* v, int beta) const {
    const double* p = v + base + static_cast<long long>(beta) * w + e0;
    return make_double2(__ldcg(p), pair ? -__ldcg(p + 1) : 0.0);
  }
  __device__ __forceinline__ void st(double* v, int beta, double2 z) const {
    double* p = v + base + static_cast<long long>(beta) * w + e0;
    p[0] = z.x;
    if (pair) p[1] = -z.y;
  }
  __device__ __forceinline__ double zt(const double* omega, double2 z) const {  // omega . coordinates
    return pair ? fma(omega[e0], z.x, -omega[e0 + 1] * z.y) : omega[e0] * z.x;
  }
};

__device__ __forceinline__ ModeRef mode_ref(const SpecParams& sp, int s, int m) {
  ModeRef r;
  r.base = s * sp.k;
  r.w = sp.w;
  r.pair = m < sp.npairs;
  r.e0 = r.pair ? 2 * m : sp.npairs + m;
  return r;
}

struct ModeGamma {
  double2 wee, a, b, c, e, eww;  // W_EE, I_WW, I_WE, I_EW, I_EE, E_WW
};

__device__ __forceinline__ ModeGamma mode_gamma(const SpecParams& sp, int s, int m) {
  const double2* g = sp.gam + static_cast<long long>(s) * SK_NUM * sp.nmode + m;
  ModeGamma G;
  G.wee = g[SK_W_EE * sp.nmode];
  G.a = g[SK_I_WW * sp.nmode];
  G.b = g[SK_I_WE * sp.nmode];
  G.c = g[SK_I_EW * sp.nmode];
  G.e = g[SK_I_EE * sp.nmode];
  G.eww = g[SK_E_WW * sp.nmode];
  return G;
}

// x = M_blk^{-1} y for block blk of one mode (4 slots, or 2 for the trailing
// single block); without BJ x = y
template <bool BJ>
__device__ __forceinline__ void spec_block_solve(const SpecParams& sp, const ModeGamma& g, int blk, const double2 (&y)[4],
                                                 double2 (&x)[4]) {
  if (!BJ) {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = y[j];
    return;
  }
  const double2 one = make_double2(1.0, 0.0);
  if (blk == sp.nbf) {
    // trailing interface d-1 alone: y0 = x0 + G_E x1 ; y1 = Gee x0 + x1
    const double2 h = sp.d >= 2 ? g.e : g.wee;
    x[0] = cdiv(csub(y[0], cmul(g.eww, y[1])), csub(one, cmul(g.eww, h)));
    x[1] = csub(y[1], cmul(h, x[0]));
    x[2] = x[3] = make_double2(0.0, 0.0);
    return;
  }
  // y0 = x0 + a x1 + b x2 ; y1 = ex x0 + x1 ; y2 = x2 + wx x3 ; y3 = c x1 + e x2 + x3
  const double2 ex = blk == 0 ? g.wee : g.e;
  const double2 wx = 2 * blk + 2 <= sp.mx - 2 ? g.a : g.eww;
  const double2 r0 = csub(csub(y[0], cmul(g.a, y[1])), cmul(g.b, y[2]));
  const double2 r3 = csub(csub(y[3], cmul(g.c, y[1])), cmul(g.e, y[2]));
  const double2 k00 = csub(one, cmul(g.a, ex)), k11 = csub(one, cmul(g.e, wx));
  const double2 k01 = cmul(g.b, wx), k10 = cmul(g.c, ex);  // K = [[k00, -k01], [-k10, k11]]
  const double2 det = csub(cmul(k00, k11), cmul(k01, k10));
  x[0] = cdiv(cfma(k01, r3, cmul(k11, r0)), det);
  x[3] = cdiv(cfma(k10, r0, cmul(k00, r3)), det);
  x[1] = csub(y[1], cmul(ex, x[0]));
  x[2] = csub(y[2], cmul(wx, x[3]));
}

// t^ = S^ x^ for block blk of one mode, given the block's x, the previous
// block's last slot (xp3) and the next block's first slot (xn0)
__device__ __forceinline__ void spec_block_S(const SpecParams& sp, const ModeGamma& g, int blk, const double2 (&x)[4],
                                             double2 xp3, double2 xn0, double2 (&t)[4]) {
  if (blk == sp.nbf) {
    // interface d-1: left slot reads strip m_x-1 (E boundary), right slot strip d-1
    t[0] = cfma(g.eww, x[1], x[0]);
    t[1] = sp.d >= 2 ? cfma(g.c, xp3, cfma(g.e, x[0], x[1])) : cfma(g.wee, x[0], x[1]);
    t[2] = t[3] = make_double2(0.0, 0.0);
    return;
  }
  t[0] = cfma(g.a, x[1], cfma(g.b, x[2], x[0]));
  t[1] = blk >= 1 ? cfma(g.c, xp3, cfma(g.e, x[0], x[1])) : cfma(g.wee, x[0], x[1]);
  t[2] = 2 * blk + 2 <= sp.mx - 2 ? cfma(g.a, x[3], cfma(g.b, xn0, x[2])) : cfma(g.eww, x[3], x[2]);
  t[3] = cfma(g.c, x[1], cfma(g.e, x[2], x[3]));
}

__device__ __forceinline__ int spec_nblocks(const SpecParams& sp) { return sp.nbf + (sp.single ? 1 : 0); }
__device__ __forceinline__ int spec_bslots(const SpecParams& sp, int blk) { return blk == sp.nbf ? 2 : 4; }

template <bool BJ>
__device__ __forceinline__ void spec_load_solve(const SpecParams& sp, const ModeRef& mr, const ModeGamma& g,
                                                const double* vh, int blk, double2 (&x)[4]) {
  double2 y[4];
  const int ns = spec_bslots(sp, blk);
#pragma unroll
  for (int j = 0; j < 4; ++j) y[j] = j < ns ? mr.ld(vh, 4 * blk + j) : make_double2(0.0, 0.0);
  spec_block_solve<BJ>(sp, g, blk, y, x);
}

// One mode, block-Jacobi blocks [b0, b1): th = S^ M^^{-1} vh (or S^ vh), and
// the Z^T partial sums of th for the interfaces of those blocks -> zt[0..)
// (zt indexed from interface 2*b0; nullptr: skipped)
template <bool BJ>
__device__ __forceinline__ void spec_mode_segment(const SpecParams& sp, const ModeRef& mr, const ModeGamma& g,
                                                  const double* vh, double* th, int b0, int b1, double* zt) {
  const int nb = spec_nblocks(sp);
  double2 xp[4], xc[4], xn[4];
  if (b0 > 0) spec_load_solve<BJ>(sp, mr, g, vh, b0 - 1, xp);
  spec_load_solve<BJ>(sp, mr, g, vh, b0, xc);
  for (int blk = b0; blk < b1; ++blk) {
    if (blk + 1 < nb) spec_load_solve<BJ>(sp, mr, g, vh, blk + 1, xn);
    double2 t[4];
    spec_block_S(sp, g, blk, xc, xp[3], xn[0], t);
    const int ns = spec_bslots(sp, blk);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < ns) mr.st(th, 4 * blk + j, t[j]);
    if (zt) {
      zt[2 * (blk - b0)] = mr.zt(sp.omega, cadd(t[0], t[1]));
      if (ns == 4) zt[2 * (blk - b0) + 1] = mr.zt(sp.omega, cadd(t[2], t[3]));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xp[j] = xc[j];
      xc[j] = xn[j];
    }
  }
}

// th = T^-1-space operator of the live systems; with zpart, the last CTA of
// each system also solves the coarse system for c = C^{-1} Z^T (T th) -> cout
template <bool BJ>
__global__ void __launch_bounds__(SP_THREADS) spec_op_kernel(SpecParams sp, const double* vh, double* th,
                                                             DeflateParams P, double* zpart, int* counter,
                                                             double* cout) {
  extern __shared__ double sm[];  // 2 d doubles (coarse solve)
  __shared__ double zs[SP_THREADS / 32][2 * SP_SEGB];
  int s;
  if (!defl_slot(P, blockIdx.y, s)) return;
  const int mc = blockIdx.x / sp.nseg, sg = blockIdx.x % sp.nseg;
  const int m = mc * SP_THREADS + threadIdx.x;
  const int nb = spec_nblocks(sp);
  const int b0 = sg * SP_SEGB, b1 = min(nb, b0 + SP_SEGB);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double zt[2 * SP_SEGB];
#pragma unroll
  for (int i = 0; i < 2 * SP_SEGB; ++i) zt[i] = 0.0;
  if (m < sp.nmode) {
    const ModeRef mr = mode_ref(sp, s, m);
    const ModeGamma g = mode_gamma(sp, s, m);
    spec_mode_segment<BJ>(sp, mr, g, vh, th, b0, b1, zpart ? zt : nullptr);
  }
  if (!zpart) return;
  // Z^T partials of this CTA's modes for its interfaces, fixed-order reductions
  const int i0 = 2 * b0, i1 = min(sp.d, 2 * b1);
#pragma unroll
  for (int i = 0; i < 2 * SP_SEGB; ++i) {
    const double v = warp_sum(zt[i]);
    if (lane == 0) zs[warp][i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < i1 - i0; i += blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < SP_THREADS / 32; ++q) v += zs[q][i];
    zpart[(static_cast<long long>(s) * sp.nmc + mc) * sp.d + i0 + i] = v;
  }
  if (!last_cta(counter + s, sp.nmc * sp.nseg)) return;
  double* sums = sm;
  double* c = sm + sp.d;
  for (int i = threadIdx.x; i < sp.d; i += blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < sp.nmc; ++q) v += __ldcg(zpart + (static_cast<long long>(s) * sp.nmc + q) * sp.d + i);
    sums[i] = v;
  }
  __syncthreads();
  coarse_solve_block(P, s, sums, c);
  for (int i = threadIdx.x; i < sp.d; i += blockDim.x) cout[static_cast<long long>(s) * sp.d + i] = c[i];
}

}  // namespace smpm
