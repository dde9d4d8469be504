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
  const double2* kinv;         // nsys x 5 x 4 x nmode: reduced block inverses (variants first|last<<1, 4 = single)
  const double* omega;         // w: column sums of T (Z^T weights)
  const double* nu;            // w: T^{-1} 1, a constant w-block in spectral coordinates
  const double* cadd;          // nullable, nsys x d: 2LAS coarse solutions c added as Z c before S^
  int nmc, nseg, segb;         // 32-mode chunks, block segments of segb (<= SP_SEGB) blocks
  int stage;                   // spec_op_kernel: stage each warp's vh rows in shared memory first
};

constexpr int SP_MODES = 32;               // modes per warp (one lane each)
constexpr int SP_WARPS = 4;                // segments per CTA (one warp each)
constexpr int SP_THREADS = 32 * SP_WARPS;
constexpr int SP_SEGB = 4;                 // max block-Jacobi blocks per segment (8 interfaces)
constexpr int SP_SROW = 66;                // staged doubles per slot row (32 modes, pairs take 2; 16-byte aligned start)
constexpr int SP_SSLOTS = 4 * (SP_SEGB + 2);  // slot rows per warp: the segment and its two halo blocks
constexpr int SP_STAGE_DOUBLES = SP_WARPS * SP_SSLOTS * SP_SROW;  // 48 KB per CTA

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
  int sys, w, e0;
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

// shared-memory copy of one warp's slot rows: slot row (blk - bs) * 4 + j holds
// coordinates [elo, elo + SP_SROW) of slot 4 blk + j
struct SpecStage {
  const double* buf;  // nullptr: read vh directly
  int bs, elo;
};

__device__ __forceinline__ double2 spec_ld(const ModeRef& mr, const SpecStage& sg, const double* vh, int beta) {
  if (!sg.buf) return mr.ld(vh, beta);
  const double* p = sg.buf + ((beta >> 2) - sg.bs) * 4 * SP_SROW + (beta & 3) * SP_SROW + (mr.e0 - sg.elo);
  return make_double2(p[0], mr.pair ? -p[1] : 0.0);
}

__device__ __forceinline__ ModeRef mode_ref(const SpecParams& sp, int s, int m) {
  ModeRef r;
  r.sys = s;
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

// reduced-system inverses of one mode (setup): K = I - G' diag(ex, wx) with
// G' = [[a, b], [c, e]]; variant v = first | last << 1 picks ex = W_EE | I_EE
// and wx = E_WW | I_WW; variant 4 is the trailing single interface
__global__ void spec_setup_kernel(SpecParams sp, double2* kinv, int nsys) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(nsys) * sp.nmode) return;
  const int s = static_cast<int>(idx / sp.nmode), m = static_cast<int>(idx % sp.nmode);
  const double2* g = sp.gam + static_cast<long long>(s) * SK_NUM * sp.nmode + m;
  const double2 wee = g[SK_W_EE * sp.nmode], ga = g[SK_I_WW * sp.nmode], gb = g[SK_I_WE * sp.nmode];
  const double2 gc = g[SK_I_EW * sp.nmode], ge = g[SK_I_EE * sp.nmode], eww = g[SK_E_WW * sp.nmode];
  const double2 one = make_double2(1.0, 0.0);
  double2* out = kinv + static_cast<long long>(s) * 5 * 4 * sp.nmode + m;
  for (int v = 0; v < 4; ++v) {
    const double2 ex = (v & 1) ? wee : ge, wx = (v & 2) ? eww : ga;
    const double2 k00 = csub(one, cmul(ga, ex)), k11 = csub(one, cmul(ge, wx));
    const double2 k01 = cmul(gb, wx), k10 = cmul(gc, ex);  // K = [[k00, -k01], [-k10, k11]]
    const double2 det = csub(cmul(k00, k11), cmul(k01, k10));
    out[(v * 4 + 0) * sp.nmode] = cdiv(k11, det);
    out[(v * 4 + 1) * sp.nmode] = cdiv(k01, det);
    out[(v * 4 + 2) * sp.nmode] = cdiv(k10, det);
    out[(v * 4 + 3) * sp.nmode] = cdiv(k00, det);
  }
  const double2 h = sp.d >= 2 ? ge : wee;
  out[16 * sp.nmode] = cdiv(one, csub(one, cmul(eww, h)));
  out[17 * sp.nmode] = out[18 * sp.nmode] = out[19 * sp.nmode] = make_double2(0.0, 0.0);
}

// x = M_blk^{-1} y for block blk of one mode (4 slots, or 2 for the trailing
// single block); without BJ x = y
template <bool BJ>
__device__ __forceinline__ void spec_block_solve(const SpecParams& sp, const ModeGamma& g, const double2* ki, int blk,
                                                 const double2 (&y)[4], double2 (&x)[4]) {
  if (!BJ) {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = y[j];
    return;
  }
  const int nm = sp.nmode;
  if (blk == sp.nbf) {
    // trailing interface d-1 alone: y0 = x0 + G_E x1 ; y1 = Gee x0 + x1
    const double2 h = sp.d >= 2 ? g.e : g.wee;
    x[0] = cmul(csub(y[0], cmul(g.eww, y[1])), ki[16 * nm]);
    x[1] = csub(y[1], cmul(h, x[0]));
    x[2] = x[3] = make_double2(0.0, 0.0);
    return;
  }
  // y0 = x0 + a x1 + b x2 ; y1 = ex x0 + x1 ; y2 = x2 + wx x3 ; y3 = c x1 + e x2 + x3
  const bool first = blk == 0, last = 2 * blk + 2 > sp.mx - 2;
  const double2 ex = first ? g.wee : g.e;
  const double2 wx = last ? g.eww : g.a;
  const double2* k = ki + ((first ? 1 : 0) | (last ? 2 : 0)) * 4 * nm;
  const double2 r0 = csub(csub(y[0], cmul(g.a, y[1])), cmul(g.b, y[2]));
  const double2 r3 = csub(csub(y[3], cmul(g.c, y[1])), cmul(g.e, y[2]));
  x[0] = cfma(k[nm], r3, cmul(k[0], r0));
  x[3] = cfma(k[2 * nm], r0, cmul(k[3 * nm], r3));
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
                                                const double2* ki, const double* __restrict__ vh, int blk,
                                                double2 (&x)[4], double ysc, const SpecStage& stg) {
  double2 y[4];
  const int ns = spec_bslots(sp, blk);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    y[j] = j < ns ? spec_ld(mr, stg, vh, 4 * blk + j) : make_double2(0.0, 0.0);
    y[j].x *= ysc;
    y[j].y *= ysc;
  }
  spec_block_solve<BJ>(sp, g, ki, blk, y, x);
  if (sp.cadd) {
    // 2LAS: (M^{-1} + Z C^{-1} Z^T) v in spectral coordinates: slot 4 blk + j of
    // interface 2 blk + j / 2 gains c_i T^{-1} 1 (proj/src/deflation.cpp:127-130)
    const double* c = sp.cadd + static_cast<long long>(mr.sys) * sp.d;
    const double2 nu = make_double2(sp.nu[mr.e0], mr.pair ? -sp.nu[mr.e0 + 1] : 0.0);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < ns) {
        const double ci = c[2 * blk + (j >> 1)];
        x[j] = make_double2(fma(ci, nu.x, x[j].x), fma(ci, nu.y, x[j].y));
      }
  }
}

// One mode, block-Jacobi blocks [b0, b1): th = S^ M^^{-1} vh (or S^ vh), and
// the Z^T partial sums of th for the interfaces of those blocks -> zt[0..)
// (zt indexed from interface 2*b0; nullptr: skipped).  uh (nullable) also
// receives M^^{-1} vh; th may be nullptr when only that is wanted.
template <bool BJ>
__device__ __forceinline__ void spec_mode_segment(const SpecParams& sp, const ModeRef& mr, const ModeGamma& g,
                                                  const double2* ki, const double* __restrict__ vh,
                                                  double* __restrict__ th, int b0, int b1, double* zt,
                                                  double* __restrict__ uh, double ysc, const SpecStage& stg) {
  const int nb = spec_nblocks(sp);
  double2 xp[4], xc[4], xn[4];
  if (th && b0 > 0) spec_load_solve<BJ>(sp, mr, g, ki, vh, b0 - 1, xp, ysc, stg);
  spec_load_solve<BJ>(sp, mr, g, ki, vh, b0, xc, ysc, stg);
  for (int blk = b0; blk < b1; ++blk) {
    const int ns = spec_bslots(sp, blk);
    if (uh) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < ns) mr.st(uh, 4 * blk + j, xc[j]);
    }
    if (th) {
      if (blk + 1 < nb) spec_load_solve<BJ>(sp, mr, g, ki, vh, blk + 1, xn, ysc, stg);
      double2 t[4];
      spec_block_S(sp, g, blk, xc, xp[3], xn[0], t);
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
    } else if (blk + 1 < b1) {
      spec_load_solve<BJ>(sp, mr, g, ki, vh, blk + 1, xc, ysc, stg);
    }
  }
}

// One warp = one segment of 32 modes of one system: th for its blocks and,
// with zout, the warp-reduced Z^T partials of its interfaces -> zout[i]
template <bool BJ>
__device__ __forceinline__ void spec_warp_item(const SpecParams& sp, int s, int mc, int sg,
                                               const double* __restrict__ vh, double* __restrict__ th, double* zout,
                                               double* __restrict__ uh = nullptr, double ysc = 1.0,
                                               double* sbuf = nullptr) {
  const int lane = threadIdx.x & 31;
  const int m = mc * SP_MODES + lane;
  const int nb = spec_nblocks(sp);
  const int b0 = sg * sp.segb, b1 = min(nb, b0 + sp.segb);
  SpecStage stg{nullptr, 0, 0};
  if (sbuf) {
    // the warp's slot rows (segment + halo blocks) into shared memory with 8-byte async
    // copies issued together, so the per-block chain below reads shared memory only
    const int bs = (th && b0 > 0) ? b0 - 1 : b0, be = th ? min(nb, b1 + 1) : b1;
    const int mf = mc * SP_MODES, ml = min(sp.nmode, mf + SP_MODES) - 1;
    // 16-byte copies of the even-aligned range (k and w even), through L2 (.cg)
    const int elo = (mf < sp.npairs ? 2 * mf : sp.npairs + mf) & ~1;
    const int ehi = ml < sp.npairs ? 2 * ml + 2 : sp.npairs + ml + 1;
    const int npr = (ehi - elo + 1) >> 1;  // <= 33 pairs
    const double* src0 = vh + s * sp.k + elo;
    for (int bl = bs; bl < be; ++bl) {
      const int ns = spec_bslots(sp, bl);
      for (int jj = 0; jj < ns; ++jj) {
        const double* src = src0 + static_cast<long long>(4 * bl + jj) * sp.w;
        double* dst = sbuf + ((bl - bs) * 4 + jj) * SP_SROW;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = lane + 32 * h;
          if (e < npr) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + 2 * e));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + 2 * e));
          }
        }
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    stg = SpecStage{sbuf, bs, elo};
  }
  double zt[2 * SP_SEGB];
#pragma unroll
  for (int i = 0; i < 2 * SP_SEGB; ++i) zt[i] = 0.0;
  if (m < sp.nmode) {
    const ModeRef mr = mode_ref(sp, s, m);
    const ModeGamma g = mode_gamma(sp, s, m);
    const double2* ki = sp.kinv + static_cast<long long>(s) * 20 * sp.nmode + m;
    spec_mode_segment<BJ>(sp, mr, g, ki, vh, th, b0, b1, zout ? zt : nullptr, uh, ysc, stg);
  }
  if (!zout) return;
  const int i0 = 2 * b0, i1 = min(sp.d, 2 * b1);
#pragma unroll
  for (int i = 0; i < 2 * SP_SEGB; ++i) {
    const double v = warp_sum(zt[i]);
    if (lane == 0 && i0 + i < i1) zout[i0 + i] = v;
  }
}

// ---- pipelined per-mode pass (per-stage path) ------------------------------
// One warp = (system, 32-mode chunk, segment of segb blocks); lane = mode.  The
// warp walks its blocks in order with the raw slot values of the next block
// already in registers and the block after it in flight (16-byte loads for a
// pair mode's two coordinates), so each block's solve overlaps two blocks of
// loads; no shared memory, so many warps per SM.  Long segments keep the halo
// (one block on each side) small.  The Z^T partial of each interface is
// warp-reduced as its block completes.  Same per-mode arithmetic as
// spec_mode_segment (bit-identical th / uh / Z^T partials).
__device__ __forceinline__ void spec_ld_raw(const SpecParams& sp, const ModeRef& mr, const double* __restrict__ vh,
                                            int blk, bool ok, double2 (&y)[4]) {
  const int ns = ok ? spec_bslots(sp, blk) : 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j < ns) {
      const double* p = vh + mr.base + static_cast<long long>(4 * blk + j) * mr.w + mr.e0;
      if (mr.pair) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
        y[j] = make_double2(v.x, -v.y);
      } else {
        y[j] = make_double2(__ldcg(p), 0.0);
      }
    } else {
      y[j] = make_double2(0.0, 0.0);
    }
  }
}

template <bool BJ>
__device__ __forceinline__ void spec_solve_raw(const SpecParams& sp, const ModeRef& mr, const ModeGamma& g,
                                               const double2* ki, int blk, const double2 (&y)[4], double2 (&x)[4]) {
  spec_block_solve<BJ>(sp, g, ki, blk, y, x);
  if (sp.cadd) {
    const int ns = spec_bslots(sp, blk);
    const double* c = sp.cadd + static_cast<long long>(mr.sys) * sp.d;
    const double2 nu = make_double2(sp.nu[mr.e0], mr.pair ? -sp.nu[mr.e0 + 1] : 0.0);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < ns) {
        const double ci = c[2 * blk + (j >> 1)];
        x[j] = make_double2(fma(ci, nu.x, x[j].x), fma(ci, nu.y, x[j].y));
      }
  }
}

__device__ __forceinline__ void spec_st_pair(const ModeRef& mr, double* v, int beta, double2 z) {
  double* p = v + mr.base + static_cast<long long>(beta) * mr.w + mr.e0;
  if (mr.pair)
    *reinterpret_cast<double2*>(p) = make_double2(z.x, -z.y);
  else
    p[0] = z.x;
}

template <bool BJ>
__device__ __forceinline__ void spec_warp_item2(const SpecParams& sp, int s, int mc, int sg, const double* __restrict__ vh,
                                                double* __restrict__ th, double* zout, double* __restrict__ uh) {
  const int lane = threadIdx.x & 31;
  const int m = mc * SP_MODES + lane;
  const int nb = spec_nblocks(sp);
  const int b0 = sg * sp.segb, b1 = min(nb, b0 + sp.segb);
  const bool ok = m < sp.nmode;
  const ModeRef mr = mode_ref(sp, s, ok ? m : 0);
  ModeGamma g{};
  if (ok) g = mode_gamma(sp, s, m);
  const double2* ki = sp.kinv + static_cast<long long>(s) * 20 * sp.nmode + (ok ? m : 0);
  // raw values: yc (block blk + 1, landed), yn (block blk + 2, in flight)
  double2 xp[4], xc[4], xn[4], yc[4], yn[4];
  const bool halo = th && b0 > 0;
  {
    double2 y0[4], y1[4];
    spec_ld_raw(sp, mr, vh, halo ? b0 - 1 : b0, ok, y0);
    spec_ld_raw(sp, mr, vh, b0, ok && halo, y1);
    spec_ld_raw(sp, mr, vh, b0 + 1, ok && b0 + 1 < nb && (th || b0 + 1 < b1), yc);
    if (halo) {
      spec_solve_raw<BJ>(sp, mr, g, ki, b0 - 1, y0, xp);
      spec_solve_raw<BJ>(sp, mr, g, ki, b0, y1, xc);
    } else {
      spec_solve_raw<BJ>(sp, mr, g, ki, b0, y0, xc);
#pragma unroll
      for (int j = 0; j < 4; ++j) xp[j] = make_double2(0.0, 0.0);
    }
  }
  // yc now holds block b0 + 1
  for (int blk = b0; blk < b1; ++blk) {
    const int ns = spec_bslots(sp, blk);
    const bool need_next = blk + 1 < nb && (th || blk + 1 < b1);
    const bool need_nn = blk + 2 < nb && (th ? blk + 2 <= b1 : blk + 2 < b1);
    spec_ld_raw(sp, mr, vh, blk + 2, ok && need_nn, yn);
    if (uh && ok) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < ns) spec_st_pair(mr, uh, 4 * blk + j, xc[j]);
    }
    if (need_next) spec_solve_raw<BJ>(sp, mr, g, ki, blk + 1, yc, xn);
    if (th) {
      double2 t[4];
      spec_block_S(sp, g, blk, xc, xp[3], xn[0], t);
      if (ok) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < ns) spec_st_pair(mr, th, 4 * blk + j, t[j]);
      }
      if (zout) {
        const double z0 = ok ? mr.zt(sp.omega, cadd(t[0], t[1])) : 0.0;
        const double z1 = ok && ns == 4 ? mr.zt(sp.omega, cadd(t[2], t[3])) : 0.0;
        const double r0 = warp_sum(z0);
        const double r1 = warp_sum(z1);
        if (lane == 0) {
          zout[2 * blk] = r0;
          if (2 * blk + 1 < sp.d) zout[2 * blk + 1] = r1;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xp[j] = xc[j];
      xc[j] = xn[j];
      yc[j] = yn[j];
    }
  }
}

// per-stage per-mode pass: grid (nmc * ceil(nseg / SP_WARPS), live slots)
template <bool BJ>
__global__ void __launch_bounds__(SP_THREADS, 4) spec_op2_kernel(SpecParams sp, const double* __restrict__ vh,
                                                              double* __restrict__ th, DeflateParams P, double* zpart,
                                                              int* counter, double* cout, double* __restrict__ uh) {
  pdl_wait();
  extern __shared__ double sm2[];  // 2 d doubles (coarse solve)
  int s;
  if (!defl_slot(P, blockIdx.y, s)) return;
  const int nsg = (sp.nseg + SP_WARPS - 1) / SP_WARPS;
  const int mc = blockIdx.x / nsg, sg = (blockIdx.x % nsg) * SP_WARPS + (threadIdx.x >> 5);
  if (sg < sp.nseg)
    spec_warp_item2<BJ>(sp, s, mc, sg, vh, th, zpart ? zpart + (static_cast<long long>(s) * sp.nmc + mc) * sp.d : nullptr,
                        uh);
  pdl_launch();  // dependents may start launching: this CTA's main work is done
  if (!zpart) return;
  if (!last_cta(counter + s, sp.nmc * nsg)) return;
  double* sums = sm2;
  double* c = sm2 + sp.d;
  for (int i = threadIdx.x; i < sp.d; i += blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < sp.nmc; ++q) v += __ldcg(zpart + (static_cast<long long>(s) * sp.nmc + q) * sp.d + i);
    sums[i] = v;
  }
  __syncthreads();
  coarse_solve_block(P, s, sums, c);
  for (int i = threadIdx.x; i < sp.d; i += blockDim.x) cout[static_cast<long long>(s) * sp.d + i] = c[i];
}

// th = T^-1-space operator of the live systems; with zpart, the last CTA of
// each system also solves the coarse system for c = C^{-1} Z^T (T th) -> cout.
// grid (nmc * ceil(nseg / SP_WARPS), live slots)
#ifndef SP_MINB
#define SP_MINB 1
#endif
template <bool BJ>
__global__ void __launch_bounds__(SP_THREADS, SP_MINB) spec_op_kernel(SpecParams sp, const double* __restrict__ vh,
                                                             double* __restrict__ th, DeflateParams P, double* zpart,
                                                             int* counter, double* cout, double* __restrict__ uh) {
  pdl_wait();
  pdl_launch();
  extern __shared__ double sm[];  // [stage: SP_STAGE_DOUBLES] 2 d doubles (coarse solve)
  int s;
  if (!defl_slot(P, blockIdx.y, s)) return;
  const int nsg = (sp.nseg + SP_WARPS - 1) / SP_WARPS;
  const int mc = blockIdx.x / nsg, sg = (blockIdx.x % nsg) * SP_WARPS + (threadIdx.x >> 5);
  double* sbuf = sp.stage ? sm + (threadIdx.x >> 5) * SP_SSLOTS * SP_SROW : nullptr;
  if (sg < sp.nseg)
    spec_warp_item<BJ>(sp, s, mc, sg, vh, th, zpart ? zpart + (static_cast<long long>(s) * sp.nmc + mc) * sp.d : nullptr,
                       uh, 1.0, sbuf);
  if (!zpart) return;
  if (!last_cta(counter + s, sp.nmc * nsg)) return;
  double* sums = sm + (sp.stage ? SP_STAGE_DOUBLES : 0);
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
