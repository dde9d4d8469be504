// Bandwidth-bound kernels of the Schur-GMRES hot path (sm_100a): deflation
// (Z^T segmented sums, coarse solve, P/Q/2LAS updates, one CTA per system so
// the whole projection is a single launch), and the batched Arnoldi
// orthogonalization (CGS2 and MGS) with deterministic "last CTA reduces"
// cross-CTA reductions, device-side Givens updates and convergence flags.
#pragma once

#include "common.cuh"

namespace smpm {

constexpr int VEC_THREADS = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Deflation: one CTA per system.
// ---------------------------------------------------------------------------
struct DeflateParams {
  int nsys, d, w;
  long long k;
  const int* active;        // nullable
  const int* cmode;         // per system: 0 dense inverse (singular or general), 1 Thomas
  const double* cinv;       // nsys x d x d (column-major)
  const double* uc;         // nsys x d (singular systems)
  const int* singular;      // per system
  const double* thomas;     // nsys x 3 x d: sub, cprime, piv
  const double* rowsum;     // nsys x 6w: rW_I(2w) rE_I(2w) rE_W(w) rW_E(w)
  int mx;
  const int* alist;         // compacted active systems for slot grids (nullable)
  const int* acount;
};

__device__ __forceinline__ bool defl_slot(const DeflateParams& P, int slot, int& s) {
  if (P.acount && slot >= *P.acount) return false;
  s = P.alist ? P.alist[slot] : slot;
  return !(P.active && !P.active[s]);
}

enum DeflateMode : int {
  DEFL_P_FUSED = 0,   // y = zin - S Z c(Z^T zin), S Z c via row sums (zin == y allowed? no)
  DEFL_Q_TAIL = 1,    // y = v - Z c(Z^T zin)   (zin = S v)
  DEFL_COARSE = 2,    // cout = c(Z^T zin)
  DEFL_ADD_ZC = 3,    // y = v + Z c(Z^T zin)   (2LAS: zin = v, v = M^{-1} v)
  DEFL_SUB_T = 4,     // y = v - zin            (literal P tail: zin = S Z c)
  DEFL_COARSE_DIRECT = 5  // cout = c(zin) with zin a coarse vector (nsys x d)
};

__device__ void coarse_solve_block(const DeflateParams& P, int s, double* sums, double* c) {
  const int d = P.d;
  const int t = threadIdx.x;
  if (P.singular[s]) {
    // rhs = b - u_C (u_C . b)  (/root/reference/proj/src/deflation.cpp:73-76)
    __shared__ double red[32];
    const double* uc = P.uc + static_cast<long long>(s) * d;
    double acc = 0.0;
    for (int i = t; i < d; i += blockDim.x) acc += uc[i] * sums[i];
    acc = warp_sum(acc);
    if ((t & 31) == 0) red[t >> 5] = acc;
    __syncthreads();
    if (t < 32) {
      double v = t < (blockDim.x >> 5) ? red[t] : 0.0;
      v = warp_sum(v);
      if (t == 0) red[0] = v;
    }
    __syncthreads();
    const double dotv = red[0];
    for (int i = t; i < d; i += blockDim.x) sums[i] -= uc[i] * dotv;
    __syncthreads();
  }
  if (P.cmode[s] == 1) {
    // Thomas algorithm with precomputed reciprocal pivots (proj/src/deflation.cpp:77-90);
    // the bands are staged in shared memory so the serial recurrence never
    // waits on global loads
    __shared__ double band[3 * 512];
    const double* gsrc = P.thomas + static_cast<long long>(s) * 3 * d;
    const bool staged = d <= 512;
    if (staged)
      for (int i = t; i < 3 * d; i += blockDim.x) band[i] = gsrc[i];
    __syncthreads();
    if (t == 0) {
      // the recurrences carry their value in a register (one fma, or fma + mul, per step on
      // the serial chain); every load is independent of the chain and unrolled ahead of it
      const double* __restrict__ sub = staged ? band : gsrc;
      const double* __restrict__ cp = sub + d;
      const double* __restrict__ rpiv = cp + d;
      const double* __restrict__ rhs = sums;
      double* __restrict__ co = c;
      double yprev = rhs[0] * rpiv[0];
      co[0] = yprev;
#pragma unroll 8
      for (int i = 1; i < d; ++i) {
        yprev = fma(-sub[i - 1], yprev, rhs[i]) * rpiv[i];
        co[i] = yprev;
      }
      double cn = yprev;
#pragma unroll 8
      for (int i = d - 2; i >= 0; --i) {
        cn = fma(-cp[i], cn, co[i]);
        co[i] = cn;
      }
    }
  } else {
    const double* ci = P.cinv + static_cast<long long>(s) * d * d;
    for (int i = t; i < d; i += blockDim.x) {
      double acc = 0.0;
      for (int j = 0; j < d; ++j) acc += ci[static_cast<long long>(j) * d + i] * sums[j];
      c[i] = acc;
    }
  }
  __syncthreads();
}

// zin: vector whose Z^T sums feed the coarse solve; v: the vector updated.
__global__ void __launch_bounds__(VEC_THREADS)
deflate_kernel(DeflateParams P, int mode, const double* __restrict__ zin, const double* __restrict__ v,
               double* __restrict__ y, double* __restrict__ cout) {
  extern __shared__ double sm[];
  const int s = blockIdx.x;
  if (P.active && !P.active[s]) return;
  const int d = P.d, w = P.w;
  const long long k = P.k;
  double* sums = sm;
  double* c = sm + d;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const double* zs = zin + static_cast<long long>(s) * (mode == DEFL_COARSE_DIRECT ? d : k);
  const int w2 = 2 * w;
  if (mode == DEFL_COARSE_DIRECT) {
    for (int i = t; i < d; i += blockDim.x) sums[i] = zin[static_cast<long long>(s) * d + i];
    __syncthreads();
    coarse_solve_block(P, s, sums, c);
    for (int i = t; i < d; i += blockDim.x) cout[static_cast<long long>(s) * d + i] = c[i];
    return;
  }
  if (mode != DEFL_SUB_T) {
    // Z^T: segmented sums over the 2w slots of each interface (proj/src/deflation.cpp:16-22)
    for (int i = warp; i < d; i += nw) {
      const double* seg = zs + static_cast<long long>(i) * w2;
      double acc = 0.0;
      for (int e = lane; e < w2; e += 32) acc += seg[e];
      acc = warp_sum(acc);
      if (lane == 0) sums[i] = acc;
    }
    __syncthreads();
    coarse_solve_block(P, s, sums, c);
  }
  if (mode == DEFL_COARSE) {
    for (int i = t; i < d; i += blockDim.x) cout[static_cast<long long>(s) * d + i] = c[i];
    return;
  }
  const double* vs = v + static_cast<long long>(s) * k;
  double* ys = y + static_cast<long long>(s) * k;
  if (mode == DEFL_SUB_T) {
    for (long long e = t; e < k; e += blockDim.x) ys[e] = vs[e] - zs[e];
    return;
  }
  if (mode == DEFL_Q_TAIL || mode == DEFL_ADD_ZC) {
    const double sg = mode == DEFL_Q_TAIL ? -1.0 : 1.0;
    for (long long e = t; e < k; e += blockDim.x) ys[e] = vs[e] + sg * c[e / w2];
    return;
  }
  // DEFL_P_FUSED: y = v - Z c - scatter(strip row sums) ; here v == zin (t = S u)
  const double* rs = P.rowsum + static_cast<long long>(s) * 6 * w;
  const double* rWI = rs;           // interior strip, W-own column sums, rows [W-readers; E-readers]
  const double* rEI = rs + w2;      // interior strip, E-own column sums
  const double* rEW = rs + 2 * w2;  // west-boundary strip (E-readers x E-own)
  const double* rWE = rEW + w;      // east-boundary strip (W-readers x W-own)
  const int mx = P.mx;
  for (long long e = t; e < k; e += blockDim.x) {
    const int blk = static_cast<int>(e / w);
    const int r = static_cast<int>(e - static_cast<long long>(blk) * w);
    const int i = blk >> 1;  // interface
    double sz;
    if ((blk & 1) == 0) {
      // left side of interface i = west-readers of strip i+1 (reads c_i on its W-own, c_{i+1} on E-own)
      const int st = i + 1;
      if (st == mx - 1)
        sz = c[i] * rWE[r];
      else
        sz = c[i] * rWI[r] + c[i + 1] * rEI[r];
    } else {
      // right side of interface i = east-readers of strip i (c_{i-1} on W-own, c_i on E-own)
      const int st = i;
      if (st == 0)
        sz = c[i] * rEW[r];
      else
        sz = c[i - 1] * rWI[w + r] + c[i] * rEI[w + r];
    }
    ys[e] = vs[e] - (c[i] + sz);
  }
}

// y = Z c broadcast (c: nsys x d)
__global__ void zbroadcast_kernel(int nsys, int d, int w2, long long k, const int* active, const double* __restrict__ c,
                                  double* __restrict__ y) {
  const long long tot = static_cast<long long>(nsys) * k;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(e / k);
    if (active && !active[s]) continue;
    const long long r = e - static_cast<long long>(s) * k;
    y[e] = c[static_cast<long long>(s) * d + r / w2];
  }
}

// Z^T only (nsys x d out), one warp per interface
__global__ void zt_kernel(int nsys, int d, int w2, long long k, const double* __restrict__ v, double* __restrict__ y) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= nsys * d) return;
  const int s = gw / d, i = gw % d;
  const double* seg = v + static_cast<long long>(s) * k + static_cast<long long>(i) * w2;
  double acc = 0.0;
  for (int e = lane; e < w2; e += 32) acc += seg[e];
  acc = warp_sum(acc);
  if (lane == 0) y[gw] = acc;
}

// ---------------------------------------------------------------------------
// Batched GMRES state (structure of arrays, one entry per system)
// ---------------------------------------------------------------------------
enum GmState : int { GM_RUN = 0, GM_CONV = 1, GM_BREAK = 2, GM_MAXED = 3, GM_CYCLE = 4 };

struct GmState_ {
  int* jcyc;      // Arnoldi index inside the current cycle (0-based column being built)
  int* iters;     // total iterations
  int* state;     // GmState
  int* active;    // 1 while the operator/orthogonalization must run for the system
  int* counter;   // last-CTA counters, one per system
  int* hist_len;
  double* bnorm;  // ||rhs of GMRES||
  double* target; // absolute tolerance
  double* hmax;
  double* nrm;    // norm of the latest Arnoldi vector
  double* R;      // nsys x (m+1) x m  (triangularized Hessenberg columns)
  double* cs;     // nsys x m
  double* sn;     // nsys x m
  double* g;      // nsys x (m+1)
  double* h1;     // nsys x (m+2)
  double* h2;     // nsys x (m+2)
  double* y;      // nsys x m
  double* hist;   // nsys x histcap
  double* part;   // nsys x nchunk x (m+2) partial sums
  int m;          // cycle length
  int m_total;    // max iterations
  int histcap;
  long long k;
  long long vstride;  // (m+1)*k per system
  int chunk, nchunk;
  int nsys;
  const int* alist;   // compacted active systems for (chunk, slot) grids
  const int* acount;  // number of valid slots
  int stacked;        // one GMRES over all systems stacked (proj/src/helmholtz.cpp:187-246)
  double* snsq;       // stacked: per-system ||w||^2 of the norm pass
};

// (chunk, slot) grid -> system; false when the slot is past the live count
__device__ __forceinline__ bool gm_slot(const GmState_& G, int slot, int& s) {
  if (G.acount && slot >= *G.acount) return false;
  s = G.alist ? G.alist[slot] : slot;
  return G.active[s] != 0;
}

// partial dot products of columns [0, ncols) of V_s with x over rows [r0, r1),
// warp per column; writes part[s][chunk][col]
__device__ __forceinline__ void chunk_dots(const double* __restrict__ Vs, long long k, int ncols,
                                           const double* __restrict__ xs, int r0, int r1, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < ncols; i += nw) {
    const double* col = Vs + static_cast<long long>(i) * k;
    double acc = 0.0;
    for (int r = r0 + lane; r < r1; r += 32) acc = fma(col[r], xs[r], acc);
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

// returns true in exactly one CTA per system once all its chunks have written partials
__device__ __forceinline__ bool last_cta(int* counter, int nchunk) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(counter, 1);
    is_last = (old == nchunk - 1);
    if (is_last) *counter = 0;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// reduce part[s][0..nchunk)[0..ncols) -> out[0..ncols): warp per column,
// lanes stride the chunks, fixed butterfly -> deterministic and latency-short
__device__ __forceinline__ void reduce_parts(const double* __restrict__ part, int nchunk, int stride, int ncols,
                                             double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < ncols; i += nw) {
    double acc = 0.0;
    for (int c = lane; c < nchunk; c += 32) acc += part[static_cast<long long>(c) * stride + i];
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

// sum of part[c*stride], c < nchunk, by one warp (returns the total in every lane)
__device__ __forceinline__ double warp_reduce_strided(const double* __restrict__ part, int nchunk, int stride) {
  double acc = 0.0;
  for (int c = threadIdx.x & 31; c < nchunk; c += 32) acc += part[static_cast<long long>(c) * stride];
  return warp_sum(acc);
}

// ---- CGS2 pass 1: h1 = V^T w ----------------------------------------------
__global__ void __launch_bounds__(VEC_THREADS) cgs_dot_kernel(GmState_ G, const double* __restrict__ V,
                                                              const double* __restrict__ w) {
  const int s = blockIdx.y;
  if (!G.active[s]) return;
  const int ncols = G.jcyc[s] + 1;
  const int ch = blockIdx.x;
  const int r0 = ch * G.chunk, r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const int stride = G.m + 2;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  chunk_dots(V + s * G.vstride, G.k, ncols, w + s * G.k, r0, r1, part);
  if (last_cta(G.counter + s, G.nchunk))
    reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols,
                 G.h1 + static_cast<long long>(s) * stride);
}

__device__ void givens_step(GmState_& G, int s, int j, double nrm);

// ---- CGS2 pass 2/3: w -= V h; then (pass 2) h2 = V^T w or (pass 3) ||w|| ----
template <bool NORM>
__global__ void __launch_bounds__(VEC_THREADS) cgs_update_kernel(GmState_ G, const double* __restrict__ V,
                                                                 double* __restrict__ w, int do_update) {
  extern __shared__ double hs[];  // m + 2 doubles
  __shared__ double red[32];
  const int s = blockIdx.y;
  if (!G.active[s]) return;
  const int j = G.jcyc[s];
  const int ncols = j + 1;
  const int stride = G.m + 2;
  const double* hin = (NORM ? G.h2 : G.h1) + static_cast<long long>(s) * stride;
  for (int i = threadIdx.x; i < ncols; i += blockDim.x) hs[i] = hin[i];
  __syncthreads();
  const int ch = blockIdx.x;
  const int r0 = ch * G.chunk, r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  double sq = 0.0;
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    double acc = ws[r];
    if (do_update) {
      for (int i = 0; i < ncols; ++i) acc = fma(-Vs[static_cast<long long>(i) * G.k + r], hs[i], acc);
      ws[r] = acc;
    }
    sq = fma(acc, acc, sq);
  }
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  if (!NORM) {
    __syncthreads();  // this CTA's rows of w are final (own rows only)
    chunk_dots(Vs, G.k, ncols, ws, r0, r1, part);
    if (last_cta(G.counter + s, G.nchunk))
      reduce_parts(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride, ncols,
                   G.h2 + static_cast<long long>(s) * stride);
    return;
  }
  sq = warp_sum(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tsum = 0.0;
    for (int i = 0; i < (blockDim.x >> 5); ++i) tsum += red[i];
    part[0] = tsum;
  }
  if (!last_cta(G.counter + s, G.nchunk)) return;
  if (threadIdx.x >= 32) return;
  // ---- last CTA, warp 0: norm + Givens + convergence (proj/src/gmres.cpp:71-99)
  const double nsq = warp_reduce_strided(G.part + static_cast<long long>(s) * G.nchunk * stride, G.nchunk, stride);
  givens_step(G, s, j, sqrt(nsq));
}

// Hessenberg column j of system s from h1 + h2 (Arnoldi coefficients) and
// nrm (subdiagonal): previous rotations, a new Givens rotation, the residual
// estimate |g_{j+1}|, history and the stop tests (proj/src/gmres.cpp:71-99)
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Called by all 32 lanes of one warp. The column and the stored rotations
// are staged in shared memory so the sequential rotation sweep (lane 0)
// never waits on global loads.
__device__ void givens_step(GmState_& G, int s, int j, double nrm) {
  constexpr int SM = 256;
  __shared__ double hs[SM + 1], css[SM], sns[SM];
  const int lane = threadIdx.x & 31;
  const int stride = G.m + 2;
  const int m = G.m;
  double* h1 = G.h1 + static_cast<long long>(s) * stride;
  const double* h2 = G.h2 + static_cast<long long>(s) * stride;
  double* cs = G.cs + static_cast<long long>(s) * m;
  double* sn = G.sn + static_cast<long long>(s) * m;
  double* g = G.g + static_cast<long long>(s) * (m + 1);
  double* R = G.R + static_cast<long long>(s) * (m + 1) * m;
  const bool staged = j + 2 <= SM;
  // lane 0's scalars, loaded up front (independent loads: one round trip under the column loads)
  double p_hmax = 0.0, p_g1 = 0.0, p_g2 = 0.0, p_target = 0.0, p_bnorm = 1.0;
  int p_it = 0, p_hl = 0;
  if (lane == 0) {
    p_hmax = G.hmax[s];
    p_g1 = g[j];
    p_g2 = g[j + 1];
    p_target = G.target[s];
    p_bnorm = G.bnorm[s];
    p_it = G.iters[s];
    p_hl = G.hist_len[s];
  }
  double* H = staged ? hs : h1;
  const double* CS = staged ? css : cs;
  const double* SN = staged ? sns : sn;
  double hm = 0.0;
  for (int i = lane; i <= j; i += 32) {
    const double v = h1[i] + h2[i];
    H[i] = v;
    hm = fmax(hm, fabs(v));
  }
  if (staged)
    for (int i = lane; i < j; i += 32) {
      css[i] = cs[i];
      sns[i] = sn[i];
    }
  hm = warp_max(hm);
  __syncwarp();
  __threadfence_block();
  double hmax = 0.0, res = 0.0;
  if (lane == 0) {
    G.nrm[s] = nrm;
    hmax = fmax(fmax(p_hmax, hm), nrm);
    G.hmax[s] = hmax;
    H[j + 1] = nrm;
    for (int i = 0; i < j; ++i) {
      const double t1 = H[i], t2 = H[i + 1];
      H[i] = CS[i] * t1 + SN[i] * t2;
      H[i + 1] = -SN[i] * t1 + CS[i] * t2;
    }
    const double rad = hypot(H[j], H[j + 1]);
    const double c = rad > 0.0 ? H[j] / rad : 1.0;
    const double sv = rad > 0.0 ? H[j + 1] / rad : 0.0;
    cs[j] = c;
    sn[j] = sv;
    H[j] = rad;
    const double g1 = p_g1, g2 = p_g2;
    const double gj1 = -sv * g1 + c * g2;
    g[j] = c * g1 + sv * g2;
    g[j + 1] = gj1;
    res = fabs(gj1);
  }
  __syncwarp();
  __threadfence_block();
  for (int i = lane; i <= j; i += 32) R[static_cast<long long>(j) * (m + 1) + i] = H[i];
  if (lane != 0) return;
  const int it = p_it + 1;
  G.iters[s] = it;
  G.jcyc[s] = j + 1;
  const int hl = p_hl;
  if (hl < G.histcap) {
    G.hist[static_cast<long long>(s) * G.histcap + hl] = res / p_bnorm;
    G.hist_len[s] = hl + 1;
  }
  int st = GM_RUN;
  if (res <= p_target)
    st = GM_CONV;
  else if (nrm <= 1e-14 * hmax)
    st = GM_BREAK;
  else if (it >= G.m_total)
    st = GM_MAXED;
  else if (j + 1 >= m)
    st = GM_CYCLE;
  G.state[s] = st;
  if (st != GM_RUN) G.active[s] = 0;
}

// v_{j+1} = w / ||w|| into V[:, jcyc] and the operator input buffer
__global__ void gm_scale_kernel(GmState_ G, double* __restrict__ V, const double* __restrict__ w,
                                double* __restrict__ vin) {
  pdl_wait();
  pdl_launch();
  int s;
  if (!gm_slot(G, blockIdx.y, s)) return;
  const double inv = 1.0 / G.nrm[s];
  const int j = G.jcyc[s];
  double* col = V + s * G.vstride + static_cast<long long>(j) * G.k;
  const double* ws = w + s * G.k;
  double* vs = vin + s * G.k;
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < G.k;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double v = ws[r] * inv;
    col[r] = v;
    vs[r] = v;
  }
}

// ---- MGS: one fused step per basis vector: w -= h_{i-1} v_{i-1}; h_i = v_i . w
// (i == ncols finishes with the norm + Givens via cgs_update_kernel<true> on h2 = 0)
__global__ void __launch_bounds__(VEC_THREADS) mgs_step_kernel(GmState_ G, const double* __restrict__ V,
                                                               double* __restrict__ w, int i) {
  const int s = blockIdx.y;
  if (!G.active[s]) return;
  const int ncols = G.jcyc[s] + 1;
  if (i > ncols) return;
  const int stride = G.m + 2;
  const int ch = blockIdx.x;
  const int r0 = ch * G.chunk, r1 = static_cast<int>(min(G.k, static_cast<long long>(r0) + G.chunk));
  const double* Vs = V + s * G.vstride;
  double* ws = w + s * G.k;
  double* h1 = G.h1 + static_cast<long long>(s) * stride;
  if (i > 0) {
    const double hp = h1[i - 1];
    const double* vp = Vs + static_cast<long long>(i - 1) * G.k;
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) ws[r] = fma(-hp, vp[r], ws[r]);
    __syncthreads();
  }
  if (i == ncols) return;
  double* part = G.part + (static_cast<long long>(s) * G.nchunk + ch) * stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double red[32];
  const double* vi = Vs + static_cast<long long>(i) * G.k;
  double acc = 0.0;
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) acc = fma(vi[r], ws[r], acc);
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (blockDim.x >> 5); ++q) t += red[q];
    part[0] = t;
  }
  if (last_cta(G.counter + s, G.nchunk) && threadIdx.x == 0) {
    double t = 0.0;
    const double* p0 = G.part + static_cast<long long>(s) * G.nchunk * stride;
    for (int c = 0; c < G.nchunk; ++c) t += p0[static_cast<long long>(c) * stride];
    h1[i] = t;
  }
}

// zero h2 (MGS path has no second pass)
__global__ void gm_zero_h2_kernel(GmState_ G) {
  const int s = blockIdx.x;
  if (!G.active[s]) return;
  double* h2 = G.h2 + static_cast<long long>(s) * (G.m + 2);
  for (int i = threadIdx.x; i < G.m + 2; i += blockDim.x) h2[i] = 0.0;
}

// ---- generic batched squared norms / dots: out[s] = sum x_s . y_s --------
__global__ void __launch_bounds__(VEC_THREADS) batched_dot_kernel(int nsys, long long k, int chunk, int nchunk,
                                                                  const int* active, const double* __restrict__ x,
                                                                  const double* __restrict__ y,
                                                                  double* __restrict__ part, int* counter,
                                                                  double* __restrict__ out) {
  __shared__ double red[32];
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const int ch = blockIdx.x;
  const long long r0 = static_cast<long long>(ch) * chunk, r1 = min(k, r0 + chunk);
  const double* xs = x + s * k;
  const double* ys = y + s * k;
  double acc = 0.0;
  for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) acc = fma(xs[r], ys[r], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (blockDim.x >> 5); ++q) t += red[q];
    part[static_cast<long long>(s) * nchunk + ch] = t;
  }
  if (last_cta(counter + s, nchunk) && threadIdx.x == 0) {
    double t = 0.0;
    for (int c = 0; c < nchunk; ++c) t += part[static_cast<long long>(s) * nchunk + c];
    out[s] = t;
  }
}

// y = a[s]*x + b*y  per system (a from device array, optional)
__global__ void axpby_kernel(int nsys, long long k, const int* active, const double* __restrict__ a_dev, double a,
                             const double* __restrict__ x, double b, double* __restrict__ y) {
  const long long tot = static_cast<long long>(nsys) * k;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(e / k);
    if (active && !active[s]) continue;
    const double av = a_dev ? a_dev[s] : a;
    y[e] = fma(av, x[e], b * y[e]);
  }
}

// out = v - dir * dots[s]
__global__ void project_kernel(int nsys, long long k, const double* __restrict__ dots, const double* __restrict__ v,
                               const double* __restrict__ dir, double* __restrict__ out) {
  const long long tot = static_cast<long long>(nsys) * k;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(e / k);
    out[e] = fma(-dir[e], dots[s], v[e]);
  }
}

// ---- GMRES cycle start: bnorm/target on the first cycle, g0, v0 = r / ||r|| ----
// nrm2sq: ||r||^2 per system; first: 1 on the first cycle.
__device__ __forceinline__ void gm_start_one(GmState_& G, int s, double nrm2sq, double bs_nrm2sq, double tol, int first) {
  const double rn = sqrt(nrm2sq);
  const int m = G.m;
  if (first) {
    G.bnorm[s] = rn;
    // abs target = tol * ||b_S|| (proj/src/deflation.cpp:109)
    G.target[s] = tol * sqrt(bs_nrm2sq);
    G.hmax[s] = 0.0;
    G.iters[s] = 0;
    G.hist_len[s] = 1;
    G.hist[static_cast<long long>(s) * G.histcap] = rn > 0.0 ? 1.0 : 0.0;
  }
  double* g = G.g + static_cast<long long>(s) * (m + 1);
  for (int i = 0; i <= m; ++i) g[i] = 0.0;
  g[0] = rn;
  G.nrm[s] = rn;
  G.jcyc[s] = 0;
  const bool go = rn > 0.0 && G.iters[s] < G.m_total;
  G.state[s] = go ? GM_RUN : GM_CONV;
  G.active[s] = go ? 1 : 0;
}

__global__ void gm_start_kernel(GmState_ G, const double* __restrict__ nrm2sq, const double* __restrict__ bs_nrm2sq,
                                double tol, int first, const int* __restrict__ restart_mask) {
  pdl_wait();
  pdl_launch();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= G.nsys) return;
  if (!first && !(restart_mask && restart_mask[s] == GM_CYCLE)) return;
  gm_start_one(G, s, nrm2sq[s], first ? bs_nrm2sq[s] : 0.0, tol, first);
}

// First cycle of an independent (not stacked) solve in one launch: ||b_S||^2 and ||rhs||^2
// per system (same chunks and summation order as two batched_dot_kernel launches, so the
// same bits), then the last CTA of each system starts its GMRES state (gm_start_one) and
// keeps c_b (csrc -> cdst, d doubles per system; nullable)
__global__ void __launch_bounds__(VEC_THREADS) norm2_start_kernel(GmState_ G, long long k, int chunk, int nchunk,
                                                                  const double* __restrict__ bs,
                                                                  const double* __restrict__ rhs,
                                                                  double* __restrict__ part, int* counter,
                                                                  double* __restrict__ nb2, double* __restrict__ nr2,
                                                                  double tol, const double* __restrict__ csrc,
                                                                  double* __restrict__ cdst, int d) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[2][32];
  const int s = blockIdx.y;
  const int ch = blockIdx.x;
  const long long r0 = static_cast<long long>(ch) * chunk, r1 = min(k, r0 + chunk);
  const double* xs = bs + s * k;
  const double* ys = rhs + s * k;
  double a0 = 0.0, a1 = 0.0;
  for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const double xv = xs[r], yv = ys[r];
    a0 = fma(xv, xv, a0);
    a1 = fma(yv, yv, a1);
  }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a0;
    red[1][threadIdx.x >> 5] = a1;
  }
  __syncthreads();
  double* p0 = part + static_cast<long long>(s) * nchunk;
  double* p1 = part + (static_cast<long long>(G.nsys) + s) * nchunk;
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int q = 0; q < (blockDim.x >> 5); ++q) {
      t0 += red[0][q];
      t1 += red[1][q];
    }
    p0[ch] = t0;
    p1[ch] = t1;
  }
  if (last_cta(counter + s, nchunk)) {
    if (threadIdx.x == 0) {
      double t0 = 0.0, t1 = 0.0;
      for (int c = 0; c < nchunk; ++c) {
        t0 += p0[c];
        t1 += p1[c];
      }
      nb2[s] = t0;
      nr2[s] = t1;
      gm_start_one(G, s, t1, t0, tol, 1);
    }
    if (cdst)
      for (int i = threadIdx.x; i < d; i += blockDim.x)
        cdst[static_cast<long long>(s) * d + i] = csrc[static_cast<long long>(s) * d + i];
  }
}

// v0 = r / ||r|| into V[:,0] and vin, for systems just (re)started; first cycle: also
// x = 0 for every system (xzero) and the grid tail's barrier word (zero_word)
// and the compacted list of the live systems (alist / acount, ascending; nsys <= blockDim.x)
__global__ void gm_v0_kernel(GmState_ G, double* __restrict__ V, const double* __restrict__ r,
                             double* __restrict__ vin, double* __restrict__ xzero, unsigned* zero_word,
                             int* __restrict__ alist, int* __restrict__ acount) {
  pdl_wait();
  pdl_launch();
  const int s = blockIdx.y;
  if (zero_word && blockIdx.x == 0 && s == 0 && threadIdx.x == 0) *zero_word = 0u;
  if (alist && blockIdx.x == 0 && s == 0) {
    __shared__ int wsum[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int f = (t < G.nsys && G.active[t]) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int q = 0; q < warp; ++q) off += wsum[q];
    if (f) alist[off + __popc(bal & ((1u << lane) - 1u))] = t;
    if (t == 0) {
      int tot = 0;
      for (int q = 0; q < (blockDim.x >> 5); ++q) tot += wsum[q];
      *acount = tot;
    }
  }
  if (xzero) {
    double* xs = xzero + s * G.k;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < G.k;
         e += static_cast<long long>(gridDim.x) * blockDim.x)
      xs[e] = 0.0;
  }
  if (!G.active[s] || G.jcyc[s] != 0) return;
  const double inv = 1.0 / G.nrm[s];
  double* col = V + s * G.vstride;
  const double* rs = r + s * G.k;
  double* vs = vin + s * G.k;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < G.k;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double v = rs[e] * inv;
    col[e] = v;
    vs[e] = v;
  }
}

// back-substitution R y = g for the systems whose cycle ended (warp per system)
// (proj/src/gmres.cpp:116-125); ncyc = columns built in this cycle
__global__ void gm_backsolve_kernel(GmState_ G, const int* __restrict__ sel) {
  pdl_wait();
  pdl_launch();
  // column-oriented back substitution: y_i = b_i / r_ii, then b_r -= r_ri y_i
  // for r < i; the triangle is staged in shared memory for short cycles
  constexpr int NS = 96;
  __shared__ double tri[NS * (NS + 1) / 2];
  __shared__ double bsh[NS];
  const int s = blockIdx.x;
  if (sel && !sel[s]) return;
  const int lane = threadIdx.x;
  const int n = G.jcyc[s];
  const int m = G.m;
  const double* R = G.R + static_cast<long long>(s) * (m + 1) * m;
  const double* g = G.g + static_cast<long long>(s) * (m + 1);
  double* y = G.y + static_cast<long long>(s) * m;
  if (n <= NS) {
    // flat, independent loads of the packed triangle (column c holds rows 0..c)
    const int nt = n * (n + 1) / 2;
    for (int e = lane; e < nt; e += 32) {
      int c = static_cast<int>((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      if (c * (c + 1) / 2 > e) --c;
      if ((c + 1) * (c + 2) / 2 <= e) ++c;
      tri[e] = R[static_cast<long long>(c) * (m + 1) + (e - c * (c + 1) / 2)];
    }
    for (int r = lane; r < n; r += 32) bsh[r] = g[r];
    __syncwarp();
    for (int i = n - 1; i >= 0; --i) {
      const double rii = tri[i * (i + 1) / 2 + i];
      const double yi = fabs(rii) > 0.0 ? bsh[i] / rii : 0.0;
      if (lane == 0) y[i] = yi;
      for (int r = lane; r < i; r += 32) bsh[r] -= tri[i * (i + 1) / 2 + r] * yi;
      __syncwarp();
    }
    return;
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = 0.0;
    for (int c = i + 1 + lane; c < n; c += 32) acc += R[static_cast<long long>(c) * (m + 1) + i] * y[c];
    acc = warp_sum(acc);
    if (lane == 0) {
      const double rii = R[static_cast<long long>(i) * (m + 1) + i];
      y[i] = fabs(rii) > 0.0 ? (g[i] - acc) / rii : 0.0;
    }
    __syncwarp();
  }
}

// x (+)= V y over the columns of the finished cycle
__global__ void gm_combine_kernel(GmState_ G, const double* __restrict__ V, double* __restrict__ x,
                                  const int* __restrict__ sel, int accumulate) {
  pdl_wait();
  pdl_launch();
  const int s = blockIdx.y;
  if (sel && !sel[s]) return;
  const int n = G.jcyc[s];
  const double* y = G.y + static_cast<long long>(s) * G.m;
  const double* Vs = V + s * G.vstride;
  double* xs = x + s * G.k;
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < G.k;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    double acc = accumulate ? xs[r] : 0.0;
    for (int i = 0; i < n; ++i) acc = fma(Vs[static_cast<long long>(i) * G.k + r], y[i], acc);
    xs[r] = acc;
  }
}

// ---- stacked GMRES (proj/src/helmholtz.cpp:187-246): the systems of the batch are
// the segments of ONE Krylov vector, so every inner product is the sum of the
// per-system ones.  The per-system reductions of the passes run unchanged; these
// kernels then sum them over the systems in a fixed order (deterministic) and
// hand every system the same global value, so all systems carry an identical
// Hessenberg / Givens state and stop together.

// v[s] = sum_t v[t] for every system (one CTA)
__global__ void stack_sum_kernel(int nsys, double* __restrict__ v) {
  pdl_wait();
  pdl_launch();
  __shared__ double tot;
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int t = 0; t < nsys; ++t) a += v[t];
    tot = a;
  }
  __syncthreads();
  for (int s = threadIdx.x; s < nsys; s += blockDim.x) v[s] = tot;
}

// h[s][c] = sum_t h[t][c] for the current Arnoldi column count (one CTA, thread per column)
__global__ void stack_h_kernel(GmState_ G, double* __restrict__ h) {
  pdl_wait();
  pdl_launch();
  const int stride = G.m + 2;
  const int ncols = G.jcyc[0] + 1;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double a = 0.0;
    for (int t = 0; t < G.nsys; ++t) a += h[static_cast<long long>(t) * stride + c];
    for (int t = 0; t < G.nsys; ++t) h[static_cast<long long>(t) * stride + c] = a;
  }
}

// ---- stacked solve across ranks (one all-reduce per inner product): the local sums
// go to a small buffer, the caller's all-reduce hook sums it over the ranks, and the
// result is broadcast to every local system.  Same local summation order as the
// single-rank kernels above.
__global__ void stack_sum_local_kernel(int nsys, const double* __restrict__ v, double* __restrict__ buf) {
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int t = 0; t < nsys; ++t) a += v[t];
    buf[0] = a;
  }
}
__global__ void stack_sum_bcast_kernel(int nsys, double* __restrict__ v, const double* __restrict__ buf) {
  for (int s = threadIdx.x; s < nsys; s += blockDim.x) v[s] = buf[0];
}
__global__ void stack_h_local_kernel(GmState_ G, const double* __restrict__ h, double* __restrict__ buf) {
  const int stride = G.m + 2;
  const int ncols = G.jcyc[0] + 1;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double a = 0.0;
    for (int t = 0; t < G.nsys; ++t) a += h[static_cast<long long>(t) * stride + c];
    buf[c] = a;
  }
}
__global__ void stack_h_bcast_kernel(GmState_ G, double* __restrict__ h, const double* __restrict__ buf) {
  const int stride = G.m + 2;
  const int ncols = G.jcyc[0] + 1;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    const double a = buf[c];
    for (int t = 0; t < G.nsys; ++t) h[static_cast<long long>(t) * stride + c] = a;
  }
}
// Givens step of every system from the all-reduced ||w||^2 in buf[0]
__global__ void stack_givens_global_kernel(GmState_ G, const double* __restrict__ buf) {
  const int s = blockIdx.x;
  if (!G.active[s]) return;
  givens_step(G, s, G.jcyc[s], sqrt(buf[0]));
}

// global ||w|| from the per-system squares, then the Givens step of every system (warp each)
__global__ void stack_givens_kernel(GmState_ G) {
  pdl_wait();
  pdl_launch();
  const int s = blockIdx.x;
  if (!G.active[s]) return;
  double a = 0.0;
  for (int t = 0; t < G.nsys; ++t) a += G.snsq[t];
  givens_step(G, s, G.jcyc[s], sqrt(a));
}

}  // namespace smpm
