// Strip solves around the Schur path, sm_100a:
//   schur_rhs:        b_S = B (A - mu)^{-1} f          (/root/reference/proj/src/schur.cpp:182-186)
//   recover_solution: u   = (A - mu)^{-1} (f - E x_S)  (/root/reference/proj/src/schur.cpp:227-230)
// The reference factors each strip kind of A (and every Helmholtz shift,
// proj/src/helmholtz.cpp:58-87) and solves strip by strip. Every strip block
// is the Kronecker sum Ax_kind (x) I + I (x) Az with Az shared by all kinds,
// so in the z eigenbasis (the spectral basis T of spectral.cuh) a strip solve
// is, per z mode q, an n x n complex solve Vx diag(1/(lx_p + lz_q - mu)) Vx^{-1}
// along x (fast diagonalisation). On the device:
//   1. strip_gather_kernel: reference node order (strip, ez, ix, iz) ->
//      strip rows X[strip][ix][ez*n + iz] (minus E x_S on the interface edges);
//   2. T^{-1} on every strip row (shared-matrix transform, xform.cuh / cuBLAS);
//   3. strip_modes_kernel: one thread per (system, strip, mode): the x-direction
//      eigen-solve; either the two edge traces B needs (schur_rhs, written
//      straight into the interface slots) or the full strip row (recover);
//   4. T back to physical coordinates; strip_scatter_kernel back to node order.
#pragma once

#include "common.cuh"
#include "spectral.cuh"

namespace smpm {

struct StripParams {
  int n, mx, mz, w, nmode, npairs, nsys;
  long long r, k;        // full-grid and interface lengths per system
  const double2* fac;    // 3 kinds x (Vx n*n | Vxi n*n | lx n | tW Vx n | tE Vx n), complex
  const double2* lz;     // nmode z eigenvalues (spectral basis order)
  const double* mu;      // nsys shifts
  double tau;
};

__host__ __device__ __forceinline__ int strip_fac_len(int n) { return 2 * n * n + 3 * n; }

// X[sys][s][ix][ez*n+iz] = f[sys][s][ez][ix][iz] (- x_S on the interface edge nodes:
// E places slot (i, side 0, Z) on the east edge of strip i and (i, side 1, Z) on
// the west edge of strip i + 1, proj/src/mesh.cpp:60-76, 82-87)
__global__ void strip_gather_kernel(StripParams P, const double* __restrict__ f, const double* __restrict__ xS,
                                    double* __restrict__ X) {
  const int n = P.n, w = P.w;
  const long long tot = static_cast<long long>(P.nsys) * P.r;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int sys = static_cast<int>(e / P.r);
    const int o = static_cast<int>(e - sys * P.r);
    const int s = o / (n * w), rem = o - s * n * w, ix = rem / w, Z = rem - ix * w;
    const int ez = Z / n, iz = Z - ez * n;
    const long long src = sys * P.r + (static_cast<long long>(s) * P.mz + ez) * n * n + ix * n + iz;
    double v = f[src];
    if (xS) {
      const double* xs = xS + sys * P.k;
      if (ix == n - 1 && s <= P.mx - 2) v -= xs[static_cast<long long>(s) * 2 * w + Z];
      if (ix == 0 && s >= 1) v -= xs[static_cast<long long>(s - 1) * 2 * w + w + Z];
    }
    X[e] = v;
  }
}

// u[sys][s][ez][ix][iz] = U[sys][s][ix][ez*n+iz]
__global__ void strip_scatter_kernel(StripParams P, const double* __restrict__ U, double* __restrict__ u) {
  const int n = P.n, w = P.w;
  const long long tot = static_cast<long long>(P.nsys) * P.r;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int sys = static_cast<int>(e / P.r);
    const int o = static_cast<int>(e - sys * P.r);
    const int nn = n * n;
    const int s = o / (P.mz * nn), rem = o - s * P.mz * nn, ez = rem / nn, r2 = rem - ez * nn;
    const int ix = r2 / n, iz = r2 - ix * n;
    u[e] = U[sys * P.r + (static_cast<long long>(s) * n + ix) * w + ez * n + iz];
  }
}

// Per (system, strip, z mode): y = Vx^{-1} z, d_p = y_p / (lx_p + lz_q - mu), then
//   TRACES: -tau (tW Vx) . d into slot (s-1, side 0) and -tau (tE Vx) . d into (s, side 1)
//           of the transformed interface vector bh (nsys x k, spectral coordinates);
//   FULL:   U = Vx d into the strip row Uh (nsys x r, spectral coordinates).
// A pair's coordinates (a, b) are the complex number z = a - i b (spectral.cuh).
template <int N, bool TRACES>
__global__ void __launch_bounds__(128) strip_modes_kernel(StripParams P, const double* __restrict__ Xh,
                                                          double* __restrict__ out) {
  __shared__ double2 fac[2 * N * N + 3 * N];
  const int s = blockIdx.y, sys = blockIdx.z;
  const int kind = s == 0 ? 0 : (s == P.mx - 1 ? 2 : 1);
  const double2* gf = P.fac + static_cast<long long>(kind) * strip_fac_len(N);
  for (int i = threadIdx.x; i < strip_fac_len(N); i += blockDim.x) fac[i] = gf[i];
  __syncthreads();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= P.nmode) return;
  const double2* Vx = fac;
  const double2* Vxi = fac + N * N;
  const double2* lx = fac + 2 * N * N;
  const double2* tWV = lx + N;
  const double2* tEV = tWV + N;
  const bool pair = m < P.npairs;
  const int e0 = pair ? 2 * m : P.npairs + m;
  const int w = P.w;
  const double* xs = Xh + sys * P.r + static_cast<long long>(s) * N * w + e0;
  double2 z[N];
#pragma unroll
  for (int ix = 0; ix < N; ++ix) {
    const double* p = xs + ix * w;
    z[ix] = make_double2(p[0], pair ? -p[1] : 0.0);
  }
  const double2 shift = csub(P.lz[m], make_double2(P.mu[sys], 0.0));
  double2 dd[N];
#pragma unroll
  for (int p = 0; p < N; ++p) {
    double2 y = make_double2(0.0, 0.0);
#pragma unroll
    for (int ix = 0; ix < N; ++ix) y = cfma(Vxi[p + ix * N], z[ix], y);
    dd[p] = cdiv(y, cadd(lx[p], shift));
  }
  if (TRACES) {
    double2 tw = make_double2(0.0, 0.0), te = make_double2(0.0, 0.0);
#pragma unroll
    for (int p = 0; p < N; ++p) {
      tw = cfma(tWV[p], dd[p], tw);
      te = cfma(tEV[p], dd[p], te);
    }
    double* bh = out + sys * P.k + e0;
    if (s >= 1) {
      double* q = bh + static_cast<long long>(2 * (s - 1)) * w;
      q[0] = -P.tau * tw.x;
      if (pair) q[1] = P.tau * tw.y;
    }
    if (s <= P.mx - 2) {
      double* q = bh + static_cast<long long>(2 * s + 1) * w;
      q[0] = -P.tau * te.x;
      if (pair) q[1] = P.tau * te.y;
    }
  } else {
    double* us = out + sys * P.r + static_cast<long long>(s) * N * w + e0;
#pragma unroll
    for (int ix = 0; ix < N; ++ix) {
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = 0; p < N; ++p) y = cfma(Vx[ix + p * N], dd[p], y);
      double* q = us + ix * w;
      q[0] = y.x;
      if (pair) q[1] = -y.y;
    }
  }
}

}  // namespace smpm
