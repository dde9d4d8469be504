// Transverse Fourier transforms of the 3D extension, sm_100a:
//   fourier_transform_y  (/root/reference/proj/src/fourier.cpp:47-62): per node row of an
//     r x m_y field (column-major: plane y is a contiguous r-vector), the first m_y / 2
//     coefficients of the forward DFT, scaled by 1 / m_y;
//   inverse_fourier_y    (:64-86): the Hermitian extension of those coefficients
//     (Nyquist term zero) transformed back, real part.
// Coefficients are laid out as Schur-batch systems: system 2 j + part (part 0 = real,
// 1 = imaginary) is the r-vector of mode j, so the per-mode real / imaginary right-hand
// sides of proj/src/helmholtz.cpp:162-178 feed smpm_schur_rhs directly.
// One CTA per tile of consecutive nodes: coalesced loads along the nodes of each plane
// into shared memory (node rows padded to m_y + 1), one radix-2 FFT per node by a warp (bit reversal, log2 m_y
// butterfly stages, twiddles from a table), coalesced stores per mode.
#pragma once

#include "common.cuh"

namespace smpm {

constexpr int FY_THREADS = 256;

struct FourierArgs {
  long long r;            // nodes (rows)
  int m_y;                // planes (power of two)
  int tile;               // nodes per CTA
  const double2* tw;      // m_y / 2 twiddles exp(sign 2 pi i k / m_y) for the direction used
};

// in-place radix-2 FFT of x[0..m) (shared memory) by one warp; tw[k] = exp(sign 2 pi i k / m)
__device__ __forceinline__ void warp_fft(double2* x, int m, const double2* __restrict__ tw) {
  const int lane = threadIdx.x & 31;
  int lg = 0;
  while ((1 << lg) < m) ++lg;
  for (int i = lane; i < m; i += 32) {
    const int j = static_cast<int>(__brev(static_cast<unsigned>(i)) >> (32 - lg));
    if (i < j) {
      const double2 t = x[i];
      x[i] = x[j];
      x[j] = t;
    }
  }
  __syncwarp();
  for (int ls = 0; ls < lg; ++ls) {
    const int h = 1 << ls, sshift = lg - 1 - ls;  // half length, log2(m / len)
    for (int b = lane; b < m / 2; b += 32) {
      const int grp = b >> ls, jj = b & (h - 1);
      const int i0 = (grp << (ls + 1)) + jj, i1 = i0 + h;
      const double2 w = __ldg(tw + (jj << sshift));
      const double2 v = x[i1];
      const double2 vw = make_double2(fma(v.x, w.x, -v.y * w.y), fma(v.x, w.y, v.y * w.x));
      const double2 u = x[i0];
      x[i0] = make_double2(u.x + vw.x, u.y + vw.y);
      x[i1] = make_double2(u.x - vw.x, u.y - vw.y);
    }
    __syncwarp();
  }
}

// shared-memory address of element idx of a transformed row (XOR swizzle so the
// register FFT's per-lane contiguous stores hit distinct banks)
__device__ __forceinline__ int fy_swz(int idx, bool swz) { return swz ? idx ^ ((idx >> 3) & 7) : idx; }

__device__ __forceinline__ double2 shfl_xor_d2(double2 v, int mask) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}

// Radix-2 FFT of x[0..m) (m = 32 R) by one warp in registers: lane l gathers the
// bit-reversed elements l R .. l R + R - 1 (conflict-free), runs the log2 R short
// stages in registers and the 5 long ones across lanes with shuffles (butterfly
// partners differ in one lane bit), and stores the result in natural order with
// the fy_swz swizzle. Same butterflies and twiddles as warp_fft.
template <int R>
__device__ __forceinline__ void warp_fft_reg(double2* x, int lg, const double2* __restrict__ tw) {
  const int lane = threadIdx.x & 31;
  const int m = 32 * R;
  double2 v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int idx = lane * R + q;
    v[q] = x[static_cast<int>(__brev(static_cast<unsigned>(idx)) >> (32 - lg))];
  }
#pragma unroll
  for (int len = 2; len <= R; len <<= 1) {
    const int h = len >> 1, step = m / len;
#pragma unroll
    for (int g = 0; g < R; g += len)
#pragma unroll
      for (int jj = 0; jj < h; ++jj) {
        const double2 w = __ldg(tw + jj * step);
        const double2 a = v[g + jj], b = v[g + jj + h];
        const double2 bw = make_double2(fma(b.x, w.x, -b.y * w.y), fma(b.x, w.y, b.y * w.x));
        v[g + jj] = make_double2(a.x + bw.x, a.y + bw.y);
        v[g + jj + h] = make_double2(a.x - bw.x, a.y - bw.y);
      }
  }
#pragma unroll
  for (int sb = 0; sb < 5; ++sb) {
    const int h = R << sb, step = m / (2 * h), bit = 1 << sb;
    const bool upper = (lane & bit) != 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int jj = (lane * R + q) & (h - 1);
      const double2 w = __ldg(tw + jj * step);
      const double2 o = shfl_xor_d2(v[q], bit);
      if (!upper) {  // lower element: u + w v (v from the partner)
        const double2 ow = make_double2(fma(o.x, w.x, -o.y * w.y), fma(o.x, w.y, o.y * w.x));
        v[q] = make_double2(v[q].x + ow.x, v[q].y + ow.y);
      } else {       // upper element: u - w v (u from the partner)
        const double2 vw = make_double2(fma(v[q].x, w.x, -v[q].y * w.y), fma(v[q].x, w.y, v[q].y * w.x));
        v[q] = make_double2(o.x - vw.x, o.y - vw.y);
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int idx = lane * R + q;
    x[fy_swz(idx, true)] = v[q];
  }
  __syncwarp();
}

// one row's transform: the register FFT (R = m / 32 elements per lane) or, for R = 0,
// the shared-memory warp_fft; the kernels are instantiated per R so each carries only
// its own register footprint
template <int R>
__device__ __forceinline__ void row_fft(double2* x, int m, const double2* __restrict__ tw) {
  if constexpr (R == 0) {
    warp_fft(x, m, tw);
  } else {
    int lg = 0;
    while ((1 << lg) < m) ++lg;
    warp_fft_reg<R>(x, lg, tw);
  }
}

// field (r x m_y, plane-major) -> coeff (2 (m_y/2) systems x r)
template <int R>
__global__ void __launch_bounds__(FY_THREADS, R >= 16 ? 1 : 2) fourier_y_kernel(FourierArgs a, const double* __restrict__ field,
                                                               double* __restrict__ coeff) {
  extern __shared__ double2 fy_smem[];
  const int m = a.m_y, half = m / 2, T = a.tile;
  const long long i0 = static_cast<long long>(blockIdx.x) * T;
  const int nt = static_cast<int>(min(static_cast<long long>(T), a.r - i0));
#pragma unroll 8
  for (int e = threadIdx.x; e < T * m; e += FY_THREADS) {
    const int y = e / T, n = e - y * T;
    fy_smem[n * (m + 1) + y] = make_double2(n < nt ? __ldcs(field + static_cast<long long>(y) * a.r + i0 + n) : 0.0, 0.0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, nw = FY_THREADS / 32;
  for (int n = warp; n < nt; n += nw) row_fft<R>(fy_smem + n * (m + 1), m, a.tw);
  constexpr bool swz = R > 0;  // the register FFT stores its rows swizzled
  __syncthreads();
  const double inv = 1.0 / m;
  for (int e = threadIdx.x; e < 2 * half * T; e += FY_THREADS) {
    const int s = e / T, n = e - s * T, j = s >> 1;
    if (n < nt) {
      const double2 c = fy_smem[n * (m + 1) + fy_swz(j, swz)];
      coeff[static_cast<long long>(s) * a.r + i0 + n] = ((s & 1) ? c.y : c.x) * inv;
    }
  }
}

// coeff (2 (m_y/2) systems x r) -> field (r x m_y): Hermitian extension, Nyquist zero
template <int R>
__global__ void __launch_bounds__(FY_THREADS, R >= 16 ? 1 : 2) inverse_fourier_y_kernel(FourierArgs a, const double* __restrict__ coeff,
                                                                       double* __restrict__ field) {
  extern __shared__ double2 fy_smem[];
  const int m = a.m_y, half = m / 2, T = a.tile;
  const long long i0 = static_cast<long long>(blockIdx.x) * T;
  const int nt = static_cast<int>(min(static_cast<long long>(T), a.r - i0));
#pragma unroll 4
  for (int e = threadIdx.x; e < T * m; e += FY_THREADS) {
    const int y = e / T, n = e - y * T;
    double2 v = make_double2(0.0, 0.0);
    if (n < nt && y != half) {
      const int j = y < half ? y : m - y;  // row(m - j) = conj(coeff_j)
      const double re = __ldcs(coeff + static_cast<long long>(2 * j) * a.r + i0 + n);
      const double im = __ldcs(coeff + static_cast<long long>(2 * j + 1) * a.r + i0 + n);
      v = make_double2(re, y < half ? im : -im);
    }
    fy_smem[n * (m + 1) + y] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, nw = FY_THREADS / 32;
  for (int n = warp; n < nt; n += nw) row_fft<R>(fy_smem + n * (m + 1), m, a.tw);
  constexpr bool swz = R > 0;
  __syncthreads();
  for (int e = threadIdx.x; e < T * m; e += FY_THREADS) {
    const int y = e / T, n = e - y * T;
    if (n < nt) field[static_cast<long long>(y) * a.r + i0 + n] = fy_smem[n * (m + 1) + fy_swz(y, swz)].x;
  }
}

}  // namespace smpm
