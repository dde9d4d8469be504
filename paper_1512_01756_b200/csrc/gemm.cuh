// Grouped fp64 GEMM over precomputed job/tile lists (sm_100a).
//
// Every dense contraction of the hot path is one of these jobs: the Schur
// apply S v = v + permute(G_I X) (+ the two boundary-strip blocks), its
// transpose, the three stages of the structured block-Jacobi apply, and the
// setup-time products. One launch covers all jobs of all systems in a batch.
//
// fp64 has no tcgen05 kind on sm_100a, so the contraction runs on the FP64
// FMA pipe: 128x32 output tile per CTA, 16-deep K slices double-buffered
// through shared memory with register prefetch, each thread an 8x4 register
// tile laid out so every warp-wide LDS.128 is one conflict-free wavefront
// (FMA-bound, not shared-memory-bound). Small-N / small-tile-count problems
// (the 2D systems) split K across CTAs and finish in a deterministic
// fixed-order reduction kernel.
#pragma once

#include "common.cuh"

namespace smpm {

// thread layout: tx in [0,8) along N, ty in [0,16) along M
// rows owned: m = 32*q + 2*ty + e  (q<4, e<2); cols: n = 16*h + 2*tx + f (h<2, f<2)
__device__ __forceinline__ int gemm_row(int ty, int i) { return 32 * (i >> 1) + 2 * ty + (i & 1); }
__device__ __forceinline__ int gemm_col(int tx, int j) { return 16 * (j >> 1) + 2 * tx + (j & 1); }

__global__ void __launch_bounds__(128, 3)
gemm_jobs_kernel(const GemmJob* __restrict__ jobs, const GemmTile* __restrict__ tiles, BufTable bufs,
                 const int* __restrict__ active, double* __restrict__ ws) {
  constexpr int BM = GEMM_BM, BN = GEMM_BN, BK = GEMM_BK;
  __shared__ __align__(16) double As[2][BK][BM];
  __shared__ __align__(16) double Bs[2][BK][BN];

  const GemmTile tile = tiles[blockIdx.x];
  const GemmJob& jb = jobs[tile.job];
  if (active && !active[jb.sys]) return;

  const int t = threadIdx.x;
  const int tx = t & 7, ty = t >> 3;
  const int M = jb.M, N = jb.N, K = jb.K;
  const int m0 = tile.m0, n0 = tile.n0;

  int kb = 0, ke = K;
  if (jb.splitk > 1) {
    const int kc = ((K + jb.splitk * BK - 1) / (jb.splitk * BK)) * BK;
    kb = tile.ks * kc;
    ke = min(K, kb + kc);
  }

  const double* __restrict__ A = jb.A;
  const long long lda = jb.lda;
  const double* __restrict__ Bbuf = bufs.p[jb.b.buf];

  double ra[BK];  // A prefetch: this thread's row (non-trans: row t; trans: row t too)
  double rb[4];

  auto load_tile = [&](int k0) {
    const int m = m0 + t;
    if (!jb.transA) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const int k = k0 + kk;
        ra[kk] = (m < M && k < ke) ? __ldg(A + static_cast<long long>(k) * lda + m) : 0.0;
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const int k = k0 + kk;
        ra[kk] = (m < M && k < ke) ? __ldg(A + static_cast<long long>(m) * lda + k) : 0.0;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = t + 128 * e;
      const int c = idx >> 4, kk = idx & 15;
      const int k = k0 + kk, n = n0 + c;
      rb[e] = (n < N && k < ke) ? Bbuf[jb.b.at(k, n)] : 0.0;
    }
  };
  auto store_tile = [&](int s) {
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) As[s][kk][t] = ra[kk];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = t + 128 * e;
      Bs[s][idx & 15][idx >> 4] = rb[e];
    }
  };

  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  int stage = 0;
  if (kb < ke) {
    load_tile(kb);
    store_tile(0);
  }
  __syncthreads();
  for (int k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load_tile(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[8], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = *reinterpret_cast<const double2*>(&As[stage][kk][32 * q + 2 * ty]);
        a[2 * q] = v.x;
        a[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 v = *reinterpret_cast<const double2*>(&Bs[stage][kk][16 * h + 2 * tx]);
        b[2 * h] = v.x;
        b[2 * h + 1] = v.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_tile(stage ^ 1);
      __syncthreads();
      stage ^= 1;
    }
  }

  if (jb.splitk > 1) {
    // raw partial tile -> workspace [tile][BM][BN]; reduced in fixed K order later
    const int ntn = (N + BN - 1) / BN;
    const long long slot =
        static_cast<long long>(jb.ws_off) + (static_cast<long long>(m0 / BM) * ntn + n0 / BN) * jb.splitk + tile.ks;
    double* w = ws + slot * (BM * BN);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) w[gemm_row(ty, i) * BN + gemm_col(tx, j)] = acc[i][j];
    return;
  }

  double* __restrict__ out = bufs.p[jb.out.buf];
  const double* __restrict__ add = jb.add.buf == BUF_NONE ? nullptr : bufs.p[jb.add.buf];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + gemm_row(ty, i);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + gemm_col(tx, j);
      if (n >= N) continue;
      double v = jb.alpha * acc[i][j];
      if (add) v = fma(jb.beta, add[jb.add.at(m, n)], v);
      out[jb.out.at(m, n)] = v;
    }
  }
}

// Reduction of split-K partial tiles (fixed K order => deterministic) + epilogue.
struct SplitItem {
  int job;
  int m0, n0;
};

__global__ void __launch_bounds__(256)
gemm_splitk_reduce_kernel(const GemmJob* __restrict__ jobs, const SplitItem* __restrict__ items, BufTable bufs,
                          const int* __restrict__ active, const double* __restrict__ ws) {
  constexpr int BM = GEMM_BM, BN = GEMM_BN;
  const SplitItem it = items[blockIdx.x];
  const GemmJob& jb = jobs[it.job];
  if (active && !active[jb.sys]) return;
  const int ntn = (jb.N + BN - 1) / BN;
  const long long slot0 =
      static_cast<long long>(jb.ws_off) + (static_cast<long long>(it.m0 / BM) * ntn + it.n0 / BN) * jb.splitk;
  double* __restrict__ out = bufs.p[jb.out.buf];
  const double* __restrict__ add = jb.add.buf == BUF_NONE ? nullptr : bufs.p[jb.add.buf];
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const int r = e / BN, c = e % BN;
    const int m = it.m0 + r, n = it.n0 + c;
    if (m >= jb.M || n >= jb.N) continue;
    double s = 0.0;
    for (int ks = 0; ks < jb.splitk; ++ks) s += ws[(slot0 + ks) * (BM * BN) + e];
    double v = jb.alpha * s;
    if (add) v = fma(jb.beta, add[jb.add.at(m, n)], v);
    out[jb.out.at(m, n)] = v;
  }
}

}  // namespace smpm
