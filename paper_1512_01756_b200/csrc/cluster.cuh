// Cluster-persistent Arnoldi solver (sm_100a).
//
// One launch runs the whole GMRES cycle of every live system of a batch.
// Each thread-block cluster pulls a system from a device work queue and
// iterates it until it stops (converged, breakdown, iteration cap or cycle
// end), then pulls the next one. Inside an Arnoldi step the cluster's CTAs:
//   1. split the contraction tiles of the preconditioned operator (block-
//      Jacobi stages, S) — the same per-system job templates and tile routine
//      as the per-stage kernels (gemm2.cuh);
//   2. split the Z^T interface sums; every CTA then solves the small coarse
//      system redundantly (identical arithmetic -> identical result);
//   3. own contiguous row ranges for the CGS2 passes (the deflation update P
//      is applied on the fly in pass 1) and combine per-CTA partial sums in a
//      fixed order (deterministic);
//   4. CTA 0 applies the Givens update / stop test (gmres.cpp:71-99).
// Phases are separated by hardware cluster barriers (barrier.cluster
// release/acquire) instead of kernel boundaries, and clusters that finish
// early take new systems, so a few slow systems no longer serialise the GPU.
#pragma once

#include "common.cuh"
#include "gemm2.cuh"
#include "vec.cuh"

namespace smpm {

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_nranks() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
// cluster-wide barrier with release/acquire ordering of global memory
__device__ __forceinline__ void cl_sync() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n"
      "barrier.cluster.wait.acquire.aligned;\n" ::
          : "memory");
}

struct ClusterArgs {
  // unsplit per-system job templates: 0 BJ1, 1 BJ2, 2 BJ3, 3 S
  const GemmJob* jobs[4];
  const Tile2* tiles[4];
  int ntiles[4];
  long long a_stride;
  double* vin;   // v_j (operator input)
  double* w;     // Arnoldi vector under construction
  double* u;     // M^{-1} v
  double* t;     // S M^{-1} v (dbj) / u + Z c (2las)
  double* tmp;   // block-Jacobi scratch
  double* V;
  double* part;  // per cluster: ranks x (m + 2) partial sums
  double* zsum;  // per cluster: d interface sums
  int* queue;    // next live-list slot to take
  int* publish;  // per cluster: the system it took (-1: queue empty)
  const int* alist;
  const int* acount;
  int method;    // smpm_method
  unsigned long long* trace;  // debug: per cluster, 64 steps x 12 phase timestamps (nullable)
  GmState_ G;
  DeflateParams P;
};

// run every tile of one operator stage for system s, tiles split over the cluster
__device__ __forceinline__ void cl_stage(const ClusterArgs& a, int stage, int s, const BufTable& bufs, double* smem,
                                         unsigned rank, unsigned nr) {
  const GemmJob* jobs = a.jobs[stage];
  const Tile2* tiles = a.tiles[stage];
  for (int ti = static_cast<int>(rank); ti < a.ntiles[stage]; ti += static_cast<int>(nr)) {
    const Tile2 tile = tiles[ti];
    GemmJob jb = jobs[tile.job];
    jb.A += s * a.a_stride;
    const long long vo = s * a.G.k;
    jb.b.off += vo;
    jb.out.off += vo;
    jb.add.off += vo;
    g2_run_tile(jb, tile, bufs, nullptr, smem);
  }
}

// Z^T sums of x (system s) into zsum (interfaces split over the cluster's warps)
__device__ __forceinline__ void cl_zt(const ClusterArgs& a, const double* x, double* zsum, unsigned rank,
                                      unsigned nr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int w2 = 2 * a.P.w;
  for (int i = static_cast<int>(rank) * nw + warp; i < a.P.d; i += static_cast<int>(nr) * nw) {
    const double* seg = x + static_cast<long long>(i) * w2;
    double a0 = 0.0, a1 = 0.0;
    int e = lane;
    for (; e + 32 < w2; e += 64) {
      a0 += seg[e];
      a1 += seg[e + 32];
    }
    if (e < w2) a0 += seg[e];
    const double v = warp_sum(a0 + a1);
    if (lane == 0) zsum[i] = v;
  }
}

// partial dots of this CTA's rows of V[:, 0..ncols) with x -> out[0..ncols)
__device__ __forceinline__ void cl_col_dots(const double* __restrict__ Vs, long long k, int ncols,
                                            const double* __restrict__ x, int r0, int r1, double* out,
                                            double (*red)[129]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr int GRP = 8;
  for (int c0 = 0; c0 < ncols; c0 += GRP) {
    double acc[GRP];
#pragma unroll
    for (int u = 0; u < GRP; ++u) acc[u] = 0.0;
    for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x) {
      const double xv = x[r];
#pragma unroll
      for (int u = 0; u < GRP; ++u)
        if (c0 + u < ncols) acc[u] = fma(Vs[static_cast<long long>(c0 + u) * k + r], xv, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < GRP; ++u) {
      const double v = warp_sum(acc[u]);
      if (lane == 0 && c0 + u < ncols) red[warp][c0 + u] = v;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nw; ++q) s += red[q][c];
    out[c] = s;
  }
  __syncthreads();
}

// sum of the cluster's partials (fixed rank order) -> hs[0..ncols)
__device__ __forceinline__ void cl_gather(const double* part, int stride, unsigned nr, int ncols, double* hs) {
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double s = 0.0;
    for (unsigned q = 0; q < nr; ++q) s += part[static_cast<long long>(q) * stride + c];
    hs[c] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(G2_THREADS) arnoldi_cluster_kernel(ClusterArgs a) {
  extern __shared__ __align__(16) double cl_smem[];
  double* gsmem = cl_smem;                  // G2_SMEM bytes for the tile pipeline
  double* hs = cl_smem + G2_SMEM / 8;       // 128: h1 (then h1 + h2)
  double* h2s = hs + 128;                   // 128
  double* cs_ = h2s + 128;                  // 2 d: coarse rhs / solution
  __shared__ double red[G2_THREADS / 32][129];
  __shared__ int s_sys;

  const unsigned rank = cl_rank(), nr = cl_nranks(), cid = cl_id();
  GmState_& G = a.G;
  const long long k = G.k;
  const int stride = G.m + 2;
  double* part = a.part + static_cast<long long>(cid) * nr * stride;
  double* mypart = part + static_cast<long long>(rank) * stride;
  double* zsum = a.zsum + static_cast<long long>(cid) * a.P.d;
  const int d = a.P.d, w = a.P.w, w2 = 2 * w, mx = a.P.mx;
  const long long rows_per = (k + nr - 1) / nr;
  const int r0 = static_cast<int>(min(k, rank * rows_per)), r1 = static_cast<int>(min(k, (rank + 1) * rows_per));

  for (;;) {
    // ---- take the next live system: rank 0 pops the queue and publishes the
    // system through global memory; the cluster barrier orders it
    if (rank == 0 && threadIdx.x == 0) {
      const int slot = atomicAdd(a.queue, 1);
      a.publish[cid] = slot < *a.acount ? a.alist[slot] : -1;
    }
    cl_sync();
    if (threadIdx.x == 0) s_sys = a.publish[cid];
    __syncthreads();
    const int s = s_sys;
    cl_sync();  // everyone has read the slot before rank 0 may overwrite it
    if (s < 0) return;

    const long long so = s * k;
    BufTable bufs;
    bufs.p[BUF_IN] = a.vin;
    bufs.p[BUF_OUT] = a.u;
    bufs.p[BUF_TMP] = a.tmp;
    bufs.p[BUF_TMP2] = nullptr;
    const double* Vs = a.V + s * G.vstride;
    double* ws = a.w + so;

    int step = 0;
    unsigned long long* tr = nullptr;
    auto mark = [&](int ph) {
      if (tr && threadIdx.x == 0) tr[ph] = gtimer();
    };
    while (G.state[s] == GM_RUN) {
      tr = (a.trace && rank == 0 && step < 64) ? a.trace + (static_cast<long long>(cid) * 64 + step) * 12 : nullptr;
      ++step;
      mark(0);
      const int j = G.jcyc[s];
      const int ncols = j + 1;
      // ---- operator: u = M^{-1} vin (block-Jacobi stages), then S
      if (a.method != SMPM_SCHUR) {
        cl_stage(a, 0, s, bufs, gsmem, rank, nr);
        cl_sync();
        mark(1);
        cl_stage(a, 1, s, bufs, gsmem, rank, nr);
        cl_sync();
        mark(2);
        cl_stage(a, 2, s, bufs, gsmem, rank, nr);
        cl_sync();
        mark(3);
      }
      const double* sin = a.method == SMPM_SCHUR ? a.vin : a.u;
      if (a.method == SMPM_2LAS) {
        // minv = M^{-1} v + Z C^{-1} Z^T v : t = u + Z c(Z^T vin)
        cl_zt(a, a.vin + so, zsum, rank, nr);
        cl_sync();
        for (int i = threadIdx.x; i < d; i += blockDim.x) cs_[i] = zsum[i];
        __syncthreads();
        coarse_solve_block(a.P, s, cs_, cs_ + d);
        for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x)
          a.t[so + r] = a.u[so + r] + cs_[d + r / w2];
        cl_sync();
        sin = a.t;
      }
      BufTable sb;
      sb.p[BUF_IN] = const_cast<double*>(sin);
      // dbj: S writes t and the fused P produces w in pass 1; otherwise S writes w
      sb.p[BUF_OUT] = a.method == SMPM_DBJ ? a.t : a.w;
      sb.p[BUF_TMP] = nullptr;
      sb.p[BUF_TMP2] = nullptr;
      cl_stage(a, 3, s, sb, gsmem, rank, nr);
      cl_sync();
      mark(4);
      if (a.method == SMPM_DBJ) {
        // ---- fused deflation P: c = C^{-1} Z^T t ; w = t - Z c - (S - I) Z c
        cl_zt(a, a.t + so, zsum, rank, nr);
        cl_sync();
        for (int i = threadIdx.x; i < d; i += blockDim.x) cs_[i] = zsum[i];
        __syncthreads();
        coarse_solve_block(a.P, s, cs_, cs_ + d);
        const double* c = cs_ + d;
        const double* rs = a.P.rowsum + static_cast<long long>(s) * 6 * w;
        const double *rWI = rs, *rEI = rs + w2, *rEW = rs + 2 * w2, *rWE = rEW + w;
        const double* ts = a.t + so;
        for (int e = r0 + static_cast<int>(threadIdx.x); e < r1; e += blockDim.x) {
          const int blk = e / w, r = e - blk * w, i = blk >> 1;
          double sz;
          if ((blk & 1) == 0)
            sz = (i + 1 == mx - 1) ? c[i] * rWE[r] : c[i] * rWI[r] + c[i + 1] * rEI[r];
          else
            sz = (i == 0) ? c[i] * rEW[r] : c[i - 1] * rWI[w + r] + c[i] * rEI[w + r];
          ws[e] = ts[e] - (c[i] + sz);
        }
        __syncthreads();
        mark(5);
      }
      // ---- CGS2 pass 1: h1 = V^T w (own rows, then fixed-order combine)
      cl_col_dots(Vs, k, ncols, ws, r0, r1, mypart, red);
      cl_sync();
      cl_gather(part, stride, nr, ncols, hs);
      cl_sync();  // partials consumed before pass 2 overwrites them
      mark(6);
      // ---- pass 2: w -= V h1 ; h2 = V^T w
      for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x) {
        double a1 = 0.0, a2 = 0.0;
        int i = 0;
        for (; i + 2 <= ncols; i += 2) {
          a1 = fma(Vs[static_cast<long long>(i) * k + r], hs[i], a1);
          a2 = fma(Vs[static_cast<long long>(i + 1) * k + r], hs[i + 1], a2);
        }
        if (i < ncols) a1 = fma(Vs[static_cast<long long>(i) * k + r], hs[i], a1);
        ws[r] -= a1 + a2;
      }
      __syncthreads();
      cl_col_dots(Vs, k, ncols, ws, r0, r1, mypart, red);
      cl_sync();
      cl_gather(part, stride, nr, ncols, h2s);
      cl_sync();
      mark(7);
      // ---- pass 3: w -= V h2 ; ||w||
      double sq = 0.0;
      for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x) {
        double a1 = 0.0, a2 = 0.0;
        int i = 0;
        for (; i + 2 <= ncols; i += 2) {
          a1 = fma(Vs[static_cast<long long>(i) * k + r], h2s[i], a1);
          a2 = fma(Vs[static_cast<long long>(i + 1) * k + r], h2s[i + 1], a2);
        }
        if (i < ncols) a1 = fma(Vs[static_cast<long long>(i) * k + r], h2s[i], a1);
        const double v = ws[r] - (a1 + a2);
        ws[r] = v;
        sq = fma(v, v, sq);
      }
      sq = warp_sum(sq);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = sq;
      __syncthreads();
      if (threadIdx.x == 0) {
        double tsum = 0.0;
        for (int q = 0; q < G2_THREADS / 32; ++q) tsum += red[q][0];
        mypart[0] = tsum;
      }
      cl_sync();
      mark(8);
      double nsq = 0.0;
      for (unsigned q = 0; q < nr; ++q) nsq += part[static_cast<long long>(q) * stride];
      const double nrm = sqrt(nsq);
      // ---- Givens / stop test on CTA 0 (writes the system's global state)
      if (rank == 0) {
        double* gh1 = G.h1 + static_cast<long long>(s) * stride;
        double* gh2 = G.h2 + static_cast<long long>(s) * stride;
        for (int i = threadIdx.x; i < ncols; i += blockDim.x) {
          gh1[i] = hs[i];
          gh2[i] = h2s[i];
        }
        __syncthreads();
        if (threadIdx.x < 32) givens_step(G, s, j, nrm);
      }
      // ---- v_{j+1} = w / ||w|| (own rows; unused if the system stops)
      const double inv = 1.0 / nrm;
      double* col = a.V + s * G.vstride + static_cast<long long>(j + 1) * k;
      if (j + 1 <= G.m)
        for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x) {
          const double v = ws[r] * inv;
          col[r] = v;
          a.vin[so + r] = v;
        }
      cl_sync();  // state, jcyc and v_{j+1} visible cluster-wide
      mark(9);
      if (tr && threadIdx.x == 0) tr[10] = static_cast<unsigned long long>(s) | (static_cast<unsigned long long>(j) << 32);
    }
  }
}

}  // namespace smpm
