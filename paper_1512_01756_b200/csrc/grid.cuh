// Grid-persistent Arnoldi tail solver (sm_100a).
//
// When only a few systems of a batch are still iterating, every per-stage
// kernel of an Arnoldi step is a few microseconds of launch + fill + drain
// around almost no work, and the step becomes a chain of ~13 latency-bound
// launches.  This kernel runs ALL remaining Arnoldi steps of the live
// systems of one GMRES cycle in a single launch that covers the whole GPU
// (every SM, several CTAs each, grouped in thread-block clusters of GT_CL):
//   * operator stages (block-Jacobi 1..3, S) use the per-system tile
//     templates of the per-stage kernels (gemm2.cuh).  With few live systems
//     every 64x32 output tile is split over the K dimension across the CTAs
//     of one cluster, and the partial tiles are summed through distributed
//     shared memory in fixed rank order (no workspace, no atomics); GEMV
//     tiles run on the CTAs of the remaining clusters.  With many live
//     systems each CTA takes whole tiles;
//   * Z^T interface sums: one warp per (system, interface) over the grid;
//   * CGS2 passes: the clusters are partitioned into one contiguous group per
//     live system, each CTA owns a row range of its system; per-CTA partial
//     dots are summed inside the cluster through DSMEM, then every CTA of the
//     group sums the group's cluster partials in the same fixed order
//     (deterministic, identical in all CTAs, no atomics on data);
//   * the group leader applies the Givens update / stop test
//     (/root/reference/proj/src/gmres.cpp:71-99) through givens_step.
// Phases are separated by a two-level grid barrier: a hardware cluster
// barrier, then one release/acquire counter per cluster leader.  All CTAs
// are co-resident (cooperative launch, or a grid sized by the occupancy
// calculator); the spin has a bound and traps instead of hanging.
// Data produced inside the launch is read with ld.global.cg (L2) so no SM
// can hit a stale L1 line.
#pragma once

#include "common.cuh"
#include "gemm2.cuh"
#include "vec.cuh"
#include "spectral.cuh"

namespace smpm {

constexpr int GT_MAXSYS = 32;   // live systems one tail launch may carry
constexpr int GT_MAXCOL = 128;  // cycle length + 2
constexpr int GT_CL = 8;        // CTAs per cluster (= K splits of a tail tile)
constexpr int GT_GVR = 32;      // rows of a cluster GEMV item
#ifndef GT_STAGES_DEF
#define GT_STAGES_DEF 2
#endif
#ifndef GT_MINB
#define GT_MINB 1
#endif
constexpr int GT_STAGES = GT_STAGES_DEF;  // cp.async ring depth of the operator tiles
constexpr int GT_SMEM =
    GT_STAGES * (G2_BK * (G2_BM + G2_APAD) + G2_BN * (G2_BK + G2_BPAD)) * static_cast<int>(sizeof(double));
static_assert(GT_SMEM >= G2_BM * G2_BN * static_cast<int>(sizeof(double)), "tile partial must fit the ring");

struct GridArgs {
  // unsplit per-system templates of the operator stages: BJ1 BJ2 BJ3 S, and
  // the spectral transforms F (T^{-1}) and B (T) (tiles sorted GEMM first, then GEMV)
  const GemmJob* jobs[6];
  int njobs[6];
  const Tile2* tiles[6];
  int ntiles[6];
  int ngemm[6];            // GEMM tiles (the rest are GEMV tiles)
  const Tile2* gv[6];      // GEMV jobs as GT_GVR-row cluster items (ks = -1)
  int ngv[6];
  long long a_stride[6];   // matrix stride per system (0: shared matrix)
  int spectral;            // operator through the spectral form (spectral.cuh)
  SpecParams sp;
  double* vh;              // T^{-1} vin
  double* th;              // S^ M^^{-1} vh
  double* zp;              // GT_MAXSYS x sp.nmc x d: Z^T partial sums per mode chunk
  double* cg;              // GT_MAXSYS x d: coarse solutions c = C^{-1} Z^T t per live slot
  double* vin;             // v_j (operator input)
  double* w;               // Arnoldi vector under construction
  double* u;               // M^{-1} v
  double* t;               // S M^{-1} v (dbj) / u + Z c (2las)
  double* tmp;             // block-Jacobi scratch
  double* V;               // Krylov bases
  double* part;            // 3 x nclusters x (m + 2) cluster partial sums (h1, h2, ||w||^2)
  double* zsum;            // GT_MAXSYS x d interface sums
  unsigned* bar;           // grid barrier arrival counter (zeroed before the launch)
  const int* alist;        // candidate systems (compacted live list)
  const int* acount;
  int method;              // smpm_method
  int pythag;              // ||w|| from the second CGS2 reduction (as cgs3_pass2n)
  int defer;               // spectral + pythag: the next step's T^{-1} runs on w' (before the reorthogonalisation
                           // update, vec4.cuh), so pass 3 and that transform share one barrier interval
  int vcap;                // doubles of the tile-ring region (>= GT_SMEM / 8); with pythag, a CTA whose
                           // V rows (ncols x rows) fit there stages them once per step (gt_vblock)
  unsigned long long* trace;  // debug: 64 steps x 16 phase timestamps of CTA 0 (nullable)
  unsigned long long* trace2; // debug: 4 steps x 4 stages x gridDim.x x 8 per-CTA timestamps (nullable)
  GmState_ G;
  DeflateParams P;
};

__device__ __forceinline__ unsigned long long gt_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned gt_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void gt_cl_sync() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n"
      "barrier.cluster.wait.acquire.aligned;\n" ::
          : "memory");
}
// address of `p` (this CTA's shared memory) in the shared memory of cluster rank `r`
__device__ __forceinline__ unsigned gt_map(const void* p, unsigned r) {
  const unsigned l = static_cast<unsigned>(__cvta_generic_to_shared(p));
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(l), "r"(r));
  return o;
}
__device__ __forceinline__ double gt_ld_dsmem(unsigned addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

// all CTAs of the grid: everything written before is visible to everyone after
// (one release/acquire counter; measured ~1.1 us for 296 CTAs, cheaper than
// a cluster-then-leader hierarchy)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  epoch += gridDim.x;
  if (threadIdx.x == 0) {
    unsigned v;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(v) : "l"(bar) : "memory");
    ++v;
    long long spins = 0;
    while (v < epoch) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (++spins > (1LL << 26)) asm volatile("trap;");  // never hang the GPU
    }
  }
  __syncthreads();
}

// element (i, j, e) of a thread's 64x32 accumulator fragment inside the tile
__device__ __forceinline__ void gt_frag_rc(int q, int& r, int& c) {
  const int i = q >> 2, j = (q >> 1) & 1, e = q & 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wm = warp >> 1, wn = warp & 1;
  r = wm * 32 + i * 8 + (lane >> 2);
  c = wn * 16 + j * 8 + (lane & 3) * 2 + e;
}

// One 64x32 output tile split over K across SP consecutive CTAs of this
// cluster (ranks base..base+SP-1; sub-rank q computes K chunk q); the
// partials meet in distributed shared memory and sub-rank r sums rows
// [r*64/SP, (r+1)*64/SP) in sub-rank order.  Every CTA of the cluster calls
// this the same number of times (valid = false: barriers only).
template <int SP>
// tail_sync = false skips the trailing cluster barrier: allowed for a stage's last
// round, because every caller passes a grid barrier before the ring is reused (and a
// rank's DSMEM reads have completed before it arrives there)
__device__ __forceinline__ void gt_cluster_tile(GemmJob jb, Tile2 tile, const BufTable& bufs, double* smem,
                                                unsigned base, unsigned srank, bool valid, unsigned long long* t2,
                                                bool tail_sync) {
  __syncthreads();  // ring may still be read by this CTA's previous tile
  if (valid) {
    jb.splitk = SP;
    tile.ks = static_cast<int>(srank);
    double acc[4][2][2];
    g2_mainloop<GT_STAGES>(jb, tile, bufs, smem, acc);
    __syncthreads();  // every warp is done with the ring
    if (t2 && threadIdx.x == 0) t2[1] = gt_timer();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int r, c;
      gt_frag_rc(q, r, c);
      smem[r * G2_BN + c] = acc[q >> 2][(q >> 1) & 1][q & 1];
    }
  }
  gt_cl_sync();
  if (valid) {
    constexpr int RPR = G2_BM / SP;  // rows per sub-rank
    for (int e = threadIdx.x; e < RPR * G2_BN; e += blockDim.x) {
      const int r = static_cast<int>(srank) * RPR + e / G2_BN, c = e % G2_BN;
      const int m = tile.m0 + r, n = tile.n0 + c;
      if (m >= jb.M || n >= jb.N) continue;
      double v[SP];
#pragma unroll
      for (int q = 0; q < SP; ++q) v[q] = gt_ld_dsmem(gt_map(smem + r * G2_BN + c, base + q));
      double sum = 0.0;
#pragma unroll
      for (int q = 0; q < SP; ++q) sum += v[q];
      store_out(jb, bufs, m, n, sum);
    }
    if (t2 && threadIdx.x == 0) t2[2] = gt_timer();
  }
  if (tail_sync) gt_cl_sync();  // partials consumed before any rank reuses its ring
  if (valid && t2 && threadIdx.x == 0) t2[3] = gt_timer();
}

// stage descriptors (tiles, jobs, GEMV items): copied to shared memory at the kernel
// start when they are few (the spectral transforms: one job, 12 tiles), so a stage's
// data loads are not behind two dependent L2 round trips for its descriptors
constexpr int GT_TC = 96, GT_JC = 8, GT_GC = 32;
struct GtDesc {
  const Tile2* tiles[6];
  const GemmJob* jobs[6];
  const Tile2* gv[6];
};

__device__ __forceinline__ void gt_desc_init(const GridArgs& a, GtDesc& D, Tile2* tc, GemmJob* jc, Tile2* gc) {
  if (threadIdx.x == 0) {
    int nt = 0, nj = 0, ng = 0;
    for (int st = 0; st < 6; ++st) {
      D.tiles[st] = a.tiles[st];
      D.jobs[st] = a.jobs[st];
      D.gv[st] = a.gv[st];
      if (!a.jobs[st]) continue;
      if (a.njobs[st] > 0 && nt + a.ntiles[st] <= GT_TC && nj + a.njobs[st] <= GT_JC && ng + a.ngv[st] <= GT_GC) {
        D.tiles[st] = tc + nt;
        D.jobs[st] = jc + nj;
        D.gv[st] = gc + ng;
        nt += a.ntiles[st];
        nj += a.njobs[st];
        ng += a.ngv[st];
      }
    }
  }
  __syncthreads();
  for (int st = 0; st < 6; ++st) {
    if (!a.jobs[st] || D.jobs[st] == a.jobs[st]) continue;
    for (int i = threadIdx.x; i < a.ntiles[st]; i += blockDim.x) const_cast<Tile2*>(D.tiles[st])[i] = a.tiles[st][i];
    for (int i = threadIdx.x; i < a.ngv[st]; i += blockDim.x) const_cast<Tile2*>(D.gv[st])[i] = a.gv[st][i];
    for (int i = threadIdx.x; i < a.njobs[st]; i += blockDim.x) const_cast<GemmJob*>(D.jobs[st])[i] = a.jobs[st][i];
  }
  __syncthreads();
}

__device__ __forceinline__ GemmJob gt_job(const GridArgs& a, const GtDesc& D, int stage, const Tile2& tile, int s) {
  GemmJob jb = D.jobs[stage][tile.job];
  jb.A += s * a.a_stride[stage];
  const long long vo = s * a.G.k;
  jb.b.off += vo;
  jb.out.off += vo;
  jb.add.off += vo;
  jb.sys = s;
  return jb;
}

// One GT_GVR-row block of a GEMV job (N == 1) split over K across SP
// consecutive CTAs of the cluster: sub-rank q sums K chunk q (32 rows x 4
// k-groups, rounds of 16 independent loads), the partial columns meet in
// DSMEM, sub-rank r finishes rows [r*GT_GVR/SP, (r+1)*GT_GVR/SP) in order.
template <int SP>
__device__ __forceinline__ void gt_cluster_gemv(const GemmJob& jb, const Tile2& tile, const BufTable& bufs,
                                                double* smem, unsigned base, unsigned srank, bool valid, bool tail_sync) {
  constexpr int KG = G2_THREADS / GT_GVR;  // 4 k-groups
  constexpr int UNR = 16;
  const int t = threadIdx.x, r = t % GT_GVR, kg = t / GT_GVR;
  double* red = smem;                 // KG x GT_GVR
  double* colp = smem + KG * GT_GVR;  // GT_GVR: this CTA's partial column
  __syncthreads();  // ring / partial buffer may still be read by a previous item
  if (valid) {
    const int m = tile.m0 + r;
    const int kc = (jb.K + SP - 1) / SP;
    const int kb = static_cast<int>(srank) * kc, ke = min(jb.K, kb + kc);
    const double* x = bufs.p[jb.b.buf] + jb.b.off;
    double acc[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc[u] = 0.0;
    if (m < jb.M) {
      const double* __restrict__ A = jb.A + m;
      for (int k0 = kb + kg; k0 < ke; k0 += UNR * KG) {
        double av[UNR], xv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int k = k0 + u * KG;
          av[u] = k < ke ? __ldg(A + static_cast<long long>(k) * jb.lda) : 0.0;
          xv[u] = k < ke ? __ldcg(x + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc[u] = fma(av[u], xv[u], acc[u]);
      }
    }
    double v = 0.0;
#pragma unroll
    for (int u = 0; u < UNR; ++u) v += acc[u];
    red[kg * GT_GVR + r] = v;
    __syncthreads();
    if (t < GT_GVR) {
      double p = 0.0;
#pragma unroll
      for (int q = 0; q < KG; ++q) p += red[q * GT_GVR + t];
      colp[t] = p;
    }
  }
  gt_cl_sync();
  constexpr int RPR = GT_GVR / SP;
  if (valid && t < RPR) {
    const int rr = static_cast<int>(srank) * RPR + t, mm = tile.m0 + rr;
    if (mm < jb.M) {
      double v[SP];
#pragma unroll
      for (int q = 0; q < SP; ++q) v[q] = gt_ld_dsmem(gt_map(colp + rr, base + q));
      double sum = 0.0;
#pragma unroll
      for (int q = 0; q < SP; ++q) sum += v[q];
      store_out(jb, bufs, mm, 0, sum);
    }
  }
  if (tail_sync) gt_cl_sync();
}

// cluster items of one stage, SP CTAs per item, GT_CL / SP items per cluster
// at a time; the round count is uniform over each cluster
template <int SP>
__device__ __forceinline__ void gt_stage_split(const GridArgs& a, const GtDesc& D, int stage, const int* sl, int L,
                                               const BufTable& bufs, double* smem, unsigned long long* t2, bool rev) {
  const int ng = a.ngemm[stage], nci = ng + a.ngv[stage], items = L * nci;
  constexpr int PER = GT_CL / SP;
  const int ncl = gridDim.x / GT_CL, cid = blockIdx.x / GT_CL, nsub = ncl * PER;
  const unsigned rank = gt_rank(), sc = rank / SP, srank = rank % SP, base = sc * SP;
  // rev: items from the last cluster down (keeps them off the group leaders)
  const int gsub = (rev ? ncl - 1 - cid : cid) * PER + static_cast<int>(sc);
  const int rounds = (items + nsub - 1) / nsub;
  for (int rd = 0; rd < rounds; ++rd) {
    const int it = rd * nsub + gsub;
    const bool valid = it < items;
    const int s = valid ? sl[it / nci] : sl[0], r = valid ? it % nci : 0;
    // the item kind may differ between the sub-clusters of one cluster: both
    // kinds pass the same cluster barriers (two, one in the last round)
    const bool more = rd + 1 < rounds;
    if (r < ng) {
      const Tile2 tile = D.tiles[stage][r];
      gt_cluster_tile<SP>(gt_job(a, D, stage, tile, s), tile, bufs, smem, base, srank, valid, t2, more);
    } else {
      const Tile2 tile = D.gv[stage][r - ng];
      if (valid && t2 && threadIdx.x == 0) t2[4] = gt_timer();
      gt_cluster_gemv<SP>(gt_job(a, D, stage, tile, s), tile, bufs, smem, base, srank, valid, more);
      if (valid && t2 && threadIdx.x == 0) t2[5] = gt_timer();
    }
  }
}

// one operator stage for the live systems sl[0..L)
__device__ __forceinline__ void gt_stage(const GridArgs& a, const GtDesc& D, int stage, const int* sl, int L, const BufTable& bufs,
                                         double* smem, unsigned long long* t2, bool rev = false) {
  if (t2 && threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) t2[i] = 0;
    t2[0] = gt_timer();
  }
  const int nt = a.ntiles[stage], nci = a.ngemm[stage] + a.ngv[stage];
  const Tile2* tiles = D.tiles[stage];
  const int NB = gridDim.x, bid = blockIdx.x, ncl = NB / GT_CL;
  // split each tile over as many CTAs as the live systems leave room for
  const int items = L * nci;
  if (items <= ncl) return gt_stage_split<GT_CL>(a, D, stage, sl, L, bufs, smem, t2, rev);
  if (items <= 2 * ncl) return gt_stage_split<GT_CL / 2>(a, D, stage, sl, L, bufs, smem, t2, rev);
  if (items <= 4 * ncl) return gt_stage_split<GT_CL / 4>(a, D, stage, sl, L, bufs, smem, t2, rev);
  // many systems: whole tiles per CTA
  for (int it = bid; it < L * nt; it += NB) {
    const Tile2 tile = tiles[it % nt];
    const GemmJob jb = gt_job(a, D, stage, tile, sl[it / nt]);
    __syncthreads();
    if (tile.ks < 0) {
      g2_gemv_tile<16>(jb, tile, bufs);
      continue;
    }
    double acc[4][2][2];
    g2_mainloop<GT_STAGES>(jb, tile, bufs, smem, acc);
    g2_store_tile(jb, tile, bufs, acc);
  }
}

// Z^T sums of x for every live system: one warp per (slot, interface)
__device__ __forceinline__ void gt_zt(const GridArgs& a, const double* x, const int* sl, int L) {
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + (threadIdx.x >> 5), tw = gridDim.x * nw;
  const int d = a.P.d, w2 = 2 * a.P.w;
  for (int p = gw; p < L * d; p += tw) {
    const int q = p / d, i = p - q * d;
    const double* seg = x + sl[q] * a.G.k + static_cast<long long>(i) * w2;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    for (int e0 = lane; e0 < w2; e0 += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 32;
        if (e < w2) acc[u] += __ldcg(seg + e);
      }
    }
    const double v = warp_sum(((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7])));
    if (lane == 0) a.zsum[static_cast<long long>(q) * d + i] = v;
  }
}

// this CTA's partial dots of V_s[:, 0..ncols) with x over rows [r0, r1) -> out
// (shared memory).  Warps take groups of 8 columns; when there are fewer
// column groups than warps the rows are split between warps too, and the
// row-group partials are summed in fixed order.  Lanes run over rows, 2 rows
// per round: up to 18 independent loads in flight per lane.
__device__ __forceinline__ void gt_col_dots(const double* Vs, long long k, int ncols, const double* x, int r0, int r1,
                                            double* out) {
  constexpr int NW = G2_THREADS / 32;
  __shared__ double rgp[NW][GT_MAXCOL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncg = (ncols + 7) >> 3;
  const int nrg = ncg >= NW ? 1 : NW / ncg;
  const int rg = ncg >= NW ? 0 : warp / ncg;
  const int cg0 = ncg >= NW ? warp : warp % ncg, cgs = ncg >= NW ? NW : ncg;
  if (rg < nrg) {
    for (int cg = cg0; cg < ncg; cg += cgs) {
      const int c0 = cg * 8;
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = 0.0;
      for (int r = r0 + rg * 32 + lane; r < r1; r += 2 * 32 * nrg) {
        const int r2 = r + 32 * nrg;
        const bool two = r2 < r1;
        const double x0 = __ldcg(x + r), x1 = two ? __ldcg(x + r2) : 0.0;
        double v0[8], v1[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double* col = Vs + static_cast<long long>(min(c0 + u, ncols - 1)) * k;
          v0[u] = __ldcg(col + r);
          v1[u] = two ? __ldcg(col + r2) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = fma(v1[u], x1, fma(v0[u], x0, acc[u]));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double v = warp_sum(acc[u]);
        if (lane == 0 && c0 + u < ncols) rgp[rg][c0 + u] = v;
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double sum = 0.0;
    for (int q = 0; q < nrg; ++q) sum += rgp[q][c];
    out[c] = sum;
  }
  __syncthreads();
}

// w[r] -= sum_i V[r, i] h[i] for this CTA's rows (16 independent loads per
// round); returns the sum of squares of the updated rows
__device__ __forceinline__ double gt_update(const double* Vs, long long k, int ncols, const double* h, double* ws,
                                            int r0, int r1) {
  double sq = 0.0;
  for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x) {
    double a4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i0 = 0; i0 < ncols; i0 += 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = i0 + u < ncols ? __ldcg(Vs + static_cast<long long>(i0 + u) * k + r) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) a4[u & 3] = fma(v[u], i0 + u < ncols ? h[i0 + u] : 0.0, a4[u & 3]);
    }
    const double nv = __ldcg(ws + r) - ((a4[0] + a4[1]) + (a4[2] + a4[3]));
    ws[r] = nv;
    sq = fma(nv, nv, sq);
  }
  return sq;
}

// pass 3 with the norm known: w -= V h for this CTA's rows, then
// v_{j+1} = w * inv into the basis column and the operator input (when col != nullptr)
__device__ __forceinline__ void gt_update_scale(const double* Vs, long long k, int ncols, const double* h, double* ws,
                                                int r0, int r1, double inv, double* col, double* vin,
                                                bool store_w = true) {
  for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x) {
    double a4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i0 = 0; i0 < ncols; i0 += 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = i0 + u < ncols ? __ldcg(Vs + static_cast<long long>(i0 + u) * k + r) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) a4[u & 3] = fma(v[u], i0 + u < ncols ? h[i0 + u] : 0.0, a4[u & 3]);
    }
    const double nv = __ldcg(ws + r) - ((a4[0] + a4[1]) + (a4[2] + a4[3]));
    if (store_w) ws[r] = nv;
    if (col) {
      col[r] = nv * inv;
      vin[r] = nv * inv;
    }
  }
}

// ---- CGS2 on a shared-memory copy of this CTA's rows of V (one async load per step) ----
// vb: ncols x nr column-major (rows r0.., nr even), wb: nr rows of w

// issue the 16-byte async copies of V[r0:r0+nr, 0:ncols) (k and r0 even: aligned pairs)
__device__ __forceinline__ void gt_vblock_load(const double* Vs, long long k, int ncols, int r0, int nr, double* vb) {
  const int np = nr >> 1, tot = ncols * np;
  if (np > 0) {
    int c = static_cast<int>(threadIdx.x) / np, p = static_cast<int>(threadIdx.x) - c * np;
    const int dc = static_cast<int>(blockDim.x) / np, dp = static_cast<int>(blockDim.x) - dc * np;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      cp_async16(vb + c * nr + 2 * p, Vs + static_cast<long long>(c) * k + r0 + 2 * p, true);
      c += dc;
      p += dp;
      if (p >= np) {
        p -= np;
        ++c;
      }
    }
  }
  cp_async_commit();
}

// out[c] = sum_r vb[c, r] wb[r]: each warp takes groups of 4 columns, lanes run over rows
__device__ __forceinline__ void gt_vblock_dots(const double* vb, const double* wb, int nr, int ncols, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c0 = warp * 4; c0 < ncols; c0 += nw * 4) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int nc = min(4, ncols - c0);
    for (int r = lane; r < nr; r += 32) {
      const double x = wb[r];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < nc) acc[u] = fma(vb[(c0 + u) * nr + r], x, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = warp_sum(acc[u]);
    if (lane < nc) {
      const double v = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
      out[c0 + lane] = v;
    }
  }
}

// (V h)[r] for row r of the block (4 independent chains)
__device__ __forceinline__ double gt_vblock_row(const double* vb, int nr, int ncols, const double* h, int r) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int c = 0;
  for (; c + 4 <= ncols; c += 4) {
    a0 = fma(vb[c * nr + r], h[c], a0);
    a1 = fma(vb[(c + 1) * nr + r], h[c + 1], a1);
    a2 = fma(vb[(c + 2) * nr + r], h[c + 2], a2);
    a3 = fma(vb[(c + 3) * nr + r], h[c + 3], a3);
  }
  for (; c < ncols; ++c) a0 = fma(vb[c * nr + r], h[c], a0);
  return (a0 + a1) + (a2 + a3);
}

// sum of the cluster's CTA partials pin[0..n) (rank order, through DSMEM) ->
// gout[0..n) (this cluster's slot of a global partial buffer); ranks split the entries
__device__ __forceinline__ void gt_cluster_sum(const double* pin, int n, double* gout) {
  gt_cl_sync();
  const unsigned rank = gt_rank();
  for (int c = static_cast<int>(rank) * blockDim.x + threadIdx.x; c < n; c += GT_CL * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < GT_CL; ++q) s += gt_ld_dsmem(gt_map(pin + c, q));
    gout[c] = s;
  }
}

// every CTA of a group: sum of the group's cluster partials (fixed order,
// 16 independent loads per round: one or two L2 round trips for any group) -> dst[0..n)
__device__ __forceinline__ void gt_group_sum(const double* part, int stride, int c0, int c1, int n, double* dst) {
  constexpr int R = 16;
  if (2 * n <= static_cast<int>(blockDim.x)) {
    // T threads per entry, each summing a contiguous subset of the clusters (one
    // round of loads for up to 16 T clusters), then the T subsets in order
    __shared__ double gsp[G2_THREADS];
    const int T = static_cast<int>(blockDim.x) / n, t = threadIdx.x, col = t % n, q = t / n;
    const int sub = (c1 - c0 + T - 1) / T;
    double s = 0.0;
    if (q < T) {
      const int g0 = c0 + q * sub, g1 = min(c1, g0 + sub);
      for (int gb = g0; gb < g1; gb += R) {
        double v[R];
#pragma unroll
        for (int u = 0; u < R; ++u) v[u] = gb + u < g1 ? __ldcg(part + static_cast<long long>(gb + u) * stride + col) : 0.0;
#pragma unroll
        for (int u = 0; u < R; ++u) s += v[u];
      }
    }
    gsp[t] = s;
    __syncthreads();
    if (t < n) {
      double r = 0.0;
      for (int qq = 0; qq < T; ++qq) r += gsp[qq * n + t];
      dst[t] = r;
    }
    __syncthreads();
    return;
  }
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double s = 0.0;
    for (int g0 = c0; g0 < c1; g0 += R) {
      double v[R];
#pragma unroll
      for (int u = 0; u < R; ++u) v[u] = g0 + u < c1 ? __ldcg(part + static_cast<long long>(g0 + u) * stride + c) : 0.0;
#pragma unroll
      for (int u = 0; u < R; ++u) s += v[u];
    }
    dst[c] = s;
  }
  __syncthreads();
}

// spectral per-mode pass for the live systems: one warp per (slot, 32-mode
// chunk, block segment) over the grid; th = S^ M^^{-1} vh (or S^ vh) and the
// warp-reduced Z^T partials of each (slot, mode chunk) -> zp
// vh_from_w: vh = T^{-1} w of the previous step (unnormalised): scale by 1/||w||
__device__ __forceinline__ void gt_spec(const GridArgs& a, const int* sl, int L, bool bj, bool zt_on, bool vh_from_w) {
  const SpecParams& sp = a.sp;
  const int per = sp.nmc * sp.nseg, items = L * per;
  const int nw = blockDim.x >> 5, gw = blockIdx.x * nw + (threadIdx.x >> 5), tw = gridDim.x * nw;
  for (int it = gw; it < items; it += tw) {
    const int q = it / per, r = it % per, mc = r / sp.nseg, sg = r % sp.nseg;
    double* zo = zt_on ? a.zp + (static_cast<long long>(q) * sp.nmc + mc) * sp.d : nullptr;
    const double ysc = vh_from_w ? 1.0 / __ldcg(a.G.nrm + sl[q]) : 1.0;
    if (bj)
      spec_warp_item<true>(sp, sl[q], mc, sg, a.vh, a.th, zo, nullptr, ysc);
    else
      spec_warp_item<false>(sp, sl[q], mc, sg, a.vh, a.th, zo, nullptr, ysc);
  }
}

__global__ void __launch_bounds__(G2_THREADS, GT_MINB) arnoldi_grid_kernel(GridArgs a) {
  extern __shared__ __align__(16) double gt_smem[];
  double* gsmem = gt_smem;                // GT_SMEM bytes: tile pipeline / tile partial
  double* hs = gt_smem + max(a.vcap, GT_SMEM / 8);  // GT_MAXCOL: h1 of this CTA's system
  double* h2s = hs + GT_MAXCOL;           // GT_MAXCOL: h2
  double* pdot = h2s + GT_MAXCOL;         // GT_MAXCOL: this CTA's partial dots (read by the cluster)
  double* cs_ = pdot + GT_MAXCOL;         // 2 d: coarse rhs / solution
  __shared__ int sl[GT_MAXSYS], ncol[GT_MAXSYS], c0s[GT_MAXSYS + 1];
  __shared__ int s_L;
  __shared__ double bred[G2_THREADS / 32];
  __shared__ GtDesc gd;
  __shared__ Tile2 gd_tiles[GT_TC], gd_gv[GT_GC];
  __shared__ GemmJob gd_jobs[GT_JC];
  gt_desc_init(a, gd, gd_tiles, gd_jobs, gd_gv);

  GmState_& G = a.G;
  const long long k = G.k;
  const int stride = G.m + 2;
  const int d = a.P.d, w = a.P.w, w2 = 2 * w, mx = a.P.mx;
  const int NB = gridDim.x, bid = blockIdx.x, ncl = NB / GT_CL, cid = bid / GT_CL;
  double* part1 = a.part;
  double* part2 = a.part + static_cast<long long>(ncl) * stride;
  double* part3 = a.part + 2LL * ncl * stride;
  unsigned epoch = 0;
  int step = 0;
  bool vh_ready = false, vh_from_w = false;

  for (;;) {
    // ---- live systems of this launch (identical in every CTA: state was
    // last written before the previous barrier); warp 0, one candidate per lane
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const int na = *a.acount;
      if (na > GT_MAXSYS) asm volatile("trap;");
      int s = -1, jc = 0;
      bool run = false;
      if (lane < na) {
        s = a.alist[lane];
        run = __ldcg(G.state + s) == GM_RUN && __ldcg(G.active + s) != 0;
        jc = __ldcg(G.jcyc + s);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, run);
      if (run) {
        const int pos = __popc(bal & ((1u << lane) - 1u));
        sl[pos] = s;
        ncol[pos] = jc + 1;
      }
      const int L = __popc(bal);
      if (lane < L) c0s[lane] = static_cast<int>(static_cast<long long>(lane) * ncl / L);
      if (lane == 0) {
        c0s[L] = ncl;
        s_L = L;
      }
    }
    __syncthreads();
    const int L = s_L;
    if (L == 0) return;
    unsigned long long* tr =
        (a.trace && bid == 0 && step < 64) ? a.trace + static_cast<long long>(step) * 16 : nullptr;
    auto mark = [&](int ph) {
      if (tr && threadIdx.x == 0) tr[ph] = gt_timer();
    };
    mark(0);
    auto T2 = [&](int stg) -> unsigned long long* {
      return a.trace2 ? a.trace2 + ((static_cast<long long>(step % 4) * 4 + stg) * NB + bid) * 8 : nullptr;
    };

    // this CTA's system and rows for the vector phases (groups of whole clusters)
    int q = 0;
    while (q + 1 < L && c0s[q + 1] <= cid) ++q;
    const int gc0 = c0s[q], gc1 = c0s[q + 1];
    const int s = sl[q], nper = (gc1 - gc0) * GT_CL, idx = bid - gc0 * GT_CL;
    // even row ranges (k = 2 w (m_x - 1) is even): 16-byte aligned row pairs for gt_vblock_load
    const long long rows_per = ((k + nper - 1) / nper + 1) & ~1LL;
    const int r0 = static_cast<int>(min(k, idx * rows_per)), r1 = static_cast<int>(min(k, (idx + 1) * rows_per));
    const long long so = s * k;
    const int j = ncol[q] - 1, ncols = ncol[q];
    const double* Vs = a.V + s * G.vstride;
    double* ws = a.w + so;
    const int nr = r1 - r0;
    // V-row block: beyond the tile ring (loaded at the step start, under the operator
    // phases) when it fits there, else over the ring after the operator stages
    const long long vneed = static_cast<long long>(ncols + 1) * nr;
    const bool vc_early = a.pythag && (k & 1) == 0 && vneed <= a.vcap - GT_SMEM / 8;
    const bool vc = vc_early || (a.pythag && (k & 1) == 0 && vneed <= a.vcap);
    double* vb = vc_early ? gsmem + GT_SMEM / 8 : gsmem;
    double* wb = vb + ncols * nr;
    if (vc_early) gt_vblock_load(Vs, k, ncols, r0, nr, vb);

    // ---- operator: u = M^{-1} vin (block-Jacobi stages), then S
    BufTable bj;
    bj.p[BUF_IN] = a.vin;
    bj.p[BUF_OUT] = a.u;
    bj.p[BUF_TMP] = a.tmp;
    bj.p[BUF_TMP2] = nullptr;
    if (a.spectral) {
      // T^{-1} v -> per-mode S^ M^^{-1} (+ Z^T partials) -> T.  The first step
      // of the launch transforms vin; later steps find T^{-1} w of the
      // previous step already in vh (computed with the norm, see below).
      BufTable f;
      f.p[BUF_TMP] = f.p[BUF_TMP2] = nullptr;
      if (!vh_ready) {
        f.p[BUF_IN] = a.vin;
        f.p[BUF_OUT] = a.vh;
        gt_stage(a, gd, 4, sl, L, f, gsmem, T2(0));
        grid_sync(a.bar, epoch);
        vh_ready = true;
      }
      mark(1);
      gt_spec(a, sl, L, a.method != SMPM_SCHUR, a.method == SMPM_DBJ, vh_from_w);
      grid_sync(a.bar, epoch);
      mark(2);
      f.p[BUF_IN] = a.th;
      f.p[BUF_OUT] = a.method == SMPM_DBJ ? a.t : a.w;
      gt_stage(a, gd, 5, sl, L, f, gsmem, T2(1));
      if (a.method == SMPM_DBJ) {
        // coarse solves c = C^{-1} Z^T t, one idle CTA per live slot (from the end of the grid)
        const int qc = NB - 1 - bid;
        if (qc < L) {
          for (int i = threadIdx.x; i < d; i += blockDim.x) {
            double v = 0.0;
            for (int mc = 0; mc < a.sp.nmc; ++mc) v += __ldcg(a.zp + (static_cast<long long>(qc) * a.sp.nmc + mc) * d + i);
            cs_[i] = v;
          }
          __syncthreads();
          coarse_solve_block(a.P, sl[qc], cs_, cs_ + d);
          for (int i = threadIdx.x; i < d; i += blockDim.x) a.cg[static_cast<long long>(qc) * d + i] = cs_[d + i];
        }
      }
      grid_sync(a.bar, epoch);
      mark(3);
      mark(4);
    } else if (a.method != SMPM_SCHUR) {
      for (int stg = 0; stg < 3; ++stg) {
        gt_stage(a, gd, stg, sl, L, bj, gsmem, T2(stg));
        grid_sync(a.bar, epoch);
        mark(1 + stg);
      }
    }
    const double* sin = a.method == SMPM_SCHUR ? a.vin : a.u;
    if (a.method == SMPM_2LAS) {
      // minv = M^{-1} v + Z C^{-1} Z^T v : t = u + Z c(Z^T vin)
      gt_zt(a, a.vin, sl, L);
      grid_sync(a.bar, epoch);
      for (int i = threadIdx.x; i < d; i += blockDim.x) cs_[i] = __ldcg(a.zsum + static_cast<long long>(q) * d + i);
      __syncthreads();
      coarse_solve_block(a.P, s, cs_, cs_ + d);
      for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x)
        a.t[so + r] = __ldcg(a.u + so + r) + cs_[d + r / w2];
      grid_sync(a.bar, epoch);
      sin = a.t;
    }
    if (!a.spectral) {
      BufTable sb;
      sb.p[BUF_IN] = const_cast<double*>(sin);
      // dbj: S writes t and the fused P produces w in pass 1; otherwise S writes w
      sb.p[BUF_OUT] = a.method == SMPM_DBJ ? a.t : a.w;
      sb.p[BUF_TMP] = nullptr;
      sb.p[BUF_TMP2] = nullptr;
      gt_stage(a, gd, 3, sl, L, sb, gsmem, T2(3));
      grid_sync(a.bar, epoch);
      mark(4);
    }
    if (vc && !vc_early) {
      __syncthreads();  // the tile ring (same region) is free from here to the next operator stage
      gt_vblock_load(Vs, k, ncols, r0, nr, vb);
    }
    if (a.method == SMPM_DBJ) {
      // ---- fused deflation P: c = C^{-1} Z^T t ; w = t - Z c - (S - I) Z c
      if (a.spectral) {
        // c was solved in the transform phase
        for (int i = threadIdx.x; i < d; i += blockDim.x) cs_[d + i] = __ldcg(a.cg + static_cast<long long>(q) * d + i);
        __syncthreads();
        mark(5);
      } else {
        gt_zt(a, a.t, sl, L);
        grid_sync(a.bar, epoch);
        mark(5);
        for (int i = threadIdx.x; i < d; i += blockDim.x) cs_[i] = __ldcg(a.zsum + static_cast<long long>(q) * d + i);
        __syncthreads();
        coarse_solve_block(a.P, s, cs_, cs_ + d);
      }
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
        const double wv = __ldcg(ts + e) - (c[i] + sz);
        ws[e] = wv;
        if (vc) wb[e - r0] = wv;
      }
      __syncthreads();
      mark(6);
    } else if (vc) {
      for (int r = threadIdx.x; r < nr; r += blockDim.x) wb[r] = __ldcg(ws + r0 + r);
    }
    if (vc) {
      cp_async_wait<0>();
      __syncthreads();
    }
    // ---- CGS2 pass 1: h1 = V^T w
    if (vc) {
      gt_vblock_dots(vb, wb, nr, ncols, pdot);
      __syncthreads();
    } else {
      gt_col_dots(Vs, k, ncols, ws, r0, r1, pdot);
    }
    gt_cluster_sum(pdot, ncols, part1 + static_cast<long long>(cid) * stride);
    grid_sync(a.bar, epoch);
    gt_group_sum(part1, stride, gc0, gc1, ncols, hs);
    mark(7);
    // ---- pass 2: w -= V h1 ; h2 = V^T w (and ||w||^2 of the updated w)
    double sq1 = 0.0;
    if (vc) {
      // deferred form: w' goes to global memory here, before the reduction's barrier — the next
      // step's transform reads it right after that barrier (otherwise pass 3 writes w)
      const bool w1_out = a.defer && a.spectral && a.pythag;
      for (int r = threadIdx.x; r < nr; r += blockDim.x) {
        const double nv = wb[r] - gt_vblock_row(vb, nr, ncols, hs, r);
        wb[r] = nv;
        if (w1_out) ws[r0 + r] = nv;
        sq1 = fma(nv, nv, sq1);
      }
      __syncthreads();
      gt_vblock_dots(vb, wb, nr, ncols, pdot);
      __syncthreads();
    } else {
      sq1 = gt_update(Vs, k, ncols, hs, ws, r0, r1);
      __syncthreads();
      gt_col_dots(Vs, k, ncols, ws, r0, r1, pdot);
    }
    const int n2 = a.pythag ? ncols + 1 : ncols;
    if (a.pythag) {
      const double q1 = warp_sum(sq1);
      if ((threadIdx.x & 31) == 0) bred[threadIdx.x >> 5] = q1;
      __syncthreads();
      if (threadIdx.x == 0) {
        double tsum = 0.0;
        for (int i = 0; i < G2_THREADS / 32; ++i) tsum += bred[i];
        pdot[ncols] = tsum;
      }
    }
    gt_cluster_sum(pdot, n2, part2 + static_cast<long long>(cid) * stride);
    grid_sync(a.bar, epoch);
    gt_group_sum(part2, stride, gc0, gc1, n2, h2s);
    mark(8);
    if (a.pythag) {
      // ||w - V h2||^2 = ||w||^2 - ||h2||^2 (h2 is the O(eps) reorthogonalisation
      // correction); every CTA of the group computes it in the same order
      if (threadIdx.x < 32) {
        double hh = 0.0;
        for (int i = threadIdx.x; i < ncols; i += 32) hh = fma(h2s[i], h2s[i], hh);
        hh = warp_sum(hh);
        if (threadIdx.x == 0) bred[0] = sqrt(fmax(h2s[ncols] - hh, 0.0));
      }
      __syncthreads();
      const double nrm = bred[0];
      if (idx == 0) {
        double* gh1 = G.h1 + static_cast<long long>(s) * stride;
        double* gh2 = G.h2 + static_cast<long long>(s) * stride;
        for (int i = threadIdx.x; i < ncols; i += blockDim.x) {
          gh1[i] = hs[i];
          gh2[i] = h2s[i];
        }
        __syncthreads();
        if (threadIdx.x < 32) givens_step(G, s, j, nrm);
      }
      // ---- pass 3: w -= V h2 ; v_{j+1} = w / ||w|| (own rows; unused if the system stops)
      // deferred form (spectral): w keeps w' — the next step's transform runs on it without
      // waiting for this update (the operator is linear; the O(eps) term is dropped exactly
      // as in the per-stage path, vec4.cuh) — and only the basis column takes the update
      double* col = a.V + s * G.vstride + static_cast<long long>(j + 1) * k;
      const bool wr = j + 1 <= G.m;
      const bool dfr = a.defer && a.spectral;
      if (vc) {
        const double inv = 1.0 / nrm;
        double* vs = a.vin + so;
        for (int r = threadIdx.x; r < nr; r += blockDim.x) {
          const double nv = wb[r] - gt_vblock_row(vb, nr, ncols, h2s, r);
          if (!dfr) ws[r0 + r] = nv;
          if (wr) {
            col[r0 + r] = nv * inv;
            vs[r0 + r] = nv * inv;
          }
        }
      } else {
        gt_update_scale(Vs, k, ncols, h2s, ws, r0, r1, 1.0 / nrm, wr ? col : nullptr, a.vin + so, !dfr);
      }
      mark(9);
      if (a.spectral) {
        // next step's T^{-1} v_{j+1} = T^{-1} w / ||w|| (1/||w|| applied in the per-mode pass)
        if (!dfr) grid_sync(a.bar, epoch);
        BufTable f;
        f.p[BUF_IN] = a.w;
        f.p[BUF_OUT] = a.vh;
        f.p[BUF_TMP] = f.p[BUF_TMP2] = nullptr;
        gt_stage(a, gd, 4, sl, L, f, gsmem, nullptr, true);
        vh_from_w = true;
      }
      grid_sync(a.bar, epoch);
      mark(10);
      if (tr && threadIdx.x == 0) tr[11] = static_cast<unsigned long long>(L);
      ++step;
      continue;
    }
    // ---- pass 3: w -= V h2 ; ||w||
    double sq = gt_update(Vs, k, ncols, h2s, ws, r0, r1);
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) bred[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tsum = 0.0;
      for (int i = 0; i < G2_THREADS / 32; ++i) tsum += bred[i];
      pdot[GT_MAXCOL - 1] = tsum;
    }
    gt_cluster_sum(pdot + GT_MAXCOL - 1, 1, part3 + static_cast<long long>(cid) * stride);
    grid_sync(a.bar, epoch);
    mark(9);
    // ---- ||w||: every CTA of the group sums the group's partials in the same order
    gt_group_sum(part3, stride, gc0, gc1, 1, bred);
    const double nrm = sqrt(bred[0]);
    // ---- Givens / stop test on the group leader (writes the system's state)
    if (idx == 0) {
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
        const double v = __ldcg(ws + r) * inv;
        col[r] = v;
        a.vin[so + r] = v;
      }
    if (a.spectral) {
      // next step's T^{-1} v_{j+1} = T^{-1} w / ||w||: transform w now (the
      // 1/||w|| is applied in the per-mode pass), saving a phase per step
      BufTable f;
      f.p[BUF_IN] = a.w;
      f.p[BUF_OUT] = a.vh;
      f.p[BUF_TMP] = f.p[BUF_TMP2] = nullptr;
      gt_stage(a, gd, 4, sl, L, f, gsmem, nullptr, true);
      vh_from_w = true;
    }
    grid_sync(a.bar, epoch);
    mark(10);
    if (tr && threadIdx.x == 0) tr[11] = static_cast<unsigned long long>(L);
    ++step;
  }
}

}  // namespace smpm
