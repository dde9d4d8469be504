// Arnoldi step, grid-persistent tail launch, the batched / stacked solve driver (part of batch.cu's translation unit).
// Included by batch.cu; not a standalone header.
// ---- stacked solve: sums over all systems (vec.cuh); with an all-reduce hook
// (smpm_batch_set_allreduce) the systems of the stack are spread over ranks and
// every sum is all-reduced across them (one all-reduce per inner product,
// proj/src/helmholtz.cpp:187-246 run across GPUs)
void stack_allreduce(smpm_batch* b, int count, cudaStream_t st) {
  const int rc = b->ar_fn(b->ar_user, b->dstack.p, count, st);
  if (rc != 0) fail(SMPM_ERUNTIME, "all-reduce hook failed (" + std::to_string(rc) + ")");
}
void stack_sum(smpm_batch* b, double* v, cudaStream_t st) {
  if (!b->ar_fn) {
    launch_pdl(b, stack_sum_kernel, dim3(1), dim3(128), 0, st, b->nsys, v);
    return;
  }
  stack_sum_local_kernel<<<1, 32, 0, st>>>(b->nsys, v, b->dstack.p);
  check_launch(b);
  stack_allreduce(b, 1, st);
  stack_sum_bcast_kernel<<<1, 128, 0, st>>>(b->nsys, v, b->dstack.p);
  check_launch(b);
}
void stack_h(smpm_batch* b, double* h, cudaStream_t st) {
  if (!b->ar_fn) {
    launch_pdl(b, stack_h_kernel, dim3(1), dim3(128), 0, st, b->G, h);
    return;
  }
  stack_h_local_kernel<<<1, 128, 0, st>>>(b->G, h, b->dstack.p);
  check_launch(b);
  stack_allreduce(b, b->jhost + 1, st);
  stack_h_bcast_kernel<<<1, 128, 0, st>>>(b->G, h, b->dstack.p);
  check_launch(b);
}
void stack_givens(smpm_batch* b, cudaStream_t st) {
  if (!b->ar_fn) {
    launch_pdl(b, stack_givens_kernel, dim3(b->nsys), dim3(32), 0, st, b->G);
    return;
  }
  stack_sum_local_kernel<<<1, 32, 0, st>>>(b->nsys, b->G.snsq, b->dstack.p);
  check_launch(b);
  stack_allreduce(b, 1, st);
  stack_givens_global_kernel<<<b->nsys, 32, 0, st>>>(b->G, b->dstack.p);
  check_launch(b);
}

// row chunking of a CGS2 pass kernel for `nslots` live systems: (live systems x chunks)
// <= the kernel's resident CTA count `res` (one wave)
GmState_ cgs3_chunked(smpm_batch* b, long long res, int nslots, dim3& g) {
  GmState_ Gk = b->G;
  const long long kc = std::max(1LL, res / std::max(1, nslots));
  long long ck = (b->k + kc - 1) / kc;
  ck = std::max(256LL, (ck + 255) / 256 * 256);
  Gk.chunk = static_cast<int>(ck);
  Gk.nchunk = static_cast<int>((b->k + ck - 1) / ck);
  g = dim3(Gk.nchunk, nslots);
  return Gk;
}

// deferred CGS2: materialise the pending basis vector (pass 3': v = (w' - V h2) / nrm
// into the basis and the operator input) before a path that needs it
void flush_pending(smpm_batch* b, int nslots, cudaStream_t st) {
  if (!b->pending) return;
  b->pending = false;
  if (nslots <= 0) return;
  if (b->cgs3_kres[2] == 0) {
    int o = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, cgs3_pass3s_kernel, V3_THREADS, 0));
    b->cgs3_kres[2] = static_cast<long long>(std::max(1, o)) * b->ctx->num_sms;
  }
  dim3 g3;
  const GmState_ G3 = cgs3_chunked(b, b->cgs3_kres[2], nslots, g3);
  launch_pdl(b, cgs3_pass3s_kernel, g3, dim3(V3_THREADS), 0, st, G3, b->dV.p, b->vbuf[3].p, b->vbuf[2].p);
}

void arnoldi_step(smpm_batch* b, const SolveCfg& c, const Live& lv, cudaStream_t st) {
  GmState_& G = b->G;
  double* V = b->dV.p;
  double* vin = b->vbuf[2].p;
  double* wv = b->vbuf[3].p;
  // dbj with fused P on the CGS2 path: the deflation update is applied inside
  // the first Gram-Schmidt pass (only Z^T + the coarse solve run here)
  const bool fuse_into_cgs = c.method == SMPM_DBJ && c.fused && c.orth == SMPM_ORTH_CGS2 && G.m + 2 <= V2_MAXCOL;
  double* cbuf = b->dcoarse.p + static_cast<size_t>(b->nsys) * b->d;
  const double* tdefl = nullptr;
  // deferred CGS2 (vec4.cuh): after a cycle's first step the newest basis vector stays
  // pending as (w', h2); the operator runs on w' and pass 1B forms the vector
  const bool defer = fuse_into_cgs && b->tune.cgs_defer && !G.stacked && b->pythag;
  const bool pend = defer && b->pending;
  const double* opin = pend ? wv : vin;
  if (fuse_into_cgs && spec_ok(b, c)) {
    // spectral: t = S M^{-1} v and c = C^{-1} Z^T t from the per-mode pass
    double* t = b->vbuf[5].p;
    spec_SMinv(b, true, opin, t, cbuf, lv, st);
    tdefl = t;
  } else if (fuse_into_cgs) {
    double* u = b->vbuf[4].p;
    double* t = b->vbuf[5].p;
    op_BJ(b, opin, u, lv, st);
    op_S(b, u, t, lv, st);
    run_deflate(b, DEFL_COARSE, t, nullptr, nullptr, cbuf, lv, st);
    tdefl = t;
  } else {
    apply_op(b, c, vin, wv, lv, st);
  }
  ProfScope ps(b, PC_ORTH, st);
  dim3 grid(G.nchunk, b->nsys);      // system-indexed kernels (MGS, long cycles)
  dim3 sgrid(G.nchunk, lv.nslots);   // live-slot kernels
  const size_t hsm = sizeof(double) * static_cast<size_t>(G.m + 2);
  if (c.orth == SMPM_ORTH_MGS) {
    for (int i = 0; i <= std::min(G.m, G.m_total); ++i) {
      mgs_step_kernel<<<grid, VEC_THREADS, 0, st>>>(G, V, wv, i);
      check_launch(b);
    }
    gm_zero_h2_kernel<<<b->nsys, 128, 0, st>>>(G);
    check_launch(b);
    cgs2_update_kernel<true><<<grid, V2_THREADS, 0, st>>>(G, V, wv, 0);  // norm + Givens only
    check_launch(b);
  } else if (G.m + 2 > V2_MAXCOL) {
    // long cycles: column-count-agnostic kernels (dynamic shared memory)
    cgs_dot_kernel<<<grid, VEC_THREADS, 0, st>>>(G, V, wv);
    check_launch(b);
    cgs_update_kernel<false><<<grid, VEC_THREADS, hsm, st>>>(G, V, wv, 1);
    check_launch(b);
    cgs_update_kernel<true><<<grid, VEC_THREADS, hsm, st>>>(G, V, wv, 1);
    check_launch(b);
  } else {
    // long row chunks: (live systems x chunks) <= the resident CTA count of the
    // passes, so a batch of live systems is one wave (a 5 % second wave would
    // double the pass) and per-system partial sums stay few
    GmState_ Gl = G;
    if (b->cgs3_res == 0) {
      int o1 = 0, o2 = 0, o3 = 0;
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, cgs3_dot_kernel, V3_THREADS, 0));
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, cgs3_update_kernel<false>, V3_THREADS, 0));
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, cgs3_update_kernel<true>, V3_THREADS, 0));
      b->cgs3_res = std::max(1, std::min(o1, std::min(o2, o3))) * b->ctx->num_sms;
    }
    const long long target = b->cgs3_res;
    const long long cps = std::max(1LL, target / lv.nslots);
    long long chunk = (b->k + cps - 1) / cps;
    chunk = std::max(256LL, (chunk + 255) / 256 * 256);
    Gl.chunk = static_cast<int>(chunk);
    Gl.nchunk = static_cast<int>((b->k + chunk - 1) / chunk);
    dim3 cgrid(Gl.nchunk, lv.nslots);
    DeflateParams P = deflate_params(b, nullptr);
    if (!G.stacked && b->pythag) {
      // ||w|| from the second reduction (||w1||^2 - ||h2||^2), the scale folded into pass 3:
      // one reduction and one kernel less per step; iteration counts measured unchanged
      // on 9 right-hand sides (tools/seed_sweep.py).
      // Each pass gets its own row chunking sized to ITS resident CTA count (the
      // passes differ in registers: one wave each; partials and counters are per
      // kernel, the work vector is exchanged only between kernels)
      if (b->cgs3_kres[0] == 0) {
        int o[3] = {0, 0, 0};
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o[0], cgs3_dot_kernel, V3_THREADS, 0));
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o[1], cgs3_pass2n_kernel, V3_THREADS, 0));
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o[2], cgs3_pass3s_kernel, V3_THREADS, 0));
        for (int i = 0; i < 3; ++i) b->cgs3_kres[i] = std::max(1, o[i]) * b->ctx->num_sms;
      }
      auto chunked = [&](long long res, dim3& g) { return cgs3_chunked(b, res, lv.nslots, g); };
      dim3 g1, g2, g3;
      const GmState_ G1 = chunked(b->cgs3_kres[0], g1), G2 = chunked(b->cgs3_kres[1], g2),
                     G3 = chunked(b->cgs3_kres[2], g3);
      const int ncols_h = b->jhost + 1;
      if (pend) {
        // pass 1B: v_j = (w' - V h2) / nrm -> V[:, j], w = (P t) / nrm, h1 = [V, v_j]^T w
        const int nold = b->jhost;
        if (nold <= 2 * V3_GRP) {
          if (b->p1b_res == 0) {
            int o = 0;
            CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, cgs4_pass1b_kernel, V3_THREADS, 0));
            b->p1b_res = static_cast<long long>(std::max(1, o)) * b->ctx->num_sms;
          }
          dim3 gb;
          const GmState_ Gb = chunked(b->p1b_res, gb);
          launch_pdl(b, cgs4_pass1b_kernel, gb, dim3(V3_THREADS), 0, st, Gb, V, wv, tdefl, 1, P,
                     static_cast<const double*>(cbuf));
        } else if (b->tune.cgs_lanes) {
          const int wide = nold > 64 ? 1 : 0;
          auto kern = wide ? cgs5_pass1bl_kernel<true> : cgs5_pass1bl_kernel<false>;
          if (b->p1bl_res[wide] == 0) {
            int o = 0;
            CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, V3_THREADS, 0));
            b->p1bl_res[wide] = static_cast<long long>(std::max(1, o)) * b->ctx->num_sms;
          }
          dim3 gb;
          const GmState_ Gb = chunked(b->p1bl_res[wide], gb);
          launch_pdl(b, kern, gb, dim3(V3_THREADS), 0, st, Gb, V, wv, tdefl, 1, P, static_cast<const double*>(cbuf));
        } else {
          const size_t smem = sizeof(double) * p1bt_smem_doubles(nold);
          if (!b->p1bt_attr) {
            size_t mx = 0;
            for (int cc = 2 * V3_GRP + 1; cc <= 8 * P2T_MAXC; ++cc) mx = std::max(mx, p1bt_smem_doubles(cc));
            CUDA_CHECK(cudaFuncSetAttribute(cgs4_pass1bt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(sizeof(double) * mx)));
            b->p1bt_attr = true;
          }
          if (b->p1bt_res[nold] == 0) {
            int o = 0;
            CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, cgs4_pass1bt_kernel, V3_THREADS, smem));
            b->p1bt_res[nold] = static_cast<long long>(std::max(1, o)) * b->ctx->num_sms;
          }
          dim3 gb;
          const GmState_ Gb = chunked(b->p1bt_res[nold], gb);
          launch_pdl(b, cgs4_pass1bt_kernel, gb, dim3(V3_THREADS), smem, st, Gb, V, wv, tdefl, 1, P,
                     static_cast<const double*>(cbuf));
        }
      } else {
        launch_pdl(b, cgs3_dot_kernel, g1, dim3(V3_THREADS), 0, st, G1, V, wv, tdefl, P, cbuf);
      }
      if (b->tune.p2fuse && b->tune.cgs_lanes && ncols_h > 2 * V3_GRP && ncols_h <= LN_MAXCOL &&
          ncols_h <= G.m + 1) {
        // more than 16 columns: update and dots in one read of V, eight lanes per row (cgs5_pass2l_kernel)
        const int wide = ncols_h > 64 ? 1 : 0;
        auto kern = wide ? cgs5_pass2l_kernel<true> : cgs5_pass2l_kernel<false>;
        if (b->p2l_res[wide] == 0) {
          int o = 0;
          CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, V3_THREADS, 0));
          b->p2l_res[wide] = static_cast<long long>(std::max(1, o)) * b->ctx->num_sms;
        }
        dim3 g2l;
        const GmState_ G2l = chunked(b->p2l_res[wide], g2l);
        launch_pdl(b, kern, g2l, dim3(V3_THREADS), 0, st, G2l, static_cast<const double*>(V), wv);
      } else if (b->tune.p2fuse && ncols_h > 2 * V3_GRP && ncols_h <= 8 * P2T_MAXC && ncols_h <= G.m + 1) {
        // more than 16 columns: update and dots in one read of V through
        // shared-memory row tiles (cgs3_pass2t_kernel)
        const size_t smem = sizeof(double) * p2t_smem_doubles(ncols_h);
        if (!b->p2t_attr) {
          size_t mx = 0;
          for (int cc = 2 * V3_GRP + 1; cc <= 8 * P2T_MAXC; ++cc) mx = std::max(mx, p2t_smem_doubles(cc));
          CUDA_CHECK(cudaFuncSetAttribute(cgs3_pass2t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(sizeof(double) * mx)));
          b->p2t_attr = true;
        }
        if (b->p2t_res[ncols_h] == 0) {
          int o = 0;
          CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, cgs3_pass2t_kernel, V3_THREADS, smem));
          b->p2t_res[ncols_h] = std::max(1, o) * b->ctx->num_sms;
        }
        dim3 g2t;
        const GmState_ G2t = chunked(b->p2t_res[ncols_h], g2t);
        launch_pdl(b, cgs3_pass2t_kernel, g2t, dim3(V3_THREADS), smem, st, G2t, static_cast<const double*>(V), wv,
                   ncols_h);
      } else {
        // ncols <= 16: update and dots in one read of V (tuning p2fuse = 0: two reads)
        launch_pdl(b, cgs3_pass2n_kernel, g2, dim3(V3_THREADS), 0, st, G2, static_cast<const double*>(V), wv,
                   b->tune.p2fuse ? 1 : 0);
      }
      if (defer)
        b->pending = true;  // v_{j+1} is formed by the next step's pass 1B (or flush_pending)
      else
        launch_pdl(b, cgs3_pass3s_kernel, g3, dim3(V3_THREADS), 0, st, G3, V, wv, vin);
      ++b->jhost;
      return;
    }
    launch_pdl(b, cgs3_dot_kernel, cgrid, dim3(V3_THREADS), 0, st, Gl, V, wv, tdefl, P, cbuf);
    if (G.stacked) stack_h(b, G.h1, st);
    launch_pdl(b, cgs3_update_kernel<false>, cgrid, dim3(V3_THREADS), 0, st, Gl, V, wv);
    if (G.stacked) stack_h(b, G.h2, st);
    launch_pdl(b, cgs3_update_kernel<true>, cgrid, dim3(V3_THREADS), 0, st, Gl, V, wv);
    if (G.stacked) stack_givens(b, st);
  }
  (void)hsm;
  dim3 sg(std::max(1, std::min(G.nchunk, 64)), lv.nslots);
  launch_pdl(b, gm_scale_kernel, sg, dim3(256), 0, st, G, V, wv, vin);
  ++b->jhost;
}

// Report staging: four double arrays and one int array gathered into one mapped host block
__global__ void report_pack_kernel(const double* __restrict__ a0, long long n0, const double* __restrict__ a1,
                                   long long n1, const double* __restrict__ a2, long long n2,
                                   const double* __restrict__ a3, long long n3, const int* __restrict__ ai,
                                   long long ni, double* __restrict__ outd, int* __restrict__ outi) {
  pdl_wait();
  pdl_launch();
  const long long nd = n0 + n1 + n2 + n3;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < nd + ni;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (e < n0)
      outd[e] = a0[e];
    else if (e < n0 + n1)
      outd[e] = a1[e - n0];
    else if (e < n0 + n1 + n2)
      outd[e] = a2[e - n0 - n1];
    else if (e < nd)
      outd[e] = a3[e - n0 - n1 - n2];
    else
      outi[e - nd] = ai[e - nd];
  }
}

// Compacted list of live systems (ascending index, so deterministic) from a
// flag array, plus RUN / CYCLE state counts for the host; single CTA.
__global__ void __launch_bounds__(1024) compact_kernel(const int* flags, const int* state, int nsys, int* alist,
                                                       int* acount, int* counts) {
  pdl_wait();
  pdl_launch();
  __shared__ int wsum[32];
  __shared__ int base, run, cyc;
  if (threadIdx.x == 0) {
    base = 0;
    run = 0;
    cyc = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int s0 = 0; s0 < nsys; s0 += blockDim.x) {
    const int s = s0 + threadIdx.x;
    const int f = (s < nsys && flags[s]) ? 1 : 0;
    if (s < nsys && state) {
      if (state[s] == GM_RUN) atomicAdd(&run, 1);
      if (state[s] == GM_CYCLE) atomicAdd(&cyc, 1);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int q = 0; q < warp; ++q) off += wsum[q];
    if (f) alist[off + __popc(bal & ((1u << lane) - 1u))] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int q = 0; q < nw; ++q) t += wsum[q];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *acount = base;
    if (counts) {
      counts[0] = run;
      counts[1] = cyc;
    }
  }
}

// early / late split of the epilogue: systems in a final state (converged, breakdown,
// iteration cap) when the grid tail starts, and the rest
__global__ void early_select_kernel(const int* state, int nsys, int* early, int* late, int* hearly) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys) return;
  const int f = (state[s] != GM_RUN && state[s] != GM_CYCLE) ? 1 : 0;
  early[s] = f;
  late[s] = 1 - f;
  hearly[s] = f;
}

__global__ void select_state_kernel(const int* state, int nsys, int want, int* sel) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nsys) sel[s] = state[s] == want ? 1 : 0;
}

// Runs the remaining Arnoldi steps of the current cycle of the (few) live
// systems in one cooperative, grid-persistent launch (grid.cuh).
// grid of the tail solver: as many CTAs (multiple of the cluster size) as
// can be co-resident, up to SMPM_GRID_PER_SM (default 2) per SM
int grid_blocks(smpm_batch* b) {
  if (b->gt_blocks) return b->gt_blocks;
  // the tile-ring region doubles as the per-step V-row block of the CGS2 passes
  // (SMPM_GT_VBLOCK: 0 off, 1 ring size, 2 as large as two CTAs per SM allow)
  const size_t rest = sizeof(double) * (3 * GT_MAXCOL + 2 * static_cast<size_t>(b->d));
  size_t region = GT_SMEM;
  int vmode = 2;  // 0: no V-row block, 1: within the ring region, 2: as large as 2 CTAs / SM allow (measured best)
  vmode = b->tune.gt_vblock;
  if (vmode >= 2) {
    cudaFuncAttributes fa{};
    CUDA_CHECK(cudaFuncGetAttributes(&fa, arnoldi_grid_kernel));
    int dev = 0, per_sm = 0, resv = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev));
    const long long avail = static_cast<long long>(per_sm) / 2 - resv - static_cast<long long>(fa.sharedSizeBytes) -
                            static_cast<long long>(rest);
    region = std::max<size_t>(GT_SMEM, static_cast<size_t>(std::max(0LL, avail)) / 1024 * 1024);
  }
  b->gt_vcap = vmode > 0 ? static_cast<int>(region / sizeof(double)) : 0;
  b->gt_smem = region + rest;
  const size_t smem = b->gt_smem;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = GT_CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(G2_THREADS);
  cfg.dynamicSmemBytes = smem;
  CUDA_CHECK(cudaFuncSetAttribute(arnoldi_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  int per = 0;
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, arnoldi_grid_kernel, G2_THREADS, smem));
  int cap = 2;
  cap = std::max(1, b->tune.grid_per_sm);
  const int want = b->ctx->num_sms * std::max(1, std::min(per, cap));
  // every CTA must be resident: bound by the cluster occupancy calculator
  cfg.gridDim = dim3(want / GT_CL * GT_CL);
  int ncl = 0;
  CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, arnoldi_grid_kernel, &cfg));
  if (ncl < 1) fail(SMPM_ECUDA, "grid tail kernel cannot be resident");
  b->gt_blocks = std::min(want / GT_CL, ncl) * GT_CL;
  if (b->tune.gt_ctas > 0)  // experiment: cap the tail grid (multiple of the cluster size)
    b->gt_blocks = std::max(GT_CL, std::min(b->gt_blocks, b->tune.gt_ctas / GT_CL * GT_CL));
  return b->gt_blocks;
}

// Returns false (nothing launched) when the cooperative launch is rejected.
bool arnoldi_grid(smpm_batch* b, const SolveCfg& c, const int* alist, const int* acount, cudaStream_t st) {
  ProfScope ps(b, 6, st);  // class 6: grid-persistent tail
  GmState_& G = b->G;
  grid_blocks(b);
  const size_t smem = b->gt_smem;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = GT_CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cfg.blockDim = dim3(G2_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  grid_blocks(b);
  const int nb = b->gt_blocks;
  const size_t stride = static_cast<size_t>(G.m + 2);
  b->dgtpart.alloc(std::max(b->dgtpart.n, 3 * static_cast<size_t>(nb / GT_CL) * stride));
  b->dgtzsum.alloc(std::max(b->dgtzsum.n, static_cast<size_t>(GT_MAXSYS) * b->d));
  GridArgs A{};
  const bool spec = spec_ok(b, c) && b->pc[4].v2 && b->pc[5].v2;
  for (int i = 0; i < (spec ? 6 : 4); ++i) {
    const Plan& p = b->pc[i];
    A.a_stride[i] = p.shared_a ? 0 : b->mstride;
    A.jobs[i] = p.djobs.p;
    A.tiles[i] = p.dtiles2.p;
    A.ntiles[i] = p.ntiles;
    A.ngemm[i] = p.ngemm;
    A.gv[i] = p.dgv.p;
    A.ngv[i] = p.ngv;
    A.njobs[i] = static_cast<int>(p.jobs.size());
  }
  A.vin = b->vbuf[2].p;
  A.w = b->vbuf[3].p;
  A.u = b->vbuf[4].p;
  A.t = b->vbuf[5].p;
  A.tmp = b->vbuf[9].p;
  A.V = b->dV.p;
  A.part = b->dgtpart.p;
  if (spec) {
    A.spectral = 1;
    A.sp = spec_params(b);
    // latency-bound tail: one block per warp item (more warps, halo recomputed)
    A.sp.segb = 1;
    A.sp.nseg = b->nbf + (b->single ? 1 : 0);
    A.vh = b->dvh.p;
    A.th = b->dth.p;
    b->dgtzp.alloc(std::max(b->dgtzp.n, static_cast<size_t>(GT_MAXSYS) * A.sp.nmc * b->d));
    A.zp = b->dgtzp.p;
    b->dgtcg.alloc(std::max(b->dgtcg.n, static_cast<size_t>(GT_MAXSYS) * b->d));
    A.cg = b->dgtcg.p;
  }
  A.zsum = b->dgtzsum.p;
  A.bar = b->dgbar.p;
  A.alist = alist;
  A.acount = acount;
  A.method = c.method;
  A.pythag = b->pythag ? 1 : 0;
  A.defer = b->tune.cgs_defer && b->pythag ? 1 : 0;
  A.vcap = b->gt_vcap;
  A.G = G;
  A.P = deflate_params(b, nullptr);
  const char* tpath = b->tune.gt_trace.empty() ? nullptr : b->tune.gt_trace.c_str();
  DevArray<unsigned long long> dtr;
  if (tpath) {
    dtr.alloc(64 * 16);
    CUDA_CHECK(cudaMemsetAsync(dtr.p, 0, dtr.n * sizeof(unsigned long long), st));
    A.trace = dtr.p;
  }
  const char* t2path = b->tune.gt_trace2.empty() ? nullptr : b->tune.gt_trace2.c_str();
  DevArray<unsigned long long> dtr2;
  if (t2path) {
    dtr2.alloc(static_cast<size_t>(16) * nb * 8);
    CUDA_CHECK(cudaMemsetAsync(dtr2.p, 0, dtr2.n * sizeof(unsigned long long), st));
    A.trace2 = dtr2.p;
  }
  // the first tail of a solve finds the barrier word zeroed by gm_v0_kernel
  if (!b->gbar_clean) CUDA_CHECK(cudaMemsetAsync(b->dgbar.p, 0, sizeof(unsigned), st));
  b->gbar_clean = false;
  cfg.gridDim = dim3(nb);
  // opt-in plain cluster launch (profilers only: co-residency is then not guaranteed)
  cfg.numAttrs = b->tune.grid_nocoop ? 1 : 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arnoldi_grid_kernel, A);
  if (e != cudaSuccess && !b->tune.grid_nocoop) {
    // cooperative cluster launch rejected (e.g. MPS, or co-residency not
    // guaranteed): the software grid barrier needs every CTA resident, so the
    // caller runs the rest of the cycle with the per-step kernels instead
    (void)cudaGetLastError();
    return false;
  }
  CUDA_CHECK(e);
  check_launch(b);
  if (tpath) {
    std::vector<unsigned long long> h(dtr.n);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), dtr.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (FILE* f = std::fopen(tpath, "ab")) {
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      std::fclose(f);
    }
  }
  if (t2path) {
    std::vector<unsigned long long> h(dtr2.n);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), dtr2.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (FILE* f = std::fopen(t2path, "ab")) {
      const unsigned long long hdr = static_cast<unsigned long long>(nb);
      std::fwrite(&hdr, sizeof(hdr), 1, f);
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      std::fclose(f);
    }
  }
  return true;
}


// xS_host (optional, pinned): also deliver x_S to the host; with the early epilogue the
// rows of the early systems are copied while the grid tail runs
void solve(smpm_batch* b, const SolveCfg& c, const double* bS, double* xS, smpm_report* reps, double* history,
           cudaStream_t st, double* xS_host = nullptr) {
  need_final(b);
  // programmatic dependent launch hides launch latency when the step's kernels are short
  // (C4: +4 %); at C5 sizes (k = 277,440, ms-scale kernels) dependents that become resident
  // early only take SM resources from the running kernel (measured -5 %): auto = off above
  // 100,000 unknowns per system (also measured: chaining only the few-live-system steps of C5, -3.5 %)
  b->pdl = b->tune.pdl < 0 ? b->k <= 100000 : b->tune.pdl != 0;
  b->pythag = b->tune.pythag != 0;
  if (c.max_iter < 1) fail(SMPM_EINVAL, "max_iter must be >= 1");
  const int mtot = static_cast<int>(std::min<long long>(c.max_iter, b->k));
  int m = c.restart > 0 ? std::min(c.restart, mtot) : mtot;
  if (m > 4000) fail(SMPM_EINVAL, "Krylov cycle length above 4000 is not supported (use restart)");
  ensure_gmres(b, m, mtot);
  GmState_& G = b->G;
  G.stacked = c.stacked ? 1 : 0;
  if (c.stacked) {
    if (c.orth != SMPM_ORTH_CGS2) fail(SMPM_EINVAL, "stacked solve: CGS2 orthogonalization only");
    if (m + 2 > V2_MAXCOL) fail(SMPM_EINVAL, "stacked solve: cycle length above 126 (use restart)");
    if (c.method == SMPM_DBJ && !c.fused) fail(SMPM_EINVAL, "stacked solve: fused deflation only");
  }
  const int ns = b->nsys;
  const long long nk = static_cast<long long>(ns) * b->k;
  double* rhs = b->vbuf[0].p;  // GMRES right-hand side (P b_S for dbj)
  double* x = b->vbuf[1].p;    // Krylov iterate
  double* vin = b->vbuf[2].p;
  double* r = b->vbuf[6].p;
  double* sc = b->dsmall.p + static_cast<size_t>(ns) * b->d;  // scratch scalars
  double* nb2 = sc;        // ||b_S||^2
  double* nr2 = sc + ns;   // ||rhs||^2 / ||r||^2
  cudaEvent_t e0, e1, ev[2];
  if (!b->sev[0]) {
    CUDA_CHECK(cudaEventCreate(&b->sev[0]));
    CUDA_CHECK(cudaEventCreate(&b->sev[1]));
    CUDA_CHECK(cudaEventCreateWithFlags(&b->sev[2], cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&b->sev[3], cudaEventDisableTiming));
  }
  e0 = b->sev[0];
  e1 = b->sev[1];
  ev[0] = b->sev[2];
  ev[1] = b->sev[3];
  int* dsel = b->dsel.p;
  int* hcnt = b->hcnt;
  CUDA_CHECK(cudaEventRecord(e0, st));
  const long long launches0 = b->launches;
  long long s_applies = 0, op_applies = 0;

  const Live all = all_systems(b);
  int* alist = b->dalist.p;
  int* acount = b->dalist.p + ns;
  int* alist2 = b->dalist.p + ns + 1;
  int* acount2 = alist2 + ns;

  // ---- right-hand side
  const bool keep_cb = c.method == SMPM_DBJ && c.fused && !c.stacked;
  if (c.method == SMPM_DBJ) {
    op_P(b, bS, rhs, c.fused, all, st);  // pb = P b_S (proj/src/deflation.cpp:110)
    // keep c_b = C^{-1} Z^T b_S for the solution (proj/src/deflation.cpp:118-120):
    // copied by norm2_start_kernel (stacked: here)
    if (c.fused && c.stacked)
      CUDA_CHECK(cudaMemcpyAsync(b->dczb.p, b->dcoarse.p + static_cast<size_t>(ns) * b->d,
                                 sizeof(double) * ns * b->d, cudaMemcpyDeviceToDevice, st));
  } else {
    CUDA_CHECK(cudaMemcpyAsync(rhs, bS, sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
  }
  dim3 vg(std::max(1, std::min(G.nchunk, 64)), ns);
  if (c.stacked) {
    batched_dot(b, bS, bS, nb2, nullptr, st);
    batched_dot(b, rhs, rhs, nr2, nullptr, st);
    // ||b|| and ||rhs|| of the stacked vector (proj/src/helmholtz.cpp:193-201)
    stack_sum(b, nb2, st);
    stack_sum(b, nr2, st);
    launch_pdl(b, gm_start_kernel, dim3((ns + 127) / 128), dim3(128), 0, st, G, static_cast<const double*>(nr2),
               static_cast<const double*>(nb2), c.tol, 1, static_cast<const int*>(nullptr));
  } else {
    // both norms, the GMRES start of each system and the copy of c_b in one launch
    // (the same bits as two batched_dot launches + gm_start_kernel)
    const Chunking ck = chunking(b);
    b->dpart.alloc(std::max<size_t>(b->dpart.n, 2 * static_cast<size_t>(ns) * ck.nchunk));
    launch_pdl(b, norm2_start_kernel, dim3(ck.nchunk, ns), dim3(VEC_THREADS), 0, st, G, b->k, ck.chunk, ck.nchunk, bS,
               static_cast<const double*>(rhs), b->dpart.p, b->dcount.p, nb2, nr2, c.tol,
               static_cast<const double*>(keep_cb ? b->dcoarse.p + static_cast<size_t>(ns) * b->d : nullptr),
               keep_cb ? b->dczb.p : static_cast<double*>(nullptr), b->d);
  }
  // v_0, x = 0 and the tail's barrier word in one launch
  // (and the list of live systems, up to one block's worth of systems)
  const bool v0_lists = ns <= 256;
  launch_pdl(b, gm_v0_kernel, vg, dim3(256), 0, st, G, b->dV.p, static_cast<const double*>(rhs), vin, x,
             b->dgbar.p, v0_lists ? alist : static_cast<int*>(nullptr), v0_lists ? acount : static_cast<int*>(nullptr));
  b->gbar_clean = true;
  if (!v0_lists)
    launch_pdl(b, compact_kernel, dim3(1), dim3(1024), 0, st, static_cast<const int*>(G.active),
               static_cast<const int*>(nullptr), ns, alist, acount, static_cast<int*>(nullptr));
  G.alist = alist;
  G.acount = acount;
  b->jhost = 0;
  b->pending = false;

  int steps = 0;
  // ---- Arnoldi steps; device flags are polled one step behind the launches
  // (step i+1 is queued before the host waits on step i's counters). Grids
  // are sized by `bound`, the live count the host last read: systems only
  // stop inside a cycle, so it bounds the device-compacted live list.
  int bound = ns;
  const int per_sys_applies = c.method == SMPM_DBJ && !c.fused ? 2 : 1;
  auto issue = [&](int slot) {
    Live lv;
    lv.alist = alist;
    lv.acount = acount;
    lv.nslots = bound;
    lv.active = G.active;
    arnoldi_step(b, c, lv, st);
    ++steps;
    // live / cycle-end counts go straight into mapped host memory (no copy in the stream)
    launch_pdl(b, compact_kernel, dim3(1), dim3(1024), 0, st, static_cast<const int*>(G.active),
               static_cast<const int*>(G.state), ns, alist, acount, b->hcnt_dev + 2 * slot);
    CUDA_CHECK(cudaEventRecord(ev[slot], st));
  };
  // few live systems: the rest of the cycle runs grid-persistent (grid.cuh)
  bool use_grid = b->grid_ok && !c.stacked && c.orth == SMPM_ORTH_CGS2 && G.m + 2 <= GT_MAXCOL &&
                        (c.method != SMPM_DBJ || c.fused) && b->tune.grid;
  // The tail pays off while a step is latency-bound: measured crossovers are
  // 8-10 live systems on C4 (k = 22,176) and none on C5 (k = 277,440: the
  // per-stage kernels are faster even for one live system), so the live-count
  // threshold scales with the work per system: grid_max <= tail_rows / k.
  int grid_max = std::max(0, std::min(GT_MAXSYS, b->tune.grid_max));
  if (b->tune.tail_rows > 0)
    grid_max = static_cast<int>(std::min<long long>(grid_max, b->tune.tail_rows / std::max(1LL, b->k)));
  if (use_grid) grid_max = std::min(grid_max, grid_blocks(b) / GT_CL);  // one cluster per live system at least
  int cycles = 0;  // restarts issued: each cycle end may cost one speculative (empty) step
  auto restart = [&](int ncycv) {
    ++cycles;
    b->jhost = 0;
    b->pending = false;  // the cycle's last vector is never needed
    // ---- restart (GMRES(m) extension): x += V y ; r = b - op(x) ; new cycle
    select_state_kernel<<<(ns + 127) / 128, 128, 0, st>>>(G.state, ns, GM_CYCLE, dsel);
    check_launch(b);
    compact_kernel<<<1, 1024, 0, st>>>(dsel, nullptr, ns, alist2, acount2, nullptr);
    check_launch(b);
    Live lr;
    lr.alist = alist2;
    lr.acount = acount2;
    lr.nslots = ncycv;
    lr.active = dsel;
    gm_backsolve_kernel<<<ns, 32, 0, st>>>(G, dsel);
    check_launch(b);
    gm_combine_kernel<<<vg, 256, 0, st>>>(G, b->dV.p, x, dsel, 1);
    check_launch(b);
    apply_op(b, c, x, r, lr, st);
    ++op_applies;
    axpby_kernel<<<grid_for(nk), 256, 0, st>>>(ns, b->k, dsel, nullptr, 1.0, rhs, -1.0, r);
    check_launch(b);
    batched_dot(b, r, r, nr2, dsel, st);
    // stacked: the new cycle starts from the norm of the stacked residual
    // (proj/src/helmholtz.cpp:193-201), as the first cycle does
    if (c.stacked) stack_sum(b, nr2, st);
    gm_start_kernel<<<(ns + 127) / 128, 128, 0, st>>>(G, nr2, nb2, c.tol, 0, G.state);
    check_launch(b);
    gm_v0_kernel<<<vg, 256, 0, st>>>(G, b->dV.p, r, vin, nullptr, nullptr, nullptr, nullptr);
    check_launch(b);
    compact_kernel<<<1, 1024, 0, st>>>(G.active, nullptr, ns, alist, acount, nullptr);
    check_launch(b);
  };
  // ---- epilogue (spectral dbj): x' = V y, then one per-mode pass of x' gives both
  // u = M^{-1} x' (the solution) and t = S M^{-1} x' (the final residual, proj/src/gmres.cpp:129-136),
  // sharing T^{-1} x'; post_dbj_kernel forms x_S = Q u + Z c_b and ||r||^2
  // (proj/src/deflation.cpp:118-120) in one pass
  double* nrf = sc + 2 * ns;
  double* u = b->vbuf[4].p;
  double* tq = b->vbuf[5].p;
  const bool fuse_post = spec_ok(b, c) && ((c.method == SMPM_DBJ && c.fused) || c.method == SMPM_BJ);
  const bool post_one_pass = fuse_post && c.method == SMPM_DBJ && b->tune.post_fuse;
  auto epilogue_dbj = [&](const Live& lv, const int* sel, cudaStream_t s2) {
    launch_pdl(b, gm_backsolve_kernel, dim3(ns), dim3(32), 0, s2, G, sel);
    launch_pdl(b, gm_combine_kernel, vg, dim3(256), 0, s2, G, static_cast<const double*>(b->dV.p), x, sel, 1);
    run_xform(b, true, x, b->dvh.p, lv, s2);
    spec_apply(b, true, b->dvh.p, b->dth.p, b->dcoarse.p + static_cast<size_t>(ns) * b->d, lv, s2, b->dvh2.p);
    run_xform(b, false, b->dvh2.p, u, lv, s2, b->dth.p, tq);
    ProfScope psd(b, PC_DEFL, s2);
    DeflateParams P = deflate_params(b, sel);
    P.alist = lv.alist;
    P.acount = lv.acount;
    const int gx = static_cast<int>(std::min<long long>((b->k + V2_THREADS * 4 - 1) / (V2_THREADS * 4), 64));
    launch_pdl(b, post_dbj_kernel, dim3(gx, lv.nslots), dim3(V2_THREADS), 0, s2, P, static_cast<const double*>(tq),
               static_cast<const double*>(u), static_cast<const double*>(rhs),
               static_cast<const double*>(b->dcoarse.p + static_cast<size_t>(ns) * b->d),
               static_cast<const double*>(b->dczb.p), xS, b->dpost.p, b->dcount.p, nrf, c.final_check ? 1 : 0);
  };
  // early epilogue: the systems that have stopped when the grid tail starts are
  // finished before it (same total work), so that their rows of x_S can travel to
  // the host (solve_host) on a side stream while the tail runs. Running the epilogue
  // itself beside the tail was measured slower: its kernels compete with the
  // latency-bound tail for the SMs. Tuning early = 0: off.
  const bool early_ok = post_one_pass && xS_host && b->tune.early;
  bool early_done = false;
  int* eflag = b->dearly.p;
  int* elist = eflag + ns;
  int* ecount = elist + ns;
  int* lflag = ecount + 1;
  int* llist = lflag + ns;
  int* lcount = llist + ns;
  // (per-stage path without a tail, e.g. C5: the same early epilogue once at most an eighth of
  // the systems is still running; the slow low-wavenumber modes then iterate for tens of steps
  // while the finished rows travel)
  auto do_early = [&](int nslots_bound) {
    {
      if (!b->st2) {
        int lo = 0, hi = 0;
        CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_CHECK(cudaStreamCreateWithPriority(&b->st2, cudaStreamNonBlocking, lo));
        for (auto& e : b->eev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      early_select_kernel<<<(ns + 127) / 128, 128, 0, st>>>(G.state, ns, eflag, lflag, b->hearly_dev);
      check_launch(b);
      compact_kernel<<<1, 1024, 0, st>>>(eflag, nullptr, ns, elist, ecount, nullptr);
      check_launch(b);
      Live le;
      le.alist = elist;
      le.acount = ecount;
      le.nslots = nslots_bound;
      le.active = eflag;
      epilogue_dbj(le, eflag, st);
      CUDA_CHECK(cudaEventRecord(b->eev[1], st));
      // every row (the late systems' rows are copied again at the end)
      CUDA_CHECK(cudaStreamWaitEvent(b->st2, b->eev[1], 0));
      CUDA_CHECK(cudaMemcpyAsync(xS_host, xS, sizeof(double) * nk, cudaMemcpyDeviceToHost, b->st2));
      CUDA_CHECK(cudaEventRecord(b->eev[2], b->st2));
      early_done = true;
    }
  };
  auto launch_tail = [&](int nrun) {
    if (early_ok && !early_done && nrun < ns) do_early(ns - nrun);
    flush_pending(b, nrun, st);  // the tail starts from a materialised v_j
    return arnoldi_grid(b, c, alist, acount, st);
  };
  int cur = 0;
  // a batch small enough for the tail from the start (single 2D systems) skips the per-stage
  // first step and its host round trip: the tail's first step transforms v_0 itself
  bool tail_first = use_grid && ns <= grid_max;
  if (!tail_first) issue(cur);
  for (;;) {
    // invariant here: exactly one step is in flight, in slot `cur` (none when tail_first)
    if (use_grid && bound <= grid_max) {
      int nrun = ns, ncyc = 0;
      if (tail_first) {
        tail_first = false;
      } else {
        CUDA_CHECK(cudaEventSynchronize(ev[cur]));
        nrun = hcnt[2 * cur];
        ncyc = hcnt[2 * cur + 1];
      }
      if (nrun > 0) {
        if (!launch_tail(nrun)) {
          // no cooperative launch: the per-step kernels finish the solve
          use_grid = false;
          issue(cur);
          continue;
        }
        ++steps;
        if (m >= mtot) {
          // one cycle holds every allowed iteration: the tail leaves no system running or waiting
          // for a restart, so the epilogue is queued right behind it (no host round trip)
          nrun = 0;
          ncyc = 0;
        } else {
          compact_kernel<<<1, 1024, 0, st>>>(G.active, G.state, ns, alist, acount, b->hcnt_dev + 2 * cur);
          check_launch(b);
          CUDA_CHECK(cudaStreamSynchronize(st));
          nrun = hcnt[2 * cur];
          ncyc = hcnt[2 * cur + 1];
          if (nrun > 0) fail(SMPM_ERUNTIME, "grid tail launch returned with running systems");
        }
      }
      if (ncyc > 0) {
        restart(ncyc);
        bound = ncyc;
        issue(cur);
        continue;
      }
      break;
    }
    // the device caps every system at max_iter (GM_MAXED); the host bound is a
    // safety limit only: max_iter steps, one speculative step per cycle end
    const int step_limit = mtot + cycles + 2;
    const bool more = steps < step_limit;
    if (more) issue(cur ^ 1);
    CUDA_CHECK(cudaEventSynchronize(ev[cur]));
    const int nrun = hcnt[2 * cur], ncyc = hcnt[2 * cur + 1];
    bound = std::min(bound, nrun);
    // no tail ahead: early epilogue of the systems that have stopped (a later step may be in
    // flight, so the early list is bounded by all systems)
    if (early_ok && !early_done && !(use_grid && grid_max > 0) && c.restart == 0 && nrun > 0 && 8 * nrun <= ns)
      do_early(ns);
    cur ^= 1;
    if (nrun > 0 && more) continue;
    if (more) CUDA_CHECK(cudaEventSynchronize(ev[cur]));  // drain the speculative step
    const int nrun2 = more ? hcnt[2 * cur] : nrun;
    const int ncyc2 = more ? hcnt[2 * cur + 1] : ncyc;
    if (nrun2 > 0 && steps < step_limit) {
      bound = std::min(bound, nrun2);
      issue(cur);
      continue;
    }
    if (ncyc2 > 0) {
      restart(ncyc2);
      bound = ncyc2;
      issue(cur);
      continue;
    }
    break;
  }
  if (post_one_pass) {
    if (early_done) {
      // the systems not finished by the early epilogue
      compact_kernel<<<1, 1024, 0, st>>>(lflag, nullptr, ns, llist, lcount, nullptr);
      check_launch(b);
      Live ll;
      ll.alist = llist;
      ll.acount = lcount;
      ll.nslots = ns;
      ll.active = lflag;
      epilogue_dbj(ll, lflag, st);
    } else {
      epilogue_dbj(all, nullptr, st);
    }
  } else {
    // ---- assemble x' = V y for the last cycle of every system
    launch_pdl(b, gm_backsolve_kernel, dim3(ns), dim3(32), 0, st, G, static_cast<const int*>(nullptr));
    launch_pdl(b, gm_combine_kernel, vg, dim3(256), 0, st, G, static_cast<const double*>(b->dV.p), x,
               static_cast<const int*>(nullptr), 1);
    // ---- final residual check (proj/src/gmres.cpp:129-136): r = rhs - op(x')
    // Spectral dbj/bj: one per-mode pass of x' gives both u = M^{-1} x' (the
    // solution) and t = S M^{-1} x' (the residual operator), sharing T^{-1} x'.
    if (fuse_post) {
      run_xform(b, true, x, b->dvh.p, all, st);
      // dbj: the per-mode pass also yields c = C^{-1} Z^T (S u) for the residual and Q
      spec_apply(b, true, b->dvh.p, b->dth.p, c.method == SMPM_DBJ ? b->dcoarse.p + static_cast<size_t>(ns) * b->d : nullptr,
                 all, st, b->dvh2.p);
      run_xform(b, false, b->dvh2.p, u, all, st, b->dth.p, tq);
    }
  }
  if (c.final_check && !post_one_pass) {
    if (fuse_post && c.method == SMPM_DBJ) {
      run_deflate(b, DEFL_P_FUSED, tq, tq, r, nullptr, all, st);
    } else if (fuse_post) {
      CUDA_CHECK(cudaMemcpyAsync(r, tq, sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
    } else {
      apply_op(b, c, x, r, all, st);
    }
    axpby_kernel<<<grid_for(nk), 256, 0, st>>>(ns, b->k, nullptr, nullptr, 1.0, rhs, -1.0, r);
    check_launch(b);
    batched_dot(b, r, r, nrf, nullptr, st);
  }
  // ---- solution (proj/src/deflation.cpp:118-120, :141; proj/src/gmres.cpp:148)
  switch (c.method) {
    case SMPM_SCHUR:
      CUDA_CHECK(cudaMemcpyAsync(xS, x, sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
      break;
    case SMPM_BJ:
      if (fuse_post)
        CUDA_CHECK(cudaMemcpyAsync(xS, u, sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
      else if (spec_on(b))
        spec_Minv(b, x, xS, nullptr, all, st);
      else
        op_BJ(b, x, xS, all, st);
      break;
    case SMPM_DBJ: {
      double* q = b->vbuf[6].p;
      if (post_one_pass) break;
      if (fuse_post) {
        run_deflate(b, DEFL_Q_TAIL, tq, u, q, nullptr, all, st);  // Q u = u - Z c(Z^T S u)
      } else if (spec_on(b)) {
        // u = M^{-1} x and S u from one per-mode pass, then Q u = u - Z c(Z^T S u)
        double* su = b->vbuf[8].p;
        spec_Minv(b, x, u, su, all, st);
        run_deflate(b, DEFL_Q_TAIL, su, u, q, nullptr, all, st);
      } else {
        op_BJ(b, x, u, all, st);
        op_Q(b, u, q, all, st);
      }
      run_deflate(b, DEFL_ADD_ZC, bS, q, xS, nullptr, all, st);
      break;
    }
    case SMPM_2LAS:
      if (spec_on(b))
        spec_Minv(b, x, u, nullptr, all, st);
      else
        op_BJ(b, x, u, all, st);
      run_deflate(b, DEFL_ADD_ZC, x, u, xS, nullptr, all, st);
      break;
  }
  if (xS_host) {
    if (early_done) {
      // the full copy of the early epilogue first, then the late systems' rows
      CUDA_CHECK(cudaStreamWaitEvent(st, b->eev[2], 0));
      for (int q = 0; q < ns;) {
        if (b->hearly[q]) {
          ++q;
          continue;
        }
        int q1 = q + 1;
        while (q1 < ns && !b->hearly[q1]) ++q1;  // one copy per run of late rows
        CUDA_CHECK(cudaMemcpyAsync(xS_host + static_cast<size_t>(q) * b->k, xS + static_cast<size_t>(q) * b->k,
                                   sizeof(double) * b->k * (q1 - q), cudaMemcpyDeviceToHost, st));
        q = q1;
      }
    } else {
      CUDA_CHECK(cudaMemcpyAsync(xS_host, xS, sizeof(double) * nk, cudaMemcpyDeviceToHost, st));
    }
  }
  // stacked across ranks: the true residual of the whole stack (every entry becomes the global sum)
  if (c.stacked && b->ar_fn && c.final_check) stack_sum(b, nrf, st);
  // report data: queued on the stream into pinned staging (one host wait)
  const size_t rep_ints = static_cast<size_t>(ns) * 8, rep_dbl = static_cast<size_t>(ns) * (8 + (m + 1) + 3);
  const size_t rep_hist = history ? static_cast<size_t>(ns) * G.histcap : 0;
  const size_t rep_bytes = rep_ints * sizeof(int) + (rep_dbl + rep_hist) * sizeof(double);
  if (b->hrep_bytes < rep_bytes) {
    if (b->hrep) cudaFreeHost(b->hrep);
    b->hrep = nullptr;
    b->hrep_dev = nullptr;
    CUDA_CHECK(cudaHostAlloc(&b->hrep, rep_bytes, cudaHostAllocMapped));
    CUDA_CHECK(cudaHostGetDevicePointer(&b->hrep_dev, b->hrep, 0));
    b->hrep_bytes = rep_bytes;
  }
  double* hsc_p = reinterpret_cast<double*>(b->hrep);
  double* hg_p = hsc_p + static_cast<size_t>(ns) * 8;
  double* hsm_p = hg_p + static_cast<size_t>(ns) * (m + 1);
  double* hh_p = hsm_p + static_cast<size_t>(ns) * 3;
  int* hint_p = reinterpret_cast<int*>(hh_p + rep_hist);
  if (reps || history) {
    // one kernel writes the five report arrays straight into the mapped staging block
    // (was: one device-to-host copy each)
    double* dd = reinterpret_cast<double*>(b->hrep_dev);
    const long long n0 = static_cast<long long>(ns) * 8, n1 = static_cast<long long>(ns) * (m + 1),
                    n2 = static_cast<long long>(ns) * 3, n3 = static_cast<long long>(rep_hist);
    const long long tot = n0 + n1 + n2 + n3 + n0;
    launch_pdl(b, report_pack_kernel, dim3(static_cast<unsigned>(std::min<long long>((tot + 255) / 256, 64))), dim3(256),
               0, st, static_cast<const double*>(b->dscal.p), n0, static_cast<const double*>(b->dg.p), n1,
               static_cast<const double*>(sc), n2, static_cast<const double*>(history ? b->dhist.p : nullptr), n3,
               static_cast<const int*>(b->dgint.p), n0, dd, reinterpret_cast<int*>(dd + n0 + n1 + n2 + n3));
  }
  CUDA_CHECK(cudaEventRecord(e1, st));
  CUDA_CHECK(cudaEventSynchronize(e1));
  prof_collect(b);
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  G.alist = nullptr;
  G.acount = nullptr;
  (void)launches0;

  // ---- reports
  if (reps || history) {
    const int* hint = hint_p;
    const double *hsc = hsc_p, *hg = hg_p, *hsm = hsm_p, *hh = hh_p;
    for (int s = 0; s < ns; ++s) {
      const int iters = hint[static_cast<size_t>(ns) + s];
      const int jc = hint[static_cast<size_t>(s)];
      const int hl = hint[static_cast<size_t>(5 * ns) + s];
      const double bn = hsc[static_cast<size_t>(s)];
      const double tgt = hsc[static_cast<size_t>(ns) + s];
      double frel = bn > 0 ? std::fabs(hg[static_cast<size_t>(s) * (m + 1) + jc]) / bn : 0.0;
      bool mismatch = false;
      if (c.final_check && bn > 0) {
        // stacked: the true residual of the stacked vector (proj/src/gmres.cpp:129-136)
        double r2 = hsm[static_cast<size_t>(2 * ns) + s];
        if (c.stacked && !b->ar_fn) {
          r2 = 0.0;
          for (int t = 0; t < ns; ++t) r2 += hsm[static_cast<size_t>(2 * ns) + t];
        }
        const double true_rel = std::sqrt(r2) / bn;
        if (true_rel * bn > 10.0 * std::max(tgt, frel * bn)) mismatch = true;
        frel = true_rel;
      }
      const long long apps = iters + (c.final_check ? 1 : 0) + op_applies;
      if (reps) {
        smpm_report& R = reps[s];
        R.iterations = iters;
        R.history_len = hl;
        R.final_rel_residual = frel;
        R.converged = bn > 0 ? (frel * bn <= tgt * (1.0 + 1e-12)) : 1;
        R.mismatch_warning = mismatch ? 1 : 0;
        R.operator_applies = apps;
        R.krylov_s_applies = apps * per_sys_applies;
        R.wall_time_s = ms * 1e-3;
      }
      if (history)
        for (int i = 0; i < G.histcap; ++i)
          history[static_cast<size_t>(s) * G.histcap + i] = i < hl ? hh[static_cast<size_t>(s) * G.histcap + i] : 0.0;
    }
  }
  (void)s_applies;
}

void launch_zt(smpm_batch* b, const double* v, double* y, cudaStream_t st) {
  zt_kernel<<<(b->nsys * b->d * 32 + 255) / 256, 256, 0, st>>>(b->nsys, b->d, 2 * b->w, b->k, v, y);
  check_launch(b);
}
void launch_z(smpm_batch* b, const double* c, double* y, cudaStream_t st) {
  zbroadcast_kernel<<<grid_for(b->nsys * b->k), 256, 0, st>>>(b->nsys, b->d, 2 * b->w, b->k, nullptr, c, y);
  check_launch(b);
}

SolveCfg cfg_from(int method, const smpm_solve_options* o) {
  SolveCfg c;
  c.method = method;
  c.tol = o ? o->tol : 1e-10;
  c.max_iter = o ? o->max_iter : 100;
  c.restart = o ? o->restart : 0;
  c.orth = o ? o->orth : SMPM_ORTH_CGS2;
  c.fused = o ? o->fuse_deflation != 0 : true;
  c.final_check = o ? o->final_residual_check != 0 : true;
  if (c.method < 0 || c.method > 3) fail(SMPM_EINVAL, "unknown method");
  return c;
}
