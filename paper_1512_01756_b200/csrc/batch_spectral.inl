// Spectral operator: transform kernel setup / launch, per-mode pass, preconditioned operator (part of batch.cu's translation unit).
// Included by batch.cu; not a standalone header.
// --------------------------------------------------------------------------
// Spectral operator (spectral.cuh): T^{-1} GEMM, per-mode S^ M^^{-1}, T GEMM
// --------------------------------------------------------------------------
SpecParams spec_params(const smpm_batch* b) {
  SpecParams sp{};
  sp.w = b->w;
  sp.d = b->d;
  sp.mx = b->mx;
  sp.nbf = b->nbf;
  sp.single = b->single ? 1 : 0;
  sp.npairs = b->sp_npairs;
  sp.nmode = b->sp_nmode;
  sp.k = b->k;
  sp.gam = reinterpret_cast<const double2*>(b->dgam.p);
  sp.kinv = reinterpret_cast<const double2*>(b->dkinv.p);
  sp.omega = b->domega.p;
  sp.nu = b->dnu.p;
  sp.cadd = nullptr;
  sp.nmc = (b->sp_nmode + SP_MODES - 1) / SP_MODES;
  sp.segb = SP_SEGB;
  if (b->tune.segb > 0) sp.segb = std::max(1, std::min(SP_SEGB, b->tune.segb));
  sp.nseg = (b->nbf + (b->single ? 1 : 0) + sp.segb - 1) / sp.segb;
  return sp;
}

// ---- shared-matrix transforms (xform.cuh): the largest row slice of T / T^{-1}
// that fits in shared memory next to a two-deep column ring, P slices per column group
template <int MB>
bool xform_try(smpm_batch* b, int P) {
  const int w = b->w;
  const size_t smem =
      sizeof(double) * (static_cast<size_t>(w / 8) * MB * 64 + static_cast<size_t>(XF_NS) * XF_NT * xf_bstr(w / 2));
  if (smem > 232448 || 8 * MB * P < w || P > b->ctx->num_sms) return false;
  CUDA_CHECK(cudaFuncSetAttribute(xform_kernel<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  std::vector<double> f(static_cast<size_t>(P) * (w / 8) * MB * 64), fi(f.size());
  xform_frag_order(b->hT.data(), w, P, MB, f.data());
  xform_frag_order(b->hTi.data(), w, P, MB, fi.data());
  b->dTfrag.upload(f, b->ctx->stream);
  b->dTifrag.upload(fi, b->ctx->stream);
  CUDA_CHECK(cudaStreamSynchronize(b->ctx->stream));
  b->xf_P = P;
  b->xf_MB = MB;
  b->xf_smem = smem;
  return true;
}

// K-streamed kernel (xformk.cuh) for w whose resident slice does not fit
template <int MB, int NS>
bool xformk_try(smpm_batch* b, int P) {
  const int w = b->w;
  const size_t smem = xformk_smem<MB, NS>();
  if (smem > 232448 || 8 * MB * P < w || P > b->ctx->num_sms) return false;
  CUDA_CHECK(cudaFuncSetAttribute(xformk_kernel<MB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  std::vector<double> f(static_cast<size_t>(P) * (w / 8) * MB * 64), fi(f.size());
  xform_frag_order(b->hT.data(), w, P, MB, f.data());
  xform_frag_order(b->hTi.data(), w, P, MB, fi.data());
  b->dTfrag.upload(f, b->ctx->stream);
  b->dTifrag.upload(fi, b->ctx->stream);
  CUDA_CHECK(cudaStreamSynchronize(b->ctx->stream));
  b->xf_P = P;
  b->xf_MB = MB;
  b->xf_smem = smem;
  b->xf_stream = true;
  return true;
}

// ---- parity-split transforms (xformp.cuh) -----------------------------------
// True when every column of T (row of T^{-1}) is even or odd under the reversal of
// the node index and the modes are ordered pairs (even, odd), reals (even, odd);
// fills the mode segments of each parity.
bool parity_detect(smpm_batch* b) {
  const int w = b->w, h = w / 2, np2 = 2 * b->sp_npairs;
  if (w % 16 != 0) return false;
  std::vector<int> par(static_cast<size_t>(w), 0);
  const double tol = 1e-14;
  for (int m = 0; m < w; ++m) {
    double amax = 0.0, ce = 0.0, co = 0.0, rmax = 0.0, re = 0.0, ro = 0.0;
    for (int r = 0; r < w; ++r) {
      const double x = b->hT[static_cast<size_t>(m) * w + r], y = b->hT[static_cast<size_t>(m) * w + (w - 1 - r)];
      amax = std::max(amax, std::fabs(x));
      ce = std::max(ce, std::fabs(x - y));
      co = std::max(co, std::fabs(x + y));
      const double p = b->hTi[static_cast<size_t>(r) * w + m], q = b->hTi[static_cast<size_t>(w - 1 - r) * w + m];
      rmax = std::max(rmax, std::fabs(p));
      re = std::max(re, std::fabs(p - q));
      ro = std::max(ro, std::fabs(p + q));
    }
    if (ce <= tol * amax && re <= tol * rmax)
      par[m] = 1;
    else if (co <= tol * amax && ro <= tol * rmax)
      par[m] = -1;
    else
      return false;
  }
  int npe = 0;
  while (2 * npe < np2 && par[2 * npe] == 1) ++npe;
  for (int q = 0; q < b->sp_npairs; ++q) {
    const int want = q < npe ? 1 : -1;
    if (par[2 * q] != want || par[2 * q + 1] != want) return false;
  }
  int nre = 0;
  while (np2 + nre < w && par[np2 + nre] == 1) ++nre;
  for (int m = np2 + nre; m < w; ++m)
    if (par[m] != -1) return false;
  if (2 * npe + nre != h) return false;
  b->xp_h = h;
  b->xp_ks = (h + XK_KS - 1) / XK_KS;
  b->xp_seg_start[0][0] = 0;
  b->xp_seg_len0[0] = 2 * npe;
  b->xp_seg_start[0][1] = np2;
  b->xp_seg_start[1][0] = 2 * npe;
  b->xp_seg_len0[1] = np2 - 2 * npe;
  b->xp_seg_start[1][1] = np2 + nre;
  return true;
}

// the xformp_kernel instances: (m-blocks per slice, ring depth) per direction
struct XpKernel {
  int MB;
  void (*fn)(XformPArgs);
  size_t smem;
  void (*fn_ws[2])(XformPArgs);  // warp-specialised variants (xformq.cuh): 2 or 3 consumer warpgroups
  size_t smem_ws;
  void (*fn_ares)(XformPArgs);   // ... with the slice's matrix resident in shared memory (small w)
  size_t (*smem_ares)(int nstage);
};
template <int MB, int NS, bool BWD>
XpKernel xp_instance() {
  // resident-matrix variant: the ring carries column slabs only (forward 24.6 KB, backward 12.3 KB a stage)
  constexpr int NSA = BWD ? 6 : 4;
  return XpKernel{MB, xformp_kernel<MB, NS, BWD>, xformp_smem<MB, NS, BWD>(),
                  {xformq_kernel<MB, NS, BWD, 2>, xformq_kernel<MB, NS, BWD, 3>}, xformq_smem<MB, NS, BWD>(),
                  xformq_kernel<MB, NSA, BWD, 2, true>, xformq_ares_smem<MB, NSA, BWD>};
}
const XpKernel* xp_kernels(bool bwd, int& count) {
  static const XpKernel fwd[] = {xp_instance<9, 6, false>(), xp_instance<11, 6, false>(), xp_instance<17, 5, false>(),
                                 xp_instance<26, 4, false>(), xp_instance<34, 3, false>()};
  static const XpKernel back[] = {xp_instance<5, 8, true>(), xp_instance<9, 8, true>(), xp_instance<11, 8, true>(),
                                  xp_instance<13, 8, true>(), xp_instance<17, 7, true>()};
  count = 5;
  return bwd ? back : fwd;
}
const XpKernel& xp_kernel_for(bool bwd, int MB) {
  int n = 0;
  const XpKernel* ks = xp_kernels(bwd, n);
  for (int i = 0; i < n; ++i)
    if (ks[i].MB == MB) return ks[i];
  fail(SMPM_ERUNTIME, "no parity transform kernel instance for this slice height");
}

void setup_xformp(smpm_batch* b) {
  const int w = b->w, h = b->xp_h, ks = b->xp_ks, mbt = h / 8;
  auto mode = [&](int par, int kap) { return xp_mode(b->xp_seg_start, b->xp_seg_len0, par, kap); };
  std::vector<double> f;
  for (int dir = 0; dir < 2; ++dir) {
    const bool bwd = dir == 1;
    b->xp_var[dir].clear();
    int n = 0;
    const XpKernel* kern = xp_kernels(bwd, n);
    const int mbmax = kern[n - 1].MB;
    // slice counts S = S0, 2 S0, 4 S0 (per parity in the forward direction): the instance of least
    // padding for each; variants whose padding exceeds 45 % of the rows are skipped (the cost model
    // below charges a variant its padded height, so a padded thin variant is only picked when the
    // launch has so few columns that spreading the rows over more SMs still wins: single 2D systems)
    const int S0 = (mbt + mbmax - 1) / mbmax;
    for (int S = S0; S <= 4 * S0; S *= 2) {
      const int need = (mbt + S - 1) / S;
      int MB = 0;
      for (int i = 0; i < n; ++i)
        if (kern[i].MB >= need) {
          MB = kern[i].MB;
          break;
        }
      if (MB == 0) continue;
      if (S > S0 && static_cast<long long>(MB) * S * 100 > 145LL * mbt) continue;
      const int P = bwd ? S : 2 * S;
      if (P > b->ctx->num_sms) continue;
      const XpKernel& kk = xp_kernel_for(bwd, MB);
      CUDA_CHECK(cudaFuncSetAttribute(kk.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kk.smem)));
      for (auto fw : kk.fn_ws)
        CUDA_CHECK(cudaFuncSetAttribute(fw, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kk.smem_ws)));
      const size_t sa = kk.smem_ares(bwd ? 2 * ks : ks);
      const bool ares = sa <= 232448 && b->tune.xform_ares;
      b->xp_var[dir].push_back(std::make_unique<smpm_batch::XpVariant>());
      smpm_batch::XpVariant& v = *b->xp_var[dir].back();
      v.P = P;
      v.MB = MB;
      v.ares_smem = 0;
      if (ares) {
        CUDA_CHECK(cudaFuncSetAttribute(kk.fn_ares, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sa)));
        v.ares_smem = sa;
      }
      if (!bwd)
        xformp_image(2 * S, ks, MB, [&](int sl, int r, int kk2) {
          const int par = sl / S, kap = (sl % S) * 8 * MB + r;
          if (kap >= h || kk2 >= h) return 0.0;
          return b->hTi[static_cast<size_t>(kk2) * w + mode(par, kap)];
        }, f);
      else
        xformp_image(S, 2 * ks, MB, [&](int sl, int r, int kk2) {
          const int k = sl * 8 * MB + r, pq = kk2 / (XK_KS * ks), kap = kk2 - pq * XK_KS * ks;
          if (k >= h || kap >= h) return 0.0;
          return b->hT[static_cast<size_t>(mode(pq, kap)) * w + k];
        }, f);
      v.img.upload(f, b->ctx->stream);
    }
  }
  CUDA_CHECK(cudaStreamSynchronize(b->ctx->stream));
  b->xp_on = !b->xp_var[0].empty() && !b->xp_var[1].empty();
}

void setup_xform(smpm_batch* b) {
  b->xf_P = 0;
  b->xf_stream = false;
  b->xp_on = false;
  if (b->w % 16 != 0 || !b->tune.xform) return;
  bool found = false;
  for (int P = 1; P <= 4 && !found; ++P) {
    const int need = (b->w / 8 + P - 1) / P;
    found = need <= 4 ? xform_try<4>(b, P) : need <= 8 ? xform_try<8>(b, P) : need <= 11 ? xform_try<11>(b, P) : false;
  }
  if (!found) {
    // w > 176: A streams with the columns; P row slices of at most 34 m-blocks
    const int K8 = b->w / 8;
    const int P = (K8 + 33) / 34;
    const int need = (K8 + P - 1) / P;
    if (need <= 26)
      found = xformk_try<26, 5>(b, P);
    else if (need <= 34)
      found = xformk_try<34, 4>(b, P);
  }
  // parity-pure basis: two half-size contractions instead (half the MMA work)
  const int pm = b->tune.xform_parity;
  if (found && pm > 0 && (pm >= 2 || b->xf_stream) && parity_detect(b)) setup_xformp(b);
}

// one transform launch over the columns described by `a` (a.P set), groups column groups
// parity-split launch: `a` as for launch_xform (a.Af / a.P are replaced by the direction's image / slices).
// The slicing variant is the one with the least estimated time for this many columns: a CTA's time is
// (chunks of 64 columns in its share) x (stages) x (fixed cost per stage + cost per m-block).
void launch_xformp(smpm_batch* b, const XformArgs& a, bool inverse, cudaStream_t st, bool pdl) {
  const int dir = inverse ? 0 : 1;
  const long long ncols = static_cast<long long>(a.nslots) * a.ncol_sys * a.nv;
  const long long nch = (ncols + 15) / 16;
  const smpm_batch::XpVariant* best = nullptr;
  int best_groups = 1;
  double best_t = 0.0;
  for (const auto& vp : b->xp_var[dir]) {
    const smpm_batch::XpVariant& v = *vp;
    const int groups = static_cast<int>(std::max(1LL, std::min<long long>(b->ctx->num_sms / v.P, nch)));
    const long long share = ((ncols + groups - 1) / groups + 7) / 8 * 8;
    const long long full = share / XF_NT, rem = share % XF_NT;
    // a trailing chunk of <= 32 columns runs one n-block per warp: half the MMA work
    const double chunks = static_cast<double>(full) + (rem == 0 ? 0.0 : rem <= 32 ? 0.6 : 1.0);
    // backward: two K sweeps (E, O); resident matrix: no A slab traffic per stage
    const double t = chunks * (inverse ? 1.0 : 2.0) * ((v.ares_smem ? 0.15 : 0.25) + 0.065 * v.MB);
    if (!best || t < best_t) {
      best = &v;
      best_t = t;
      best_groups = groups;
    }
  }
  XformPArgs pa;
  pa.x = a;
  pa.x.Af = best->img.p;
  pa.x.P = best->P;
  pa.h = b->xp_h;
  pa.ks = b->xp_ks;
  for (int p = 0; p < 2; ++p) {
    pa.seg_start[p][0] = b->xp_seg_start[p][0];
    pa.seg_start[p][1] = b->xp_seg_start[p][1];
    pa.seg_len0[p] = b->xp_seg_len0[p];
  }
  const XpKernel& kk = xp_kernel_for(!inverse, best->MB);
  // xform_ws: 0 CTA barrier per stage (xformp.cuh), 2 / 3: producer warp + that many consumer
  // warpgroups (xformq.cuh); slices of fewer than 3 m-blocks keep two
  const int nw = b->tune.xform_ws >= 3 && best->MB >= 3 ? 3 : 2;
  const bool ws = b->tune.xform_ws != 0;
  const bool ares = ws && best->ares_smem != 0;
  const dim3 grid(best_groups * best->P), blk(ares ? 384 : ws ? 128 * nw + 128 : XF_THREADS);
  auto fn = ares ? kk.fn_ares : ws ? kk.fn_ws[nw - 2] : kk.fn;
  const size_t smem = ares ? best->ares_smem : ws ? kk.smem_ws : kk.smem;
  if (pdl) {
    launch_pdl(b, fn, grid, blk, smem, st, pa);
  } else {
    fn<<<grid, blk, smem, st>>>(pa);
    check_launch(b);
  }
}

void launch_xform(smpm_batch* b, const XformArgs& a, int groups, cudaStream_t st, bool pdl) {
  const dim3 grid(groups * a.P), blk(XF_THREADS);
  auto go = [&](auto kern) {
    if (pdl) {
      launch_pdl(b, kern, grid, blk, b->xf_smem, st, a);
    } else {
      kern<<<grid, blk, b->xf_smem, st>>>(a);
      check_launch(b);
    }
  };
  if (b->xf_stream) {
    if (b->xf_MB == 26)
      go(xformk_kernel<26, 5>);
    else
      go(xformk_kernel<34, 4>);
    return;
  }
  switch (b->xf_MB) {
    case 4: go(xform_kernel<4>); break;
    case 8: go(xform_kernel<8>); break;
    default: go(xform_kernel<11>); break;
  }
}

// out = A in (and out2 = A in2) for every w-block of the live systems, A = T^{-1} (inverse) or T
void run_xform(smpm_batch* b, bool inverse, const double* in, double* out, const Live& lv, cudaStream_t st,
               const double* in2 = nullptr, double* out2 = nullptr) {
  if (lv.nslots == 0) return;
  ProfScope psx(b, 8, st);  // class 8: shared-matrix transforms
  if (b->xf_P == 0) {
    run_plan(b, inverse ? b->pF : b->pB, in, out, nullptr, lv, st);
    if (in2) run_plan(b, inverse ? b->pF : b->pB, in2, out2, nullptr, lv, st);
    return;
  }
  XformArgs a;
  a.Af = inverse ? b->dTifrag.p : b->dTfrag.p;
  a.w = b->w;
  a.ncol_sys = 2 * b->d;
  a.k = b->k;
  a.alist = lv.alist;
  a.acount = lv.acount;
  a.nslots = lv.nslots;
  a.nv = in2 ? 2 : 1;
  a.in[0] = in;
  a.out[0] = out;
  a.in[1] = in2;
  a.out[1] = out2;
  a.P = b->xf_P;
  // column groups: every SM busy unless a group's share would drop below 16 columns
  const long long nch = (static_cast<long long>(lv.nslots) * a.ncol_sys * a.nv + 15) / 16;
  const int groups = static_cast<int>(std::max(1LL, std::min<long long>(b->ctx->num_sms / a.P, nch)));
  if (b->xp_on)
    launch_xformp(b, a, inverse, st, true);
  else
    launch_xform(b, a, groups, st, true);
}

// th = S^ M^^{-1} vh (bj) or S^ vh in T-coordinates; with cout, also
// c = C^{-1} Z^T (T th) per system (deflation coarse solve)
// (sums_only, spec_op3_kernel only: cout receives the coarse right-hand sides instead)
void spec_apply(smpm_batch* b, bool bj, const double* vh, double* th, double* cout, const Live& lv, cudaStream_t st,
                double* uh = nullptr, const double* cadd = nullptr, bool sums_only = false) {
  if (lv.nslots == 0) return;
  ProfScope ps(b, 7, st);  // class 7: per-mode pass
  SpecParams sp = spec_params(b);
  sp.cadd = cadd;
  DeflateParams P = deflate_params(b, lv.active);
  P.alist = lv.alist;
  P.acount = lv.acount;
  double* zp = cout ? b->dzpart.p : nullptr;
  if (b->tune.spec_v2) {
    // pipelined pass: segments as long as ~32 warps per SM still allow (shorter halo), at
    // least 4 and at most 16 blocks.  spec_v2 = 2 (default): spec_op3_kernel, 16 bytes per
    // lane for every mode (a pair, or two real modes); 1: spec_op2_kernel, one mode per lane
    const bool v3 = b->tune.spec_v2 >= 2;
    const int nch = v3 ? spec3_chunks(sp.npairs, sp.nmode) : sp.nmc;
    const long long nbk = b->nbf + (b->single ? 1 : 0);
    const long long warps = nbk * nch * lv.nslots;
    int segb = static_cast<int>(std::max(4LL, std::min(16LL, warps / (32LL * b->ctx->num_sms))));
    if (b->tune.segb > 0) segb = b->tune.segb;
    sp.segb = segb;
    sp.nseg = static_cast<int>((nbk + segb - 1) / segb);
    const dim3 grid2(nch * ((sp.nseg + SP_WARPS - 1) / SP_WARPS), lv.nslots);
    const size_t shm2 = cout ? sizeof(double) * 2 * static_cast<size_t>(b->d) : 0;
    if (v3) {
      if (bj)
        launch_pdl(b, spec_op3_kernel<true>, grid2, dim3(SP_THREADS), shm2, st, sp, vh, th, P, zp, b->dcount.p, cout,
                   uh, sums_only ? 1 : 0);
      else
        launch_pdl(b, spec_op3_kernel<false>, grid2, dim3(SP_THREADS), shm2, st, sp, vh, th, P, zp, b->dcount.p, cout,
                   uh, sums_only ? 1 : 0);
      return;
    }
    if (bj)
      launch_pdl(b, spec_op2_kernel<true>, grid2, dim3(SP_THREADS), shm2, st, sp, vh, th, P, zp, b->dcount.p, cout, uh);
    else
      launch_pdl(b, spec_op2_kernel<false>, grid2, dim3(SP_THREADS), shm2, st, sp, vh, th, P, zp, b->dcount.p, cout,
                 uh);
    return;
  }
  const dim3 grid(sp.nmc * ((sp.nseg + SP_WARPS - 1) / SP_WARPS), lv.nslots);
  // staged slot rows (tuning sp_stage = 0: direct loads)
  sp.stage = sp.segb <= SP_SEGB && b->tune.sp_stage ? 1 : 0;
  const size_t shm = (cout ? sizeof(double) * 2 * static_cast<size_t>(b->d) : 0) +
                     (sp.stage ? sizeof(double) * SP_STAGE_DOUBLES : 0);
  if (sp.stage && !b->sp_smem_set) {
    const int mx = static_cast<int>(sizeof(double) * (SP_STAGE_DOUBLES + 2 * 256));
    CUDA_CHECK(cudaFuncSetAttribute(spec_op_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CUDA_CHECK(cudaFuncSetAttribute(spec_op_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    b->sp_smem_set = true;
  }
  if (bj)
    launch_pdl(b, spec_op_kernel<true>, grid, dim3(SP_THREADS), shm, st, sp, vh, th, P, zp, b->dcount.p, cout, uh);
  else
    launch_pdl(b, spec_op_kernel<false>, grid, dim3(SP_THREADS), shm, st, sp, vh, th, P, zp, b->dcount.p, cout, uh);
}

// u = M^{-1} v through the spectral form, and (su != nullptr) S u as well
void spec_Minv(smpm_batch* b, const double* v, double* u, double* su, const Live& lv, cudaStream_t st) {
  run_xform(b, true, v, b->dvh.p, lv, st);
  spec_apply(b, true, b->dvh.p, su ? b->dth.p : nullptr, nullptr, lv, st, b->dvh2.p);
  run_xform(b, false, b->dvh2.p, u, lv, st, su ? b->dth.p : nullptr, su);
}

bool spec_on(const smpm_batch* b) { return b->spectral && b->tune.spectral; }

bool spec_ok(const smpm_batch* b, const SolveCfg& c) {
  return spec_on(b) && (c.method == SMPM_SCHUR || c.method == SMPM_BJ || c.method == SMPM_DBJ);
}
// 2LAS through the spectral form in the per-stage steps (many live systems); the grid
// tail keeps its dense stages for 2LAS (a coarse solve before the per-mode pass would
// add two grid barriers per step; measured: per-stage spectral 2LAS with one live
// system is slower than the dense tail, 12.1 vs 10.2 ms on C3)
bool spec_2las(const smpm_batch* b, const SolveCfg& c) {
  return spec_on(b) && c.method == SMPM_2LAS && b->tune.spec_2las;
}

// S M^{-1} v (bj) or S v through the spectral form; out may be any buffer
void spec_SMinv(smpm_batch* b, bool bj, const double* v, double* out, double* cout, const Live& lv, cudaStream_t st) {
  run_xform(b, true, v, b->dvh.p, lv, st);
  // The coarse solve is a serial recurrence (Thomas, d steps of dependent fp64 operations: 20 us
  // at d = 255) that the per-mode pass's last CTA per system ran with the rest of the GPU idle
  // (ncu: SMs active 28 % of a launch with two live systems).  Its result is first needed after
  // the T transform (fused P of pass 1B), so it runs in zt_coarse_kernel on a side stream beside
  // that transform (C5 +1.6 %; C4, where the events cut the programmatic launch chain once per
  // step, still +3 %).
  const bool fork = cout && b->tune.coarse_fork && b->tune.spec_v2 >= 2 && lv.nslots > 0;
  if (!fork) {
    spec_apply(b, bj, b->dvh.p, b->dth.p, cout, lv, st);
    run_xform(b, false, b->dth.p, out, lv, st);
    return;
  }
  if (!b->st4) {
    int lo = 0, hi = 0;
    CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_CHECK(cudaStreamCreateWithPriority(&b->st4, cudaStreamNonBlocking, hi));
    for (auto& e : b->cfev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  b->dzsum.alloc(std::max<size_t>(b->dzsum.n, static_cast<size_t>(b->nsys) * b->d));
  spec_apply(b, bj, b->dvh.p, b->dth.p, b->dzsum.p, lv, st, nullptr, nullptr, true);
  CUDA_CHECK(cudaEventRecord(b->cfev[0], st));
  CUDA_CHECK(cudaStreamWaitEvent(b->st4, b->cfev[0], 0));
  DeflateParams P = deflate_params(b, lv.active);
  P.alist = lv.alist;
  P.acount = lv.acount;
  zt_coarse_kernel<<<dim3(1, lv.nslots), V2_THREADS, sizeof(double) * 2 * static_cast<size_t>(b->d), b->st4>>>(
      P, b->dzsum.p, b->dcoarse.p, cout, b->dcount.p, 1);
  check_launch(b);
  CUDA_CHECK(cudaEventRecord(b->cfev[1], b->st4));
  run_xform(b, false, b->dth.p, out, lv, st);
  CUDA_CHECK(cudaStreamWaitEvent(st, b->cfev[1], 0));
}

// the preconditioned operator GMRES iterates on (proj/src/deflation.cpp:105-107,131; proj/src/gmres.cpp:144-150)
// returns the number of S applications it made per system
int apply_op(smpm_batch* b, const SolveCfg& c, const double* vin, double* wout, const Live& act, cudaStream_t st) {
  double* u = b->vbuf[4].p;
  double* t = b->vbuf[5].p;
  if (spec_ok(b, c)) {
    if (c.method == SMPM_DBJ) {
      spec_SMinv(b, true, vin, t, nullptr, act, st);
      op_P(b, t, wout, c.fused, act, st);
      return c.fused ? 1 : 2;
    }
    spec_SMinv(b, c.method == SMPM_BJ, vin, wout, nullptr, act, st);
    return 1;
  }
  if (spec_2las(b, c)) {
    // S (M^{-1} + Z C^{-1} Z^T) v: c = C^{-1} Z^T v, then one per-mode pass of
    // T^{-1} v that adds Z c before S^ (proj/src/deflation.cpp:127-131)
    double* cb = b->dcoarse.p + static_cast<size_t>(b->nsys) * b->d;
    run_deflate(b, DEFL_COARSE, vin, nullptr, nullptr, cb, act, st);
    run_xform(b, true, vin, b->dvh.p, act, st);
    spec_apply(b, true, b->dvh.p, b->dth.p, nullptr, act, st, nullptr, cb);
    run_xform(b, false, b->dth.p, wout, act, st);
    return 1;
  }
  switch (c.method) {
    case SMPM_SCHUR:
      op_S(b, vin, wout, act, st);
      return 1;
    case SMPM_BJ:
      op_BJ(b, vin, u, act, st);
      op_S(b, u, wout, act, st);
      return 1;
    case SMPM_DBJ:
      op_BJ(b, vin, u, act, st);
      op_S(b, u, t, act, st);
      op_P(b, t, wout, c.fused, act, st);
      return c.fused ? 1 : 2;
    case SMPM_2LAS: {
      op_BJ(b, vin, u, act, st);
      run_deflate(b, DEFL_ADD_ZC, vin, u, t, nullptr, act, st);  // minv = M^{-1} + Z C^{-1} Z^T
      op_S(b, t, wout, act, st);
      return 1;
    }
  }
  fail(SMPM_EINVAL, "unknown method");
}
