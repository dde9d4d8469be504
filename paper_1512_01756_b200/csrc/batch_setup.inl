// Setup: operator plans, block-Jacobi inverses, coarse spaces, device-side FDM setup, finalize (part of batch.cu's translation unit).
// Included by batch.cu; not a standalone header.
// --------------------------------------------------------------------------
// Setup: plans, structured block-Jacobi inverses, coarse spaces
// --------------------------------------------------------------------------
void build_plans(smpm_batch* b) {
  const int w = b->w, d = b->d, mx = b->mx;
  const long long k = b->k;
  const long long w2 = 2LL * w;
  cudaStream_t st = b->ctx->stream;
  b->pS.jobs.clear();
  b->pSt.jobs.clear();
  b->pBJ1.jobs.clear();
  b->pBJ2.jobs.clear();
  b->pBJ3.jobs.clear();
  b->pF.jobs.clear();
  b->pB.jobs.clear();
  b->pF.shared_a = b->pB.shared_a = true;
  for (int s = 0; s < b->nsys; ++s) {
    const long long o = s * k;
    if (b->spectral) {
      // every w-block through T^{-1} (forward) / T (back): w x 2d per system
      b->pF.add(b->dTi.p, w, false, w, 2 * d, w, s, view(BUF_IN, o, w), view(BUF_OUT, o, w), kNoView, 1.0, 0.0);
      b->pB.add(b->dT.p, w, false, w, 2 * d, w, s, view(BUF_IN, o, w), view(BUF_OUT, o, w), kNoView, 1.0, 0.0);
    }
    // ---- S v = v + sum_s G_s [v_{2s-1}; v_{2s}] -> [y_{2s-2}; y_{2s+1}]
    if (mx >= 3)
      b->pS.add(b->GI(s), w2, false, 2 * w, mx - 2, 2 * w, s, view(BUF_IN, o + w, w2),
                view(BUF_OUT, o, w2, w, 2LL * w), view(BUF_IN, o, w2, w, 2LL * w), 1.0, 1.0);
    b->pS.add(b->GW(s), w, false, w, 1, w, s, view(BUF_IN, o), view(BUF_OUT, o + w), view(BUF_IN, o + w), 1.0, 1.0);
    b->pS.add(b->GE(s), w, false, w, 1, w, s, view(BUF_IN, o + (2LL * d - 1) * w), view(BUF_OUT, o + (2LL * d - 2) * w),
              view(BUF_IN, o + (2LL * d - 2) * w), 1.0, 1.0);
    // ---- S^T: own blocks += G^T reader blocks
    if (mx >= 3)
      b->pSt.add(b->GI(s), w2, true, 2 * w, mx - 2, 2 * w, s, view(BUF_IN, o, w2, w, 2LL * w),
                 view(BUF_OUT, o + w, w2), view(BUF_IN, o + w, w2), 1.0, 1.0);
    b->pSt.add(b->GW(s), w, true, w, 1, w, s, view(BUF_IN, o + w), view(BUF_OUT, o), view(BUF_IN, o), 1.0, 1.0);
    b->pSt.add(b->GE(s), w, true, w, 1, w, s, view(BUF_IN, o + (2LL * d - 2) * w), view(BUF_OUT, o + (2LL * d - 1) * w),
               view(BUF_IN, o + (2LL * d - 1) * w), 1.0, 1.0);

    // ---- block-Jacobi, blocks of two interfaces b = 0..nbf-1 (w-blocks 4b..4b+3):
    //   r = [v0; v3] - G'[v1; v2] ; [x0; x3] = K_b^{-1} r ; x1 = v1 - Gee x0 ; x2 = v2 - Gww x3
    const int nbf = b->nbf;
    const long long w4 = 4LL * w;
    if (nbf > 0)
      b->pBJ1.add(b->GI(s), w2, false, 2 * w, nbf, 2 * w, s, view(BUF_IN, o + w, w4), view(BUF_TMP, o, w4),
                  view(BUF_IN, o, w4, w, 2LL * w), -1.0, 1.0);
    for (int bb = 0; bb < nbf;) {
      const bool first = bb == 0;
      const bool last = 2 * bb + 2 == mx - 1;
      int e = bb + 1;
      while (e < nbf && (e == 0) == first && (2 * e + 2 == mx - 1) == last) ++e;
      const int var = (first ? 1 : 0) | (last ? 2 : 0);
      b->pBJ2.add(b->Kinv(s, var), w2, false, 2 * w, e - bb, 2 * w, s, view(BUF_TMP, o + bb * w4, w4),
                  view(BUF_OUT, o + bb * w4, w4, w, 2LL * w), kNoView, 1.0, 0.0);
      bb = e;
    }
    if (nbf > 0) {
      // x1 = v1 - Gee0 x0 : strip 2b is the west-boundary strip for b = 0
      b->pBJ3.add(b->GW(s), w, false, w, 1, w, s, view(BUF_OUT, o), view(BUF_OUT, o + w), view(BUF_IN, o + w), -1.0, 1.0);
      if (nbf > 1)
        b->pBJ3.add(b->GI(s) + w2 * w + w, w2, false, w, nbf - 1, w, s, view(BUF_OUT, o + w4, w4),
                    view(BUF_OUT, o + w4 + w, w4), view(BUF_IN, o + w4 + w, w4), -1.0, 1.0);
      // x2 = v2 - Gww2 x3 : strip 2b+2 is the east-boundary strip when 2b+2 == mx-1
      const bool last_east = 2 * (nbf - 1) + 2 == mx - 1;
      const int ninner = last_east ? nbf - 1 : nbf;
      if (ninner > 0)
        b->pBJ3.add(b->GI(s), w2, false, w, ninner, w, s, view(BUF_OUT, o + 3LL * w, w4), view(BUF_OUT, o + 2LL * w, w4),
                    view(BUF_IN, o + 2LL * w, w4), -1.0, 1.0);
      if (last_east) {
        const long long ob = o + (nbf - 1) * w4;
        b->pBJ3.add(b->GE(s), w, false, w, 1, w, s, view(BUF_OUT, ob + 3LL * w), view(BUF_OUT, ob + 2LL * w),
                    view(BUF_IN, ob + 2LL * w), -1.0, 1.0);
      }
    }
    if (b->single) {
      // trailing interface d-1 (w-blocks 2d-2, 2d-1): r = v0 - G_E v1 ; x0 = K_s^{-1} r ; x1 = v1 - Gee x0
      const long long o0 = o + (2LL * d - 2) * w, o1 = o0 + w;
      b->pBJ1.add(b->GE(s), w, false, w, 1, w, s, view(BUF_IN, o1), view(BUF_TMP, o0), view(BUF_IN, o0), -1.0, 1.0);
      b->pBJ2.add(b->Ksingle(s), w, false, w, 1, w, s, view(BUF_TMP, o0), view(BUF_OUT, o0), kNoView, 1.0, 0.0);
      const double* gee = d >= 2 ? b->GI(s) + w2 * w + w : b->GW(s);
      const long long ldee = d >= 2 ? w2 : w;
      b->pBJ3.add(gee, ldee, false, w, 1, w, s, view(BUF_OUT, o0), view(BUF_OUT, o1), view(BUF_IN, o1), -1.0, 1.0);
    }
  }
  const int sms = b->ctx->num_sms;
  for (Plan* p : {&b->pS, &b->pBJ1, &b->pBJ2, &b->pBJ3, &b->pF, &b->pB}) {
    if (p->jobs.empty()) continue;
    if (!p->v2_ok()) {
      // odd w (16-byte alignment impossible): per-system jobs on the v1 kernel
      p->build(sms, st);
      continue;
    }
    // every system's jobs are system 0's shifted by s*mstride (matrices) and
    // s*k (vectors): keep system 0's as the per-system template
    std::vector<GemmJob> tmpl;
    for (const auto& j : p->jobs)
      if (j.sys == 0) tmpl.push_back(j);
    p->jobs.swap(tmpl);
    // tail variant: K split 4 ways so a handful of live systems still
    // spreads over many SMs (used when <= kTailSystems systems are live)
    p->tail = std::make_unique<Plan>();
    p->tail->jobs = p->jobs;
    p->tail->shared_a = p->shared_a;
    p->tail->build2(std::max(1, sms / b->nsys), st, 4);
    // split-K only when even the whole batch cannot fill the GPU
    p->build2(std::max(1, sms / b->nsys), st);
  }
  b->pSt.build(sms, st);
  // grid tail solver: unsplit copies of the hot stage templates
  b->tmpl_ok = true;
  Plan* src[6] = {&b->pBJ1, &b->pBJ2, &b->pBJ3, &b->pS, &b->pF, &b->pB};
  for (int i = 0; i < 6; ++i) {
    if (i >= 4 && !b->spectral) break;
    if (!src[i]->v2) {
      if (i < 4) {
        b->tmpl_ok = false;
        break;
      }
      continue;
    }
    b->pc[i].shared_a = src[i]->shared_a;
    b->pc[i].jobs = src[i]->jobs;
    for (auto& j : b->pc[i].jobs) j.splitk = 1;
    b->pc[i].build2(0, st);
    std::vector<Tile2> gv;
    for (size_t ji = 0; ji < b->pc[i].jobs.size(); ++ji)
      if (b->pc[i].jobs[ji].N == 1)
        for (int m0 = 0; m0 < b->pc[i].jobs[ji].M; m0 += GT_GVR) gv.push_back(Tile2{static_cast<int>(ji), m0, 0, -1});
    b->pc[i].dgv.upload(gv, st);
    b->pc[i].ngv = static_cast<int>(gv.size());
  }
  // v2 templates hold per-system workspace counts; v1 plans hold totals
  const long long ns = b->nsys;
  long long wst = b->pSt.ws_tiles;
  for (Plan* p : {&b->pS, &b->pBJ1, &b->pBJ2, &b->pBJ3, &b->pF, &b->pB}) {
    wst = std::max(wst, p->ws_tiles * (p->v2 ? ns : 1));
    if (p->tail) wst = std::max(wst, p->tail->ws_tiles * ns);
  }
  b->dws.alloc(static_cast<size_t>(std::max(1LL, wst)) * GEMM_BM * GEMM_BN);
  // grid tail solver: the unsplit templates of the four hot stages (pc)
  b->grid_ok = b->tmpl_ok;
  b->dgbar.alloc(1);
}

__global__ void add_identity_kernel(double* A, long long lda, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) A[i * lda + i] += 1.0;
}
__global__ void set_identity_kernel(double* A, long long lda, int n) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(n) * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = e / n, r = e % n;
    A[c * lda + r] = (r == c) ? 1.0 : 0.0;
  }
}

// K = I - G' diag(Gee0, Gww2) (2w x 2w) or K_single = I - G_E Gee (w x w),
// formed with the GEMM kernel, inverted with cuSOLVER getrf/getrs.
void build_bj_inverses(smpm_batch* b) {
  const int w = b->w, mx = b->mx, d = b->d;
  const long long w2 = 2LL * w;
  cudaStream_t st = b->ctx->stream;
  DevArray<double> Kt;
  Kt.alloc(static_cast<size_t>(4LL * w * w));
  DevArray<int> ipiv, info;
  ipiv.alloc(static_cast<size_t>(2 * w));
  info.alloc(1);
  int lwork = 0;
  CUSOLVER_CHECK(cusolverDnDgetrf_bufferSize(b->ctx->solver, 2 * w, 2 * w, Kt.p, 2 * w, &lwork));
  DevArray<double> work;
  work.alloc(static_cast<size_t>(std::max(lwork, 1)));
  auto invert = [&](double* K, int nn, double* out) {
    CUSOLVER_CHECK(cusolverDnDgetrf(b->ctx->solver, nn, nn, K, nn, work.p, ipiv.p, info.p));
    set_identity_kernel<<<64, 256, 0, st>>>(out, nn, nn);
    check_launch(b);
    CUSOLVER_CHECK(cusolverDnDgetrs(b->ctx->solver, CUBLAS_OP_N, nn, nn, K, nn, ipiv.p, out, nn, info.p));
    int hinfo = 0;
    CUDA_CHECK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (hinfo != 0) fail(SMPM_ESINGULAR, "block-Jacobi: singular preconditioner block");
  };
  for (int s = 0; s < b->nsys; ++s) {
    for (int var = 0; var < 4; ++var) {
      if (!b->kneeded[var]) continue;
      const bool first = var & 1, last = var & 2;
      const double* gee = first ? b->GW(s) : b->GI(s) + w2 * w + w;
      const long long ldee = first ? w : w2;
      const double* gww = last ? b->GE(s) : b->GI(s);
      const long long ldww = last ? w : w2;
      Plan p;
      // K[:, 0:w] = -G'[:, 0:w] Gee ; K[:, w:2w] = -G'[:, w:2w] Gww ; then + I
      BufTable t;
      t.p[BUF_IN] = const_cast<double*>(gee);
      t.p[BUF_OUT] = Kt.p;
      t.p[BUF_TMP] = const_cast<double*>(gww);
      t.p[BUF_TMP2] = nullptr;
      p.add(b->GI(s), w2, false, 2 * w, w, w, 0, view(BUF_IN, 0, ldee), view(BUF_OUT, 0, w2), kNoView, -1.0, 0.0);
      p.add(b->GI(s) + w2 * w, w2, false, 2 * w, w, w, 0, view(BUF_TMP, 0, ldww), view(BUF_OUT, w2 * w, w2), kNoView,
            -1.0, 0.0);
      p.build(0, st);  // no split-K for setup products
      gemm_jobs_kernel<<<p.ntiles, 128, 0, st>>>(p.djobs.p, p.dtiles.p, t, nullptr, nullptr);
      check_launch(b);
      add_identity_kernel<<<8, 256, 0, st>>>(Kt.p, w2, 2 * w);
      check_launch(b);
      invert(Kt.p, 2 * w, b->Kinv(s, var));
    }
    if (b->single) {
      const double* gee = d >= 2 ? b->GI(s) + w2 * w + w : b->GW(s);
      const long long ldee = d >= 2 ? w2 : w;
      Plan p;
      BufTable t;
      t.p[BUF_IN] = const_cast<double*>(gee);
      t.p[BUF_OUT] = Kt.p;
      t.p[BUF_TMP] = nullptr;
      t.p[BUF_TMP2] = nullptr;
      p.add(b->GE(s), w, false, w, w, w, 0, view(BUF_IN, 0, ldee), view(BUF_OUT, 0, w), kNoView, -1.0, 0.0);
      p.build(0, st);
      gemm_jobs_kernel<<<p.ntiles, 128, 0, st>>>(p.djobs.p, p.dtiles.p, t, nullptr, nullptr);
      check_launch(b);
      add_identity_kernel<<<8, 256, 0, st>>>(Kt.p, w, w);
      check_launch(b);
      invert(Kt.p, w, b->Ksingle(s));
    }
  }
  (void)mx;
}

// dense inverse with partial pivoting (host, d <= a few hundred)
std::vector<double> host_inverse(std::vector<double> A, int n) {
  std::vector<double> inv(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i) * n + i] = 1.0;
  auto at = [n](std::vector<double>& M, int r, int c) -> double& { return M[static_cast<size_t>(c) * n + r]; };
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(at(A, r, c)) > std::fabs(at(A, p, c))) p = r;
    if (at(A, p, c) == 0.0) fail(SMPM_ESINGULAR, "coarse matrix is singular");
    if (p != c)
      for (int j = 0; j < n; ++j) {
        std::swap(at(A, p, j), at(A, c, j));
        std::swap(at(inv, p, j), at(inv, c, j));
      }
    const double piv = at(A, c, c);
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = at(A, r, c) / piv;
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        at(A, r, j) -= f * at(A, c, j);
        at(inv, r, j) -= f * at(inv, c, j);
      }
    }
  }
  for (int r = 0; r < n; ++r) {
    const double piv = at(A, r, r);
    for (int j = 0; j < n; ++j) at(inv, r, j) /= piv;
  }
  return inv;
}

// C = Z^T S Z from the couplings' row sums (S Z 1_j only touches interfaces
// j-1, j, j+1; proj/src/deflation.cpp:24-42), rank-one shift or Thomas data.
void build_coarse(smpm_batch* b) {
  const int w = b->w, d = b->d, mx = b->mx, nsys = b->nsys;
  const long long gsz = 6LL * w * w;
  std::vector<double> rows(static_cast<size_t>(nsys) * 6 * w, 0.0);
  std::vector<double> cinv(static_cast<size_t>(nsys) * d * d, 0.0), uc(static_cast<size_t>(nsys) * d, 0.0),
      th(static_cast<size_t>(nsys) * 3 * d, 0.0);
  std::vector<int> cmode(static_cast<size_t>(nsys), 0);
  b->hC.assign(static_cast<size_t>(nsys) * d * d, 0.0);
  b->htri.assign(static_cast<size_t>(nsys), 1);
  b->hsing.assign(static_cast<size_t>(nsys), 0);
  if (b->from_fdm) {
    // the couplings live on the device only: row sums by fdm_rowsum_kernel (fdm_device_setup)
    CUDA_CHECK(cudaMemcpyAsync(rows.data(), b->drowsum.p, sizeof(double) * rows.size(), cudaMemcpyDeviceToHost,
                               b->ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(b->ctx->stream));
  }
  for (int s = 0; s < nsys; ++s) {
    double* rs = rows.data() + static_cast<size_t>(s) * 6 * w;
    double* rWI = rs;
    double* rEI = rs + 2 * w;
    double* rEW = rs + 4 * w;
    double* rWE = rs + 5 * w;
    if (!b->from_fdm) {
      const double* GW = b->hG.data() + s * gsz;
      const double* GI = GW + static_cast<long long>(w) * w;
      const double* GE = GI + 4LL * w * w;
      for (int c = 0; c < w; ++c)
        for (int r = 0; r < 2 * w; ++r) {
          rWI[r] += GI[static_cast<long long>(c) * 2 * w + r];
          rEI[r] += GI[static_cast<long long>(c + w) * 2 * w + r];
        }
      for (int c = 0; c < w; ++c)
        for (int r = 0; r < w; ++r) {
          rEW[r] += GW[static_cast<long long>(c) * w + r];
          rWE[r] += GE[static_cast<long long>(c) * w + r];
        }
    }
    auto sum = [](const double* p, int n) {
      double a = 0.0;
      for (int i = 0; i < n; ++i) a += p[i];
      return a;
    };
    double* C = b->hC.data() + static_cast<size_t>(s) * d * d;
    auto Cat = [&](int i, int j) -> double& { return C[static_cast<size_t>(j) * d + i]; };
    for (int j = 0; j < d; ++j) {
      Cat(j, j) += 2.0 * w;
      if (j == 0) {
        Cat(0, 0) += sum(rEW, w);
      } else {
        Cat(j - 1, j) += sum(rEI, w);
        Cat(j, j) += sum(rEI + w, w);
      }
      if (j + 1 == mx - 1) {
        Cat(j, j) += sum(rWE, w);
      } else {
        Cat(j, j) += sum(rWI, w);
        Cat(j + 1, j) += sum(rWI + w, w);
      }
    }
    if (!b->huS[s].empty()) {
      b->hsing[s] = 1;
      const std::vector<double>& us = b->huS[s];
      double* u = uc.data() + static_cast<size_t>(s) * d;
      double nn = 0.0;
      for (int i = 0; i < d; ++i) {
        double a = 0.0;
        for (int e = 0; e < 2 * w; ++e) a += us[static_cast<size_t>(i) * 2 * w + e];
        u[i] = a;
        nn += a * a;
      }
      nn = std::sqrt(nn);
      int imax = 0;
      for (int i = 0; i < d; ++i) {
        u[i] /= nn;
        if (std::fabs(u[i]) > std::fabs(u[imax])) imax = i;
      }
      if (u[imax] < 0.0)
        for (int i = 0; i < d; ++i) u[i] = -u[i];
      std::vector<double> Cs(C, C + static_cast<size_t>(d) * d);
      for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i) Cs[static_cast<size_t>(j) * d + i] += u[i] * u[j];
      const std::vector<double> inv = host_inverse(Cs, d);
      std::copy(inv.begin(), inv.end(), cinv.begin() + static_cast<long long>(s) * d * d);
      cmode[s] = 0;
    } else {
      // Thomas pivots (proj/src/deflation.cpp:77-90)
      double* sub = th.data() + static_cast<size_t>(s) * 3 * d;
      double* cp = sub + d;
      double* piv = cp + d;
      for (int i = 0; i + 1 < d; ++i) sub[i] = Cat(i + 1, i);
      piv[0] = Cat(0, 0);
      for (int i = 1; i < d; ++i) {
        cp[i - 1] = Cat(i - 1, i) / piv[i - 1];
        piv[i] = Cat(i, i) - sub[i - 1] * cp[i - 1];
      }
      for (int i = 0; i < d; ++i) {
        if (piv[i] == 0.0) fail(SMPM_ESINGULAR, "coarse matrix is singular");
        piv[i] = 1.0 / piv[i];  // the device multiplies by reciprocal pivots
      }
      cmode[s] = 1;
    }
  }
  cudaStream_t st = b->ctx->stream;
  if (!b->from_fdm) b->drowsum.upload(rows, st);
  b->dcinv.upload(cinv, st);
  b->duc.upload(uc, st);
  b->dthomas.upload(th, st);
  b->dcmode.upload(cmode, st);
  b->dsingular.upload(b->hsing, st);
}

SpecParams spec_params(const smpm_batch* b);

// --------------------------------------------------------------------------
// Device-side fast-diagonalisation setup (smpm_batch_set_fdm).
// Replaces, per system (Fourier mode), the reference's build_kind_coupling
// (proj/src/schur.cpp:19-69: one dense LU of a q x q strip block per kind, and
// per Helmholtz shift the real-Schur solves of proj/src/helmholtz.cpp:58-143)
// and the LU of every block-Jacobi block (proj/src/schur.cpp:188-216):
//   gamma_kind(mu)[q] = -tau sum_p a_kind[p] / (lx_kind[p] + lz[q] - mu)
//   G_kind[X,Y](mu)   = T diag(gamma_kind,XY) T^{-1}
//   K_v^{-1}[X,Y]     = T diag(kinv_v,XY) T^{-1}    (the reduced block inverses:
//                       K = I - G' D is diagonalised by T as well: no LU)
// Every dense block of a system's pool is T times a diagonally (pairs: 2 x 2)
// scaled T^{-1}: one scaling kernel and ONE launch of the shared-matrix
// transform kernel over all the pool's w-blocks.
// --------------------------------------------------------------------------
__global__ void fdm_gamma_kernel(int nsys, int nmode, int n, const double2* __restrict__ a,
                                 const double2* __restrict__ lx, const double2* __restrict__ lz,
                                 const double* __restrict__ mu, double tau, double2* __restrict__ gam) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(nsys) * SK_NUM * nmode) return;
  const int m = static_cast<int>(idx % nmode);
  const int kd = static_cast<int>((idx / nmode) % SK_NUM);
  const int s = static_cast<int>(idx / (static_cast<long long>(nmode) * SK_NUM));
  const double2 z = lz[m];
  double sr = 0.0, si = 0.0;
  for (int p = 0; p < n; ++p) {
    const double2 l = lx[kd * n + p], ap = a[kd * n + p];
    const double dr = l.x + z.x - mu[s], di = l.y + z.y;
    const double den = fma(dr, dr, di * di);
    sr += fma(ap.x, dr, ap.y * di) / den;
    si += fma(ap.y, dr, -ap.x * di) / den;
  }
  gam[idx] = make_double2(-tau * sr, -tau * si);
}

struct FdmRegion {
  int start, count;  // w-blocks [start, start + count) of a system's pool
  int type;          // 0: w x w block of gamma kind `idx`; 1: 2w x 2w interior coupling; 2: 2w x 2w K variant `idx`;
  int idx;           // 3: w x w single-interface inverse
};
struct FdmRegions {
  FdmRegion r[8];
  int n;
};

// M[s][cc][:] = Diag(cc) T^{-1}[:, c(cc)] for every w-block cc of the pools of systems [s0, s0 + ns)
__global__ void fdm_scale_kernel(FdmRegions R, int w, int npairs, int nmode, long long mstride, int s0,
                                 const double* __restrict__ Ti, const double2* __restrict__ gam,
                                 const double2* __restrict__ kinv, double* __restrict__ M) {
  const int cc = blockIdx.x, sl = blockIdx.y, s = s0 + sl;
  const double2* diag = nullptr;
  int c = 0;
  for (int q = 0; q < R.n; ++q) {
    const FdmRegion g = R.r[q];
    if (cc < g.start || cc >= g.start + g.count) continue;
    const int o = cc - g.start;
    if (g.type == 0) {
      diag = gam + (static_cast<long long>(s) * SK_NUM + g.idx) * nmode;
      c = o;
    } else if (g.type == 3) {
      diag = kinv + (static_cast<long long>(s) * 20 + 16) * nmode;
      c = o;
    } else {
      const int col = o >> 1, X = o & 1, Y = col >= w ? 1 : 0;
      c = col - Y * w;
      if (g.type == 1)
        diag = gam + (static_cast<long long>(s) * SK_NUM + (X == 0 ? (Y ? SK_I_WE : SK_I_WW) : (Y ? SK_I_EE : SK_I_EW))) * nmode;
      else
        diag = kinv + (static_cast<long long>(s) * 20 + g.idx * 4 + 2 * X + Y) * nmode;
    }
  }
  double* out = M + static_cast<long long>(sl) * mstride + static_cast<long long>(cc) * w;
  if (!diag) {  // padding past the last region
    for (int r = threadIdx.x; r < w; r += blockDim.x) out[r] = 0.0;
    return;
  }
  const double* tc = Ti + static_cast<long long>(c) * w;
  for (int m = threadIdx.x; m < nmode; m += blockDim.x) {
    const double2 g = diag[m];
    if (m < npairs) {
      // coordinates (a, b) <-> z = a - i b; z' = g z: a' = gr a + gi b, b' = gr b - gi a
      const double a = tc[2 * m], bb = tc[2 * m + 1];
      out[2 * m] = fma(g.x, a, g.y * bb);
      out[2 * m + 1] = fma(g.x, bb, -g.y * a);
    } else {
      out[npairs + m] = g.x * tc[npairs + m];
    }
  }
}

// strip row sums of the couplings (the fused deflation's S Z c): rW_I(2w) rE_I(2w) rE_W(w) rW_E(w)
__global__ void fdm_rowsum_kernel(int w, long long mstride, long long oGW, long long oGI, long long oGE,
                                  const double* __restrict__ pool, double* __restrict__ rows) {
  const int s = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 2 * w) return;
  const double* base = pool + static_cast<long long>(s) * mstride;
  double* rs = rows + static_cast<long long>(s) * 6 * w;
  double a = 0.0, e = 0.0;
  for (int c = 0; c < w; ++c) {
    a += base[oGI + static_cast<long long>(c) * 2 * w + r];
    e += base[oGI + static_cast<long long>(c + w) * 2 * w + r];
  }
  rs[r] = a;
  rs[2 * w + r] = e;
  if (r < w) {
    double gw = 0.0, ge = 0.0;
    for (int c = 0; c < w; ++c) {
      gw += base[oGW + static_cast<long long>(c) * w + r];
      ge += base[oGE + static_cast<long long>(c) * w + r];
    }
    rs[4 * w + r] = gw;
    rs[5 * w + r] = ge;
  }
}

void fdm_gamma(smpm_batch* b, cudaStream_t st) {
  const int n = b->n, nm = b->sp_nmode;
  DevArray<double> da, dlx, dlz, dmu;
  da.upload(b->fdm_a, st);
  dlx.upload(b->fdm_lx, st);
  dlz.upload(b->fdm_lz, st);
  dmu.upload(b->fdm_mu, st);
  b->dgam.alloc(static_cast<size_t>(b->nsys) * SK_NUM * nm * 2);
  const long long tot = static_cast<long long>(b->nsys) * SK_NUM * nm;
  fdm_gamma_kernel<<<static_cast<int>((tot + 127) / 128), 128, 0, st>>>(
      b->nsys, nm, n, reinterpret_cast<const double2*>(da.p), reinterpret_cast<const double2*>(dlx.p),
      reinterpret_cast<const double2*>(dlz.p), dmu.p, b->fdm_tau, reinterpret_cast<double2*>(b->dgam.p));
  check_launch(b);
  CUDA_CHECK(cudaStreamSynchronize(st));  // the staging arrays go out of scope
}

// dense couplings, block-Jacobi inverses and row sums of every system, on the device
void fdm_device_setup(smpm_batch* b, cudaStream_t st) {
  const int w = b->w;
  const long long ww = 1LL * w * w;
  if (b->xf_P == 0) fail(SMPM_EINVAL, "smpm_batch_set_fdm needs w % 16 == 0 (the shared-matrix transform kernels)");
  if (b->mstride % w != 0) fail(SMPM_ERUNTIME, "pool stride is not a whole number of w-blocks");
  FdmRegions R{};
  auto add = [&](long long off, long long count, int type, int idx) {
    R.r[R.n++] = FdmRegion{static_cast<int>(off / w), static_cast<int>(count), type, idx};
  };
  add(b->oGW, w, 0, SK_W_EE);
  add(b->oGI, 4LL * w, 1, 0);
  add(b->oGE, w, 0, SK_E_WW);
  for (int v = 0; v < 4; ++v)
    if (b->kneeded[v]) add(b->oK[v], 4LL * w, 2, v);
  if (b->single) add(b->oKs, w, 3, 0);
  const int nblk = static_cast<int>(b->mstride / w);
  // systems per pass: scaled T^{-1} copies of at most ~1.5 GB
  const int chunk = static_cast<int>(std::max<long long>(1, std::min<long long>(b->nsys, (3LL << 27) / b->mstride)));
  DevArray<double> M;
  M.alloc(static_cast<size_t>(chunk) * b->mstride);
  for (int s0 = 0; s0 < b->nsys; s0 += chunk) {
    const int ns = std::min(chunk, b->nsys - s0);
    fdm_scale_kernel<<<dim3(nblk, ns), 128, 0, st>>>(R, w, b->sp_npairs, b->sp_nmode, b->mstride, s0, b->dTi.p,
                                                       reinterpret_cast<const double2*>(b->dgam.p),
                                                       reinterpret_cast<const double2*>(b->dkinv.p), M.p);
    check_launch(b);
    xf_columns(b, false, M.p, b->dmat.p + static_cast<long long>(s0) * b->mstride, nblk, b->mstride, st, ns);
  }
  b->drowsum.alloc(static_cast<size_t>(b->nsys) * 6 * w);
  fdm_rowsum_kernel<<<dim3((2 * w + 127) / 128, b->nsys), 128, 0, st>>>(w, b->mstride, b->oGW, b->oGI, b->oGE, b->dmat.p,
                                                                       b->drowsum.p);
  check_launch(b);
  CUDA_CHECK(cudaStreamSynchronize(st));
  (void)ww;
}

void finalize(smpm_batch* b) {
  if (b->finalized) return;
  for (int s = 0; s < b->nsys; ++s)
    if (!b->have[s]) fail(SMPM_EINVAL, "smpm_batch_finalize: couplings of system " + std::to_string(s) + " not set");
  const int w = b->w, mx = b->mx, d = b->d;
  cudaStream_t st = b->ctx->stream;
  // which K variants occur ([first][last] over the two-interface blocks)
  for (int bb = 0; bb < b->nbf; ++bb) b->kneeded[(bb == 0 ? 1 : 0) | (2 * bb + 2 == mx - 1 ? 2 : 0)] = true;
  long long off = 0;
  b->oGW = off;
  off += 1LL * w * w;
  b->oGI = off;
  off += 4LL * w * w;
  b->oGE = off;
  off += 1LL * w * w;
  for (int v = 0; v < 4; ++v)
    if (b->kneeded[v]) {
      b->oK[v] = off;
      off += 4LL * w * w;
    }
  if (b->single) {
    b->oKs = off;
    off += 1LL * w * w;
  }
  b->mstride = (off + 31) / 32 * 32;
  b->dmat.alloc(static_cast<size_t>(b->mstride) * b->nsys);
  if (!b->from_fdm)
    for (int s = 0; s < b->nsys; ++s)
      CUDA_CHECK(cudaMemcpyAsync(b->GW(s), b->hG.data() + s * 6LL * w * w, sizeof(double) * 6LL * w * w,
                                 cudaMemcpyHostToDevice, st));
  if (b->spectral) {
    b->dT.upload(b->hT, st);
    b->dTi.upload(b->hTi, st);
    if (b->from_fdm)
      fdm_gamma(b, st);
    else
      b->dgam.upload(b->hgam, st);
    std::vector<double> om(static_cast<size_t>(w), 0.0);  // omega = T^T 1
    for (int e = 0; e < w; ++e)
      for (int r = 0; r < w; ++r) om[e] += b->hT[static_cast<size_t>(e) * w + r];
    b->domega.upload(om, st);
    std::vector<double> nu(static_cast<size_t>(w), 0.0);  // nu = T^{-1} 1
    for (int c2 = 0; c2 < w; ++c2)
      for (int r = 0; r < w; ++r) nu[r] += b->hTi[static_cast<size_t>(c2) * w + r];
    b->dnu.upload(nu, st);
    const int nmc = (b->sp_nmode + SP_MODES - 1) / SP_MODES;
    b->dzpart.alloc(static_cast<size_t>(b->nsys) * std::max(nmc, spec3_chunks(b->sp_npairs, b->sp_nmode)) * d);
    b->dkinv.alloc(static_cast<size_t>(b->nsys) * 20 * b->sp_nmode * 2);
    b->dvh.alloc(static_cast<size_t>(b->nsys) * b->k);
    b->dth.alloc(static_cast<size_t>(b->nsys) * b->k);
    b->dvh2.alloc(static_cast<size_t>(b->nsys) * b->k);
  }
  build_plans(b);
  if (b->spectral && !(b->pF.v2 && b->pB.v2)) b->spectral = false;  // odd w: dense operator path
  if (b->spectral) setup_xform(b);
  if (b->spectral) {
    const SpecParams sp = spec_params(b);
    const long long n = 1LL * b->nsys * b->sp_nmode;
    spec_setup_kernel<<<static_cast<int>((n + 127) / 128), 128, 0, st>>>(sp, reinterpret_cast<double2*>(b->dkinv.p), b->nsys);
    check_launch(b);
  }
  if (b->from_fdm) {
    if (!b->spectral) fail(SMPM_EINVAL, "smpm_batch_set_fdm needs an even interface width w");
    fdm_device_setup(b, st);
  } else {
    build_bj_inverses(b);
  }
  build_coarse(b);
  std::vector<double>().swap(b->hG);  // the host staging copy is not needed any more
  for (auto& v : b->vbuf) v.alloc(static_cast<size_t>(b->nsys) * b->k);
  b->dsmall.alloc(static_cast<size_t>(b->nsys) * (d + 8));
  b->dcoarse.alloc(static_cast<size_t>(b->nsys) * 2 * d);
  b->dczb.alloc(static_cast<size_t>(b->nsys) * d);
  b->dpost.alloc(static_cast<size_t>(b->nsys) * 64);
  std::vector<int> ones(static_cast<size_t>(b->nsys), 1);
  b->dones.upload(ones, st);
  b->dcount.alloc(static_cast<size_t>(b->nsys) + 1);
  CUDA_CHECK(cudaMemsetAsync(b->dcount.p, 0, sizeof(int) * (b->nsys + 1), st));
  b->dsel.alloc(static_cast<size_t>(b->nsys));
  b->dalist.alloc(2 * static_cast<size_t>(b->nsys) + 2);
  b->dcnt.alloc(4);
  CUDA_CHECK(cudaHostAlloc(&b->hcnt, 4 * sizeof(int), cudaHostAllocMapped));
  CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&b->hcnt_dev), b->hcnt, 0));
  b->dearly.alloc(4 * static_cast<size_t>(b->nsys) + 2);
  CUDA_CHECK(cudaHostAlloc(&b->hearly, sizeof(int) * b->nsys, cudaHostAllocMapped));
  CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&b->hearly_dev), b->hearly, 0));
  CUDA_CHECK(cudaStreamSynchronize(st));
  b->finalized = true;
}

void need_final(smpm_batch* b) {
  if (!b || !b->finalized) fail(SMPM_EINVAL, "batch not finalized");
}
