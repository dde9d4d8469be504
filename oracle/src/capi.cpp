// ORACLE — TEST INFRASTRUCTURE ONLY. C entry points used by tests/ (ctypes),
// __graft_entry__.smoke() and bench.py's CPU-baseline legs. Not the product.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "smpm.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return E_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_RUNTIME;
  }
}

struct Problem {
  std::shared_ptr<Operator> op;
};
struct System {
  std::shared_ptr<Operator> op;
  SchurSystem sys;
};

Vec vin(const double* p, Index n) { return Vec(p, p + n); }
void vout(const Vec& v, double* p) { std::copy(v.begin(), v.end(), p); }

struct Report {
  int iterations, converged, mismatch, history_len;
  long long operator_applies, krylov_s_applies;
  double final_rel_residual, wall_time_s;
};

void fill_report(const SchurSolveResult& r, Report* rep, double* hist, int cap) {
  if (!rep) return;
  rep->iterations = r.report.iterations;
  rep->converged = r.report.converged ? 1 : 0;
  rep->mismatch = r.report.mismatch ? 1 : 0;
  rep->history_len = static_cast<int>(r.report.history.size());
  rep->operator_applies = r.report.operator_applies;
  rep->krylov_s_applies = static_cast<long long>(r.krylov_s_applies);
  rep->final_rel_residual = r.report.final_rel_residual;
  rep->wall_time_s = r.report.wall_time_s;
  if (hist)
    for (int i = 0; i < std::min(cap, rep->history_len); ++i) hist[i] = r.report.history[i];
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// n uniforms of Rng(seed) (stream < 0) or Rng(seed).stream(stream) (proj/include/smpm/rng.hpp)
int orc_rng_uniforms(unsigned long long seed, long long stream, int n, double* out) {
  return guard([&] {
    Rng r = stream < 0 ? Rng(seed) : Rng(seed).stream(static_cast<std::uint64_t>(stream));
    for (int i = 0; i < n; ++i) out[i] = r.uniform();
  });
}

int orc_set_threads(int n) {
  return guard([&] { set_blas_threads(n); });
}

int orc_gll(int n, double* nodes, double* weights, double* diff) {
  return guard([&] {
    const Gll g = gll_basis(n);
    vout(g.nodes, nodes);
    vout(g.weights, weights);
    std::copy(g.diff.a.begin(), g.diff.a.end(), diff);
  });
}

void* orc_problem_create(int n, int mx, int mz, double lx, double lz, double c_tau) {
  Problem* p = nullptr;
  const int rc = guard([&] {
    const Mesh mesh = build_mesh(n, mx, mz, lx, lz);
    const Decomposition dec = build_decomposition(mesh);
    const double tau = penalty_tau(n, mesh.h_x, mesh.h_z, c_tau);
    p = new Problem{std::make_shared<Operator>(assemble_operator(mesh, dec, tau))};
  });
  return rc == E_OK ? p : nullptr;
}

void orc_problem_free(void* p) { delete static_cast<Problem*>(p); }

// info: r, k, d, w, q, nkinds ; dinfo: tau, h_x, h_z, eta
int orc_problem_info(void* vp, long long* info, double* dinfo) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    info[0] = op.dec.r;
    info[1] = op.dec.k;
    info[2] = op.dec.d;
    info[3] = op.dec.side();
    info[4] = op.q;
    info[5] = static_cast<long long>(op.kinds.size());
    dinfo[0] = op.tau;
    dinfo[1] = op.mesh.h_x;
    dinfo[2] = op.mesh.h_z;
    dinfo[3] = op.mesh.eta;
  });
}

int orc_problem_coords(void* vp, double* x, double* z) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    vout(op.mesh.x, x);
    vout(op.mesh.z, z);
  });
}

int orc_gamma_to_node(void* vp, long long* out) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    for (Index p = 0; p < op.dec.k; ++p) out[p] = op.dec.gamma_to_node[p];
  });
}

int orc_strip_matrix(void* vp, int strip, double* out) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    if (strip < 0 || strip >= op.mesh.m_x) invalid("strip_matrix: bad strip");
    const Mat& a = op.a[op.kind_of[strip]];
    std::copy(a.a.begin(), a.a.end(), out);
  });
}

#define PROB_OP(name, fn, nin)                                              \
  int name(void* vp, const double* in, double* out) {                       \
    return guard([&] {                                                      \
      const Operator& op = *static_cast<Problem*>(vp)->op;                  \
      vout(fn(op, vin(in, nin)), out);                                      \
    });                                                                     \
  }
PROB_OP(orc_apply_A, apply_A, op.dec.r)
PROB_OP(orc_apply_B, apply_B, op.dec.r)
PROB_OP(orc_apply_Bt, apply_Bt, op.dec.k)
PROB_OP(orc_apply_L, apply_L, op.dec.r)
PROB_OP(orc_solve_A, solve_A, op.dec.r)
PROB_OP(orc_solve_At, solve_At, op.dec.r)
#undef PROB_OP

int orc_apply_E(void* vp, const double* v, double* u) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    vout(apply_E(op.dec, vin(v, op.dec.k)), u);
  });
}
int orc_apply_Et(void* vp, const double* u, double* v) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    vout(apply_Et(op.dec, vin(u, op.dec.r)), v);
  });
}
int orc_apply_Z(void* vp, const double* y, double* v) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    vout(apply_Z(op.dec, vin(y, op.dec.d)), v);
  });
}
int orc_apply_Zt(void* vp, const double* v, double* y) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    vout(apply_Zt(op.dec, vin(v, op.dec.k)), y);
  });
}

int orc_dense_L(void* vp, double* out) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    const Mat L = dense_L(op.mesh, op.tau);
    std::copy(L.a.begin(), L.a.end(), out);
  });
}

int orc_shifted_solve(void* vp, double mu, const double* b, double* x) {
  return guard([&] {
    Operator& op = *static_cast<Problem*>(vp)->op;
    factor_unshifted_blocks(op);
    vout(shifted_solve(op, mu, vin(b, op.dec.r)), x);
  });
}

// Manufactured fields at the node coordinates shifted by (+l_x/2, +l_z/2):
// u = sum_{k,l=0..kmax} a_kl cos(k pi x/l_x) cos(l pi z/l_z), a_kl ~ N(0,1)
// (optionally / (1+k^2+l^2)), drawn k-major from Rng(seed).stream(stream).
// forcing_only = 0: f = Lap(u) (g = 0 exactly, so the assembled rhs is f);
// forcing_only = 1: f = the cosine series itself (per-mode Helmholtz forcing).
// mu > 0 (with forcing_only = 0): f = (Lap - mu) u, the manufactured
// per-mode Helmholtz right-hand side.
int orc_manufactured(void* vp, int kmax, int decay, unsigned long long seed, unsigned long long stream,
                     int forcing_only, double mu, double* f, double* u) {
  return guard([&] {
    const Operator& op = *static_cast<Problem*>(vp)->op;
    const Mesh& m = op.mesh;
    Rng rng = Rng(seed).stream(stream);
    std::vector<double> a(static_cast<std::size_t>((kmax + 1) * (kmax + 1)));
    for (int k = 0; k <= kmax; ++k)
      for (int l = 0; l <= kmax; ++l) {
        double c = rng.normal();
        if (decay) c /= 1.0 + k * k + l * l;
        a[static_cast<std::size_t>(k * (kmax + 1) + l)] = c;
      }
    for (Index g = 0; g < m.r; ++g) {
      const double x = m.x[g] + 0.5 * m.l_x, z = m.z[g] + 0.5 * m.l_z;
      double fs = 0.0, us = 0.0;
      for (int k = 0; k <= kmax; ++k) {
        const double ck = std::cos(k * M_PI * x / m.l_x);
        const double kk = k * M_PI / m.l_x;
        for (int l = 0; l <= kmax; ++l) {
          const double c = a[static_cast<std::size_t>(k * (kmax + 1) + l)];
          const double ll = l * M_PI / m.l_z;
          const double mode = ck * std::cos(l * M_PI * z / m.l_z);
          us += c * mode;
          fs += forcing_only ? c * mode : -c * (kk * kk + ll * ll + mu) * mode;
        }
      }
      f[g] = fs;
      if (u) u[g] = us;
    }
  });
}

void* orc_system_create(void* vp, double mu, int layout_reference) {
  System* s = nullptr;
  const int rc = guard([&] {
    auto op = static_cast<Problem*>(vp)->op;
    s = new System{op, assemble_schur(op, mu, layout_reference != 0)};
  });
  return rc == E_OK ? s : nullptr;
}

void* orc_system_from_kinds(void* vp, double mu, const double* GW, const double* GI, const double* GE,
                            int layout_reference) {
  System* s = nullptr;
  const int rc = guard([&] {
    auto op = static_cast<Problem*>(vp)->op;
    s = new System{op, schur_from_kinds(op, mu, GW, GI, GE, layout_reference != 0)};
  });
  return rc == E_OK ? s : nullptr;
}

void orc_system_free(void* s) { delete static_cast<System*>(s); }

int orc_system_frob(void* vs, double* frob) {
  return guard([&] { *frob = static_cast<System*>(vs)->sys.frob; });
}

int orc_export_kinds(void* vs, double* GW, double* GI, double* GE) {
  return guard([&] { export_kinds(static_cast<System*>(vs)->sys, GW, GI, GE); });
}

int orc_build_bj(void* vs, int dedup) {
  return guard([&] { build_block_jacobi(static_cast<System*>(vs)->sys, dedup); });
}

unsigned long long orc_applies(void* vs) { return static_cast<System*>(vs)->sys.applies->load(); }

#define SYS_OP(name, fn, nin)                                    \
  int name(void* vs, const double* in, double* out) {            \
    return guard([&] {                                           \
      const SchurSystem& sys = static_cast<System*>(vs)->sys;    \
      vout(fn(sys, vin(in, nin)), out);                          \
    });                                                          \
  }
SYS_OP(orc_apply_S, apply_S, sys.k)
SYS_OP(orc_apply_St, apply_St, sys.k)
SYS_OP(orc_apply_S_definition, apply_S_definition, sys.k)
SYS_OP(orc_bj_inv, apply_block_jacobi_inv, sys.k)
SYS_OP(orc_schur_rhs, schur_rhs, sys.op->dec.r)
#undef SYS_OP

int orc_recover(void* vs, const double* f, const double* xs, double* u) {
  return guard([&] {
    const SchurSystem& sys = static_cast<System*>(vs)->sys;
    vout(recover_solution(sys, vin(f, sys.op->dec.r), vin(xs, sys.k)), u);
  });
}

int orc_dense_S(void* vs, double* out) {
  return guard([&] {
    const Mat s = dense_schur(static_cast<System*>(vs)->sys);
    std::copy(s.a.begin(), s.a.end(), out);
  });
}

int orc_nullspace(void* vs, double* u_S, double* u_L, int* its, double* sigma, long long dense_limit) {
  return guard([&] {
    const SchurSystem& sys = static_cast<System*>(vs)->sys;
    int it = 0;
    double sg = 0.0;
    const Vec us = left_null_vector_s(sys, 0.0, 1e-10, 25, &it, &sg, dense_limit);
    vout(us, u_S);
    if (u_L) vout(left_null_vector_l(*sys.op, us), u_L);
    if (its) *its = it;
    if (sigma) *sigma = sg;
  });
}

int orc_project_out(long long n, const double* v, const double* dir, double* out) {
  return guard([&] { vout(project_out(vin(v, n), vin(dir, n)), out); });
}

void* orc_coarse_create(void* vs, const double* u_S) {
  CoarseSpace* c = nullptr;
  const int rc = guard([&] {
    const SchurSystem& sys = static_cast<System*>(vs)->sys;
    if (u_S) {
      const Vec us = vin(u_S, sys.k);
      c = new CoarseSpace(build_coarse(sys, &us));
    } else {
      c = new CoarseSpace(build_coarse(sys, nullptr));
    }
  });
  return rc == E_OK ? c : nullptr;
}

void orc_coarse_free(void* c) { delete static_cast<CoarseSpace*>(c); }

int orc_coarse_info(void* vc, int* singular_out, int* tridiagonal, double* C, double* u_C) {
  return guard([&] {
    const CoarseSpace& cs = *static_cast<CoarseSpace*>(vc);
    *singular_out = cs.singular ? 1 : 0;
    *tridiagonal = cs.tridiagonal ? 1 : 0;
    if (C) std::copy(cs.C.a.begin(), cs.C.a.end(), C);
    if (u_C && cs.singular) vout(cs.u_C, u_C);
  });
}

int orc_coarse_solve(void* vc, const double* b, double* x) {
  return guard([&] {
    const CoarseSpace& cs = *static_cast<CoarseSpace*>(vc);
    vout(coarse_solve(cs, vin(b, cs.d)), x);
  });
}

int orc_apply_P(void* vc, void* vs, const double* v, double* y) {
  return guard([&] {
    const SchurSystem& sys = static_cast<System*>(vs)->sys;
    vout(apply_P(*static_cast<CoarseSpace*>(vc), sys, vin(v, sys.k)), y);
  });
}

int orc_apply_Q(void* vc, void* vs, const double* v, double* y) {
  return guard([&] {
    const SchurSystem& sys = static_cast<System*>(vs)->sys;
    vout(apply_Q(*static_cast<CoarseSpace*>(vc), sys, vin(v, sys.k)), y);
  });
}

// method: 0 schur, 1 bj, 2 dbj, 3 2las (proj/src/solver.cpp:11, 76-89)
int orc_solve(void* vs, void* vc, int method, const double* b, double tol, int max_iter, int restart, double* x,
              Report* rep, double* hist, int cap) {
  return guard([&] {
    const SchurSystem& sys = static_cast<System*>(vs)->sys;
    const Vec bs = vin(b, sys.k);
    SchurSolveResult r;
    const CoarseSpace* cs = static_cast<CoarseSpace*>(vc);
    switch (method) {
      case 0: r = plain_solve(sys, bs, tol, max_iter, restart); break;
      case 1: r = bj_solve(sys, bs, tol, max_iter, restart); break;
      case 2:
        if (!cs) invalid("dbj needs a coarse space");
        r = deflated_solve(sys, *cs, bs, tol, max_iter, restart);
        break;
      case 3:
        if (!cs) invalid("2las needs a coarse space");
        r = two_level_schwarz_solve(sys, *cs, bs, tol, max_iter, restart);
        break;
      default: invalid("unknown method");
    }
    vout(r.x_S, x);
    fill_report(r, rep, hist, cap);
  });
}

// proj/src/schur.cpp:246-264 (dump_schur_blocks): the reference's binary block file
// (int64 n, m_x, m_z, k; per interface block: rows, cols, nseg, (start, len) x nseg,
// then the column-major entries). Needs the materialized reference layout.
int orc_dump_schur_blocks(void* vs, const char* path) {
  return guard([&] {
    const SchurSystem& sys = static_cast<System*>(vs)->sys;
    if (!sys.materialized) invalid("dump_schur_blocks: needs the reference per-interface layout");
    std::FILE* fp = std::fopen(path, "wb");
    if (!fp) runtime(std::string("dump_schur_blocks: cannot open ") + path);
    auto put = [&](std::int64_t v) { std::fwrite(&v, sizeof v, 1, fp); };
    put(sys.op->mesh.n);
    put(sys.op->mesh.m_x);
    put(sys.op->mesh.m_z);
    put(sys.k);
    for (const auto& blk : sys.blocks) {
      put(blk.entries.rows);
      put(blk.entries.cols);
      put(static_cast<std::int64_t>(blk.segs.size()));
      for (const auto& sg : blk.segs) {
        put(sg.first);
        put(sg.second);
      }
      std::fwrite(blk.entries.data(), sizeof(double), blk.entries.a.size(), fp);
    }
    std::fclose(fp);
  });
}

// Stacked solve (proj/src/helmholtz.cpp:187-246, the reference bench's 3D
// default, proj/src/bench.cpp:129): ONE GMRES over the concatenation of every
// system's right-hand side (dbj: P_j b_j) with the block-diagonal operator
// (dbj: P_j S_j M_j^{-1}; 2las: S_j (M_j^{-1} + Z c_j Z^T)), abs_tol = tol *
// sqrt(sum_j ||b_j||^2); then per system x_j = Q_j M_j^{-1} x'_j + Z c_j(Z^T b_j)
// (dbj) or M_j^{-1} x'_j + Z c_j(Z^T x'_j) (2las). One report.
int orc_solve_stacked(void** systems, void** coarse, int nsys, int method, const double* b, double tol, int max_iter,
                      int restart, double* x, Report* rep, double* hist, int cap) {
  return guard([&] {
    if (nsys < 1) invalid("no systems");
    if (method != 2 && method != 3) invalid("stacked solve: dbj or 2las");
    std::vector<const SchurSystem*> S(static_cast<std::size_t>(nsys));
    std::vector<const CoarseSpace*> CS(static_cast<std::size_t>(nsys));
    for (int j = 0; j < nsys; ++j) {
      S[j] = &static_cast<System*>(systems[j])->sys;
      CS[j] = static_cast<CoarseSpace*>(coarse[j]);
      if (!CS[j]) invalid("stacked solve needs coarse spaces");
    }
    const Index k = S[0]->k;
    const Index total = static_cast<Index>(nsys) * k;
    Vec rhs(static_cast<std::size_t>(total));
    double bnorm2 = 0.0;
    for (int j = 0; j < nsys; ++j) {
      const Vec bj = vin(b + static_cast<Index>(j) * k, k);
      for (double v : bj) bnorm2 += v * v;
      const Vec pj = method == 2 ? apply_P(*CS[j], *S[j], bj) : bj;
      std::copy(pj.begin(), pj.end(), rhs.begin() + static_cast<Index>(j) * k);
    }
    auto seg = [&](const Vec& v, int j) { return Vec(v.begin() + static_cast<Index>(j) * k, v.begin() + static_cast<Index>(j + 1) * k); };
    LinOp op = [&](const Vec& v) {
      Vec y(static_cast<std::size_t>(total));
      for (int j = 0; j < nsys; ++j) {
        const Vec vj = seg(v, j);
        const SchurSystem& sj = *S[j];
        const Decomposition& dec = sj.op->dec;
        Vec w;
        if (method == 2) {
          w = apply_P(*CS[j], sj, apply_S(sj, apply_block_jacobi_inv(sj, vj)));
        } else {
          Vec m = apply_block_jacobi_inv(sj, vj);
          const Vec zc = apply_Z(dec, coarse_solve(*CS[j], apply_Zt(dec, vj)));
          for (std::size_t i = 0; i < m.size(); ++i) m[i] += zc[i];
          w = apply_S(sj, m);
        }
        std::copy(w.begin(), w.end(), y.begin() + static_cast<Index>(j) * k);
      }
      return y;
    };
    GmresOptions opt;
    opt.abs_tol = tol * std::sqrt(bnorm2);
    opt.max_iter = max_iter;
    opt.restart = restart;
    SchurSolveResult r;
    const Vec xp = gmres(op, rhs, opt, r.report);
    for (int j = 0; j < nsys; ++j) {
      const SchurSystem& sj = *S[j];
      const Decomposition& dec = sj.op->dec;
      const Vec xj = seg(xp, j);
      Vec out;
      if (method == 2) {
        out = apply_Q(*CS[j], sj, apply_block_jacobi_inv(sj, xj));
        const Vec zc = apply_Z(dec, coarse_solve(*CS[j], apply_Zt(dec, vin(b + static_cast<Index>(j) * k, k))));
        for (std::size_t i = 0; i < out.size(); ++i) out[i] += zc[i];
      } else {
        out = apply_block_jacobi_inv(sj, xj);
        const Vec zc = apply_Z(dec, coarse_solve(*CS[j], apply_Zt(dec, xj)));
        for (std::size_t i = 0; i < out.size(); ++i) out[i] += zc[i];
      }
      vout(out, x + static_cast<Index>(j) * k);
    }
    fill_report(r, rep, hist, cap);
  });
}

// Independent per-system deflated solves across host threads (the
// `parallel_trials` analogue, proj/src/bench.cpp:79-84). systems[i] and
// coarse[i] pair up; b and x are nsys x k, system-major.
int orc_solve_many(void** systems, void** coarse, int nsys, int method, const double* b, double tol, int max_iter,
                   int restart, double* x, Report* reps, int threads) {
  return guard([&] {
    std::vector<std::string> errs(static_cast<std::size_t>(nsys));
    const int nt = std::max(1, std::min(threads, nsys));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (int i = t; i < nsys; i += nt) {
          const SchurSystem& sys = static_cast<System*>(systems[i])->sys;
          try {
            const Vec bs = vin(b + static_cast<Index>(i) * sys.k, sys.k);
            const CoarseSpace& cs = *static_cast<CoarseSpace*>(coarse[i]);
            SchurSolveResult r = method == 3 ? two_level_schwarz_solve(sys, cs, bs, tol, max_iter, restart)
                                             : deflated_solve(sys, cs, bs, tol, max_iter, restart);
            vout(r.x_S, x + static_cast<Index>(i) * sys.k);
            fill_report(r, reps ? reps + i : nullptr, nullptr, 0);
          } catch (const std::exception& e) {
            errs[static_cast<std::size_t>(i)] = e.what();
          }
        }
      });
    for (auto& x_ : th) x_.join();
    for (const auto& e : errs)
      if (!e.empty()) runtime(e);
  });
}

// GMRES core on an explicit dense operator (SPEC gmres examples, criterion 6)
int orc_gmres_dense(long long n, const double* A, const double* b, double tol, int max_iter, int restart, double* x,
                    Report* rep, double* hist, int cap) {
  return guard([&] {
    LinOp op = [&](const Vec& v) {
      Vec y(static_cast<std::size_t>(n), 0.0);
      gemv_acc(A, n, n, n, v.data(), y.data());
      return y;
    };
    GmresOptions opt;
    opt.rel_tol = tol;
    opt.max_iter = max_iter;
    opt.restart = restart;
    SchurSolveResult r;
    r.x_S = gmres(op, vin(b, n), opt, r.report);
    vout(r.x_S, x);
    fill_report(r, rep, hist, cap);
  });
}

}  // extern "C"
