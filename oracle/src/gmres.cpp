// ORACLE — TEST INFRASTRUCTURE ONLY. Restates /root/reference/proj/src/gmres.cpp
// (Householder-Arnoldi GMRES) and the solve drivers of
// /root/reference/proj/src/deflation.cpp:102-143 and proj/src/solver.cpp:56-75.
#include <algorithm>
#include <chrono>
#include <cmath>

#include "smpm.hpp"

namespace orc {

namespace {

// v -= w (2 w.v); w_j vanishes above row j so the loops start there
// (identical values: the skipped terms are exact zeros) — proj/src/gmres.cpp:11-14
inline void reflect(const Mat& W, Index j, double* v, Index nn) {
  const double* wj = W.col(j);
  const double s = 2.0 * dot(wj + j, v + j, nn - j);
  for (Index i = j; i < nn; ++i) v[i] -= wj[i] * s;
}

struct CycleOut {
  Vec x;          // correction from this cycle
  int iters = 0;
  bool converged = false, breakdown = false;
  double g_last = 0.0;  // |g(iters)|
};

// One Householder-Arnoldi cycle on rhs r, at most m iterations
// (proj/src/gmres.cpp:35-125).
CycleOut householder_cycle(const LinOp& op, const Vec& r, int m, double target, double bnorm, KrylovReport& rep) {
  const Index nn = static_cast<Index>(r.size());
  CycleOut out;
  out.x.assign(r.size(), 0.0);
  // workspace grows by doubling from 64 columns (proj/src/gmres.cpp:35-56)
  int cap = std::min(m, 64);
  Mat W(nn, cap + 1), V(nn, std::max(cap, 1)), R(m + 1, std::max(m, 1));
  auto grow = [&](int need) {
    if (need <= cap) return;
    cap = std::min(m, 2 * cap);
    W.a.resize(static_cast<std::size_t>(nn * (cap + 1)), 0.0);
    W.cols = cap + 1;
    V.a.resize(static_cast<std::size_t>(nn * cap), 0.0);
    V.cols = cap;
  };
  Vec g(static_cast<std::size_t>(m + 1), 0.0), cs(static_cast<std::size_t>(m), 0.0), sn(static_cast<std::size_t>(m), 0.0);
  Vec z = r;
  double h_max = 0.0;
  int iters = 0;
  Vec h(static_cast<std::size_t>(m + 1));
  for (int j = 0; j <= m; ++j) {
    grow(j + 1);
    const double sigma = norm2(z.data() + j, nn - j);
    double alpha = 0.0;
    double* wj = W.col(j);
    std::fill(wj, wj + nn, 0.0);
    if (sigma > 0.0) {
      alpha = z[j] >= 0.0 ? -sigma : sigma;
      std::copy(z.begin() + j, z.end(), wj + j);
      wj[j] -= alpha;
      const double wn = norm2(wj, nn);
      if (wn > 0.0)
        for (Index i = j; i < nn; ++i) wj[i] /= wn;
    }
    if (j == 0) {
      g[0] = alpha;
    } else {
      for (int i = 0; i < j; ++i) h[i] = z[i];
      h[j] = alpha;
      for (int i = 0; i <= j; ++i) h_max = std::max(h_max, std::abs(h[i]));
      for (int i = 0; i + 1 < j; ++i) {
        const double t1 = h[i], t2 = h[i + 1];
        h[i] = cs[i] * t1 + sn[i] * t2;
        h[i + 1] = -sn[i] * t1 + cs[i] * t2;
      }
      const double rad = std::hypot(h[j - 1], h[j]);
      cs[j - 1] = rad > 0.0 ? h[j - 1] / rad : 1.0;
      sn[j - 1] = rad > 0.0 ? h[j] / rad : 0.0;
      h[j - 1] = rad;
      const double g1 = g[j - 1], g2 = g[j];
      g[j - 1] = cs[j - 1] * g1 + sn[j - 1] * g2;
      g[j] = -sn[j - 1] * g1 + cs[j - 1] * g2;
      for (int i = 0; i < j; ++i) R(i, j - 1) = h[i];
      iters = j;
      const double res_abs = std::abs(g[j]);
      rep.history.push_back(res_abs / bnorm);
      if (res_abs <= target) {
        out.converged = true;
        break;
      }
      if (std::abs(alpha) <= 1e-14 * h_max) {
        out.breakdown = true;
        break;
      }
    }
    if (j == m) break;
    // v_j = P_0 ... P_j e_j
    Vec v(static_cast<std::size_t>(nn), 0.0);
    v[j] = 1.0;
    for (int i = j; i >= 0; --i) reflect(W, i, v.data(), nn);
    std::copy(v.begin(), v.end(), V.col(j));
    // z = P_j ... P_0 op(v_j)
    z = op(v);
    ++rep.operator_applies;
    if (!all_finite(z)) throw Error(E_NONFINITE, "gmres: operator produced non-finite values");
    for (int i = 0; i <= j; ++i) reflect(W, i, z.data(), nn);
  }
  out.iters = iters;
  if (iters > 0) {
    Vec y(static_cast<std::size_t>(iters), 0.0);
    for (int i = iters - 1; i >= 0; --i) {
      double acc = g[i];
      for (int c = i + 1; c < iters; ++c) acc -= R(i, c) * y[c];
      y[i] = std::abs(R(i, i)) > 0.0 ? acc / R(i, i) : 0.0;
    }
    for (int c = 0; c < iters; ++c) {
      const double* vc = V.col(c);
      const double yc = y[c];
      for (Index i = 0; i < nn; ++i) out.x[i] += vc[i] * yc;
    }
  }
  out.g_last = std::abs(g[iters]);
  return out;
}

}  // namespace

// proj/src/gmres.cpp:18-142. With opt.restart == 0 this is the reference
// algorithm exactly; restart > 0 is this repo's GMRES(m) extension: after m
// inner iterations without convergence the correction is accumulated, the
// residual b - op(x) recomputed explicitly and a new cycle started.
Vec gmres(const LinOp& op, const Vec& b, const GmresOptions& opt, KrylovReport& rep) {
  const auto t0 = std::chrono::steady_clock::now();
  const Index nn = static_cast<Index>(b.size());
  Vec x(b.size(), 0.0);
  rep = KrylovReport{};
  rep.history.push_back(1.0);
  const double bnorm = norm2(b);
  if (!(bnorm > 0.0)) {
    rep.converged = true;
    rep.history.back() = 0.0;
    return x;
  }
  const double target = opt.abs_tol > 0.0 ? opt.abs_tol : opt.rel_tol * bnorm;
  const int m_total = static_cast<int>(std::min<Index>(opt.max_iter, nn));
  const int cyc = opt.restart > 0 ? std::min(opt.restart, m_total) : m_total;
  int done = 0;
  Vec r = b;
  double g_last = bnorm;
  for (;;) {
    const int m = std::min(cyc, m_total - done);
    CycleOut c = householder_cycle(op, r, m, target, bnorm, rep);
    for (Index i = 0; i < nn; ++i) x[i] += c.x[i];
    done += c.iters;
    g_last = c.g_last;
    if (c.converged || c.breakdown || done >= m_total || c.iters == 0) break;
    // restart: explicit residual of the accumulated iterate
    const Vec ax = op(x);
    ++rep.operator_applies;
    for (Index i = 0; i < nn; ++i) r[i] = b[i] - ax[i];
  }
  rep.iterations = done;
  rep.final_rel_residual = g_last / bnorm;
  if (opt.final_residual_check) {
    const Vec ax = op(x);
    ++rep.operator_applies;
    Vec rr(b.size());
    for (Index i = 0; i < nn; ++i) rr[i] = b[i] - ax[i];
    const double true_rel = norm2(rr) / bnorm;
    if (true_rel * bnorm > 10.0 * std::max(target, rep.final_rel_residual * bnorm)) rep.mismatch = true;
    rep.final_rel_residual = true_rel;
  }
  rep.converged = rep.final_rel_residual * bnorm <= target * (1.0 + 1e-12);
  rep.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return x;
}

namespace {
Vec add(const Vec& a, const Vec& b) {
  Vec y = a;
  for (std::size_t i = 0; i < y.size(); ++i) y[i] += b[i];
  return y;
}
}  // namespace

// proj/src/deflation.cpp:102-122
SchurSolveResult deflated_solve(const SchurSystem& sys, const CoarseSpace& cs, const Vec& b_S, double tol,
                                int max_iter, int restart) {
  const Decomposition& dec = sys.op->dec;
  LinOp op = [&](const Vec& v) { return apply_P(cs, sys, apply_S(sys, apply_block_jacobi_inv(sys, v))); };
  GmresOptions opt;
  opt.abs_tol = tol * norm2(b_S);
  opt.max_iter = max_iter;
  opt.restart = restart;
  const Vec pb = apply_P(cs, sys, b_S);
  const auto before = sys.applies->load();
  SchurSolveResult out;
  const Vec x = gmres(op, pb, opt, out.report);
  out.krylov_s_applies = sys.applies->load() - before;
  const Vec x1 = apply_Q(cs, sys, apply_block_jacobi_inv(sys, x));
  const Vec x2 = apply_Z(dec, coarse_solve(cs, apply_Zt(dec, b_S)));
  out.x_S = add(x1, x2);
  return out;
}

// proj/src/deflation.cpp:124-143
SchurSolveResult two_level_schwarz_solve(const SchurSystem& sys, const CoarseSpace& cs, const Vec& b_S, double tol,
                                         int max_iter, int restart) {
  const Decomposition& dec = sys.op->dec;
  auto minv = [&](const Vec& v) { return add(apply_block_jacobi_inv(sys, v), apply_Z(dec, coarse_solve(cs, apply_Zt(dec, v)))); };
  LinOp op = [&](const Vec& v) { return apply_S(sys, minv(v)); };
  GmresOptions opt;
  opt.abs_tol = tol * norm2(b_S);
  opt.max_iter = max_iter;
  opt.restart = restart;
  const auto before = sys.applies->load();
  SchurSolveResult out;
  const Vec x = gmres(op, b_S, opt, out.report);
  out.krylov_s_applies = sys.applies->load() - before;
  out.x_S = minv(x);
  return out;
}

// proj/src/solver.cpp:56-64 ('schur')
SchurSolveResult plain_solve(const SchurSystem& sys, const Vec& b_S, double tol, int max_iter, int restart) {
  GmresOptions opt;
  opt.rel_tol = tol;
  opt.max_iter = max_iter;
  opt.restart = restart;
  const auto before = sys.applies->load();
  SchurSolveResult out;
  out.x_S = gmres([&](const Vec& v) { return apply_S(sys, v); }, b_S, opt, out.report);
  out.krylov_s_applies = sys.applies->load() - before;
  return out;
}

// proj/src/solver.cpp:65-75 ('bj', via gmres_right_preconditioned proj/src/gmres.cpp:144-150)
SchurSolveResult bj_solve(const SchurSystem& sys, const Vec& b_S, double tol, int max_iter, int restart) {
  GmresOptions opt;
  opt.rel_tol = tol;
  opt.max_iter = max_iter;
  opt.restart = restart;
  const auto before = sys.applies->load();
  SchurSolveResult out;
  const Vec x = gmres([&](const Vec& v) { return apply_S(sys, apply_block_jacobi_inv(sys, v)); }, b_S, opt, out.report);
  out.krylov_s_applies = sys.applies->load() - before;
  out.x_S = apply_block_jacobi_inv(sys, x);
  return out;
}

}  // namespace orc
