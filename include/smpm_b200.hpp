// smpm_b200.hpp — C++ shim over the C ABI (smpm_b200.h) that restores the
// reference library's value-semantics API for its hot path, so the reference
// call sites (solve_poisson, proj/src/solver.cpp:76-89; solve_3d,
// proj/src/helmholtz.cpp:247-269) keep their shape:
//
//   reference (proj/include/smpm/...)                  here
//   Vector apply_S(const SchurSystem&, const Vector&)   smpm_b200::apply_S(sys, v)
//   Vector apply_block_jacobi_inv(sys, v)               smpm_b200::apply_block_jacobi_inv(sys, v)
//   apply_Z / apply_Zt / coarse_solve / apply_P / apply_Q
//   Vector project_out(v, dir)                          smpm_b200::project_out(sys, v, dir)
//   SchurSolveResult deflated_solve(sys, cs, b_S, tol, max_iter)
//   SchurSolveResult two_level_schwarz_solve(...)
//
// Vectors are host std::vector<double> (the reference passes Eigen vectors
// by const&; wrap them with Eigen::Map on the caller side). Every call stages
// through device buffers owned by the System; errors throw std::invalid_argument
// (SMPM_EINVAL) or std::runtime_error (everything else), as the reference does.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "smpm_b200.h"

namespace smpm_b200 {

using Vector = std::vector<double>;

inline void check(int rc) {
  if (rc == SMPM_OK) return;
  const std::string msg = std::string("smpm_b200: ") + smpm_last_error();
  if (rc == SMPM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// proj/include/smpm/gmres.hpp:20-28
struct KrylovReport {
  int iterations = 0;
  std::vector<double> rel_residual_history;
  bool converged = false;
  double final_rel_residual = 0.0;
  bool residual_mismatch_warning = false;
  long operator_applies = 0;
  double wall_time_s = 0.0;
};

// proj/include/smpm/deflation.hpp:44-48
struct SchurSolveResult {
  Vector x_S;
  KrylovReport report;
  std::uint64_t krylov_s_applies = 0;
};

class Device {
 public:
  explicit Device(int device = 0) { check(smpm_ctx_create(device, &ctx_)); }
  ~Device() { smpm_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  smpm_ctx* get() const { return ctx_; }

 private:
  smpm_ctx* ctx_ = nullptr;
};

// One Schur system (the reference's SchurSystem + CoarseSpace) resident on
// the device. Built from the per-kind couplings (or, with from_blocks, from
// the reference's per-interface block layout) and, for the singular j = 0
// system, the left null vector u_S.
class System {
 public:
  System(Device& dev, int n, int m_x, int m_z) {
    check(smpm_batch_create(dev.get(), n, m_x, m_z, 1, &b_));
    long long k;
    int d, w;
    check(smpm_batch_dims(b_, &k, &d, &w));
    k_ = k;
    d_ = d;
    const size_t bytes = sizeof(double) * static_cast<size_t>(k_ > d_ ? k_ : d_);
    for (auto& p : buf_)
      if (cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("smpm_b200: cudaMalloc failed");
  }
  ~System() {
    for (auto p : buf_) cudaFree(p);
    smpm_batch_destroy(b_);
  }
  System(const System&) = delete;
  System& operator=(const System&) = delete;

  void set_couplings(const double* G_W, const double* G_I, const double* G_E) {
    check(smpm_batch_set_couplings(b_, 0, G_W, G_I, G_E));
  }
  void set_nullspace(const Vector& u_S) {
    if (static_cast<long long>(u_S.size()) != k_) throw std::invalid_argument("u_S has wrong length");
    check(smpm_batch_set_nullspace(b_, 0, u_S.data()));
  }
  // optional spectral factors (before finalize) and strip factors (after): the
  // fast-diagonalisation operator form and the device strip solves
  void set_spectral(int npairs, const double* T, const double* T_inv, const double* gamma) {
    check(smpm_batch_set_spectral(b_, npairs, T, T_inv, gamma));
  }
  void set_strip_factors(const smpm_strip_factors& f) { check(smpm_batch_set_strip_factors(b_, &f)); }
  // device-side setup instead of set_couplings + set_spectral + set_strip_factors: the library
  // builds couplings, block-Jacobi inverses and coarse data from the fast-diagonalisation factors
  // (replaces build_kind_coupling / build_block_jacobi / build_coarse, proj/src/schur.cpp:19-69,
  // 188-216, proj/src/deflation.cpp:24-69); w % 16 == 0
  void set_fdm(int npairs, const double* T, const double* T_inv, const smpm_strip_factors& f) {
    check(smpm_batch_set_fdm(b_, npairs, T, T_inv, &f));
  }
  void finalize() { check(smpm_batch_finalize(b_)); }

  long long k() const { return k_; }
  int d() const { return d_; }
  smpm_batch* batch() const { return b_; }

  // host -> device -> op -> host
  template <class F>
  Vector run(const Vector& in, long long nin, long long nout, F&& op) const {
    if (static_cast<long long>(in.size()) != nin) throw std::invalid_argument("wrong length");
    up(buf_[0], in);
    check(op(buf_[0], buf_[1]));
    return down(buf_[1], nout);
  }
  void up(double* dst, const Vector& v) const {
    if (cudaMemcpy(dst, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("smpm_b200: H2D copy failed");
  }
  Vector down(const double* src, long long n) const {
    Vector out(static_cast<size_t>(n));
    if (cudaMemcpy(out.data(), src, sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("smpm_b200: D2H copy failed");
    return out;
  }
  double* scratch(int i) const { return buf_[i]; }

 private:
  smpm_batch* b_ = nullptr;
  long long k_ = 0;
  int d_ = 0;
  double* buf_[3] = {nullptr, nullptr, nullptr};
};

inline Vector apply_S(const System& s, const Vector& v) {
  return s.run(v, s.k(), s.k(), [&](double* i, double* o) { return smpm_apply_S(s.batch(), i, o, nullptr); });
}
inline Vector apply_St(const System& s, const Vector& v) {
  return s.run(v, s.k(), s.k(), [&](double* i, double* o) { return smpm_apply_St(s.batch(), i, o, nullptr); });
}
inline Vector apply_block_jacobi_inv(const System& s, const Vector& v) {
  return s.run(v, s.k(), s.k(),
               [&](double* i, double* o) { return smpm_apply_block_jacobi_inv(s.batch(), i, o, nullptr); });
}
inline Vector apply_Z(const System& s, const Vector& y) {
  return s.run(y, s.d(), s.k(), [&](double* i, double* o) { return smpm_apply_Z(s.batch(), i, o, nullptr); });
}
inline Vector apply_Zt(const System& s, const Vector& v) {
  return s.run(v, s.k(), s.d(), [&](double* i, double* o) { return smpm_apply_Zt(s.batch(), i, o, nullptr); });
}
inline Vector coarse_solve(const System& s, const Vector& b) {
  return s.run(b, s.d(), s.d(), [&](double* i, double* o) { return smpm_coarse_solve(s.batch(), i, o, nullptr); });
}
inline Vector apply_P(const System& s, const Vector& v) {
  return s.run(v, s.k(), s.k(), [&](double* i, double* o) { return smpm_apply_P(s.batch(), i, o, 0, nullptr); });
}
inline Vector apply_Q(const System& s, const Vector& v) {
  return s.run(v, s.k(), s.k(), [&](double* i, double* o) { return smpm_apply_Q(s.batch(), i, o, nullptr); });
}
inline Vector project_out(const System& s, const Vector& v, const Vector& dir) {
  if (dir.size() != v.size()) throw std::invalid_argument("project_out: wrong length");
  s.up(s.scratch(2), dir);
  return s.run(v, s.k(), s.k(), [&](double* i, double* o) {
    return smpm_project_out(s.batch(), s.k(), i, s.scratch(2), o, nullptr);
  });
}

// proj/src/schur.cpp:182-186 (mu = 0) / proj/src/helmholtz.cpp:172-176 (mode shift mu):
// b_S = B (A - mu)^{-1} f; needs set_strip_factors. f has r = m_x m_z n^2 entries.
inline Vector schur_rhs(const System& s, const Vector& f) {
  double* df = nullptr;
  if (cudaMalloc(&df, sizeof(double) * f.size()) != cudaSuccess) throw std::runtime_error("smpm_b200: cudaMalloc failed");
  s.up(df, f);
  const int rc = smpm_schur_rhs(s.batch(), df, s.scratch(1), nullptr);
  cudaFree(df);
  check(rc);
  return s.down(s.scratch(1), s.k());
}
// proj/src/schur.cpp:227-230 / proj/src/helmholtz.cpp:282-292: u = (A - mu)^{-1} (f - E x_S)
inline Vector recover_solution(const System& s, const Vector& f, const Vector& x_S) {
  if (static_cast<long long>(x_S.size()) != s.k()) throw std::invalid_argument("x_S has wrong length");
  double *df = nullptr, *du = nullptr;
  if (cudaMalloc(&df, sizeof(double) * f.size()) != cudaSuccess ||
      cudaMalloc(&du, sizeof(double) * f.size()) != cudaSuccess) {
    cudaFree(df);
    throw std::runtime_error("smpm_b200: cudaMalloc failed");
  }
  s.up(df, f);
  s.up(s.scratch(0), x_S);
  const int rc = smpm_recover_solution(s.batch(), df, s.scratch(0), du, nullptr);
  Vector u;
  if (rc == SMPM_OK) u = s.down(du, static_cast<long long>(f.size()));
  cudaFree(df);
  cudaFree(du);
  check(rc);
  return u;
}

namespace detail {
inline SchurSolveResult solve(const System& s, int method, const Vector& b_S, double tol, int max_iter, int restart) {
  smpm_solve_options opt{tol, max_iter, restart, SMPM_ORTH_CGS2, 1, 1};
  smpm_report rep{};
  const int cap = (max_iter < s.k() ? max_iter : static_cast<int>(s.k())) + 2;
  std::vector<double> hist(static_cast<size_t>(cap), 0.0);
  SchurSolveResult out;
  out.x_S.resize(b_S.size());
  if (static_cast<long long>(b_S.size()) != s.k()) throw std::invalid_argument("b_S has wrong length");
  s.up(s.scratch(0), b_S);
  check(smpm_solve(s.batch(), method, s.scratch(0), s.scratch(1), &opt, &rep, hist.data(), nullptr));
  out.x_S = s.down(s.scratch(1), s.k());
  out.report.iterations = rep.iterations;
  out.report.rel_residual_history.assign(hist.begin(), hist.begin() + rep.history_len);
  out.report.converged = rep.converged != 0;
  out.report.final_rel_residual = rep.final_rel_residual;
  out.report.residual_mismatch_warning = rep.mismatch_warning != 0;
  out.report.operator_applies = rep.operator_applies;
  out.report.wall_time_s = rep.wall_time_s;
  out.krylov_s_applies = static_cast<std::uint64_t>(rep.krylov_s_applies);
  return out;
}
}  // namespace detail

// proj/include/smpm/deflation.hpp:55-61 (restart = 0 reproduces the reference's
// non-restarted GMRES; pass the GMRES(m) cycle length to restart)
inline SchurSolveResult deflated_solve(const System& s, const Vector& b_S, double tol, int max_iter, int restart = 0) {
  return detail::solve(s, SMPM_DBJ, b_S, tol, max_iter, restart);
}
inline SchurSolveResult two_level_schwarz_solve(const System& s, const Vector& b_S, double tol, int max_iter,
                                                int restart = 0) {
  return detail::solve(s, SMPM_2LAS, b_S, tol, max_iter, restart);
}

}  // namespace smpm_b200
