// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product path.
//
// Minimal dense linear algebra for the CPU restatement of the reference
// (which uses Eigen3 fp64, /root/reference/proj/include/smpm/types.hpp:7-11).
// Column-major storage like Eigen's default MatrixXd. Dense factorizations
// call LAPACK from the OpenBLAS build bundled with scipy in this image
// (symbols prefixed scipy_, LP64); the solve-path loops (GEMV, triangular
// solves) are hand-written and single-threaded, matching the reference's
// single-threaded Eigen solve path.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Index = std::int64_t;
using Vec = std::vector<double>;

struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> a;  // column-major
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<std::size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return a[static_cast<std::size_t>(j * rows + i)]; }
  double operator()(Index i, Index j) const { return a[static_cast<std::size_t>(j * rows + i)]; }
  double* col(Index j) { return a.data() + j * rows; }
  const double* col(Index j) const { return a.data() + j * rows; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
  static Mat identity(Index n) {
    Mat m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

// ---- vector helpers -------------------------------------------------------
double dot(const double* x, const double* y, Index n);
double norm2(const double* x, Index n);
inline double dot(const Vec& x, const Vec& y) { return dot(x.data(), y.data(), static_cast<Index>(x.size())); }
inline double norm2(const Vec& x) { return norm2(x.data(), static_cast<Index>(x.size())); }
bool all_finite(const Vec& x);

// y += A x for a column-major rows x cols block (ld = lda); column-axpy
// order like Eigen's column-major GEMV kernel.
void gemv_acc(const double* A, Index lda, Index rows, Index cols, const double* x, double* y);
// y += A^T x
void gemv_t_acc(const double* A, Index lda, Index rows, Index cols, const double* x, double* y);
// C = A * B (LAPACK-backed dgemm), all column-major
Mat matmul(const Mat& A, const Mat& B);
Mat transpose(const Mat& A);
double frob2(const Mat& A);

// ---- LU with partial pivoting (Eigen::PartialPivLU restated) --------------
struct LU {
  Index n = 0;
  Mat f;                  // packed L\U
  std::vector<int> piv;   // LAPACK 1-based row interchanges
  double rcond_est = 0.0; // reciprocal 1-norm condition estimate (dgecon)
  void compute(const Mat& A);
  // x <- A^{-1} x, in place (hand-written substitutions, single-threaded)
  void solve_inplace(double* x) const;
  // x <- A^{-T} x
  void solve_t_inplace(double* x) const;
  // multi-column solve through LAPACK dgetrs (setup only)
  void solve_cols(Mat& B) const;
  double rcond() const { return rcond_est; }
};

// ---- banded LU (stands in for Eigen::SparseLU at
//      /root/reference/proj/src/nullspace.cpp:41-61) --------------------------
struct BandLU {
  Index n = 0, kl = 0, ku = 0, ldab = 0;
  std::vector<double> ab;
  std::vector<int> piv;
  // entries supplied through set(i,j,v) (accumulating) before factor()
  void init(Index n_, Index kl_, Index ku_);
  void add(Index i, Index j, double v);
  void factor();
  void solve_inplace(double* x) const;
};

// ---- real Schur form A = U T U^T (Eigen::RealSchur restated via dgees) ----
void real_schur(const Mat& A, Mat& U, Mat& T);

void set_blas_threads(int n);

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
// error codes mirror the reference's exception classes
enum : int { E_OK = 0, E_INVALID = 1, E_RUNTIME = 2, E_NONFINITE = 3, E_SINGULAR = 4 };
[[noreturn]] inline void invalid(const std::string& m) { throw Error(E_INVALID, m); }
[[noreturn]] inline void runtime(const std::string& m) { throw Error(E_RUNTIME, m); }
[[noreturn]] inline void singular(const std::string& m) { throw Error(E_SINGULAR, m); }

}  // namespace orc
