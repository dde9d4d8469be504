// ORACLE — TEST INFRASTRUCTURE ONLY. See la.hpp.
#include "la.hpp"

#include <algorithm>
#include <cstring>

extern "C" {
void scipy_dgetrf_(const int* m, const int* n, double* a, const int* lda, int* ipiv, int* info);
void scipy_dgetrs_(const char* trans, const int* n, const int* nrhs, const double* a, const int* lda,
                   const int* ipiv, double* b, const int* ldb, int* info, std::size_t);
void scipy_dgecon_(const char* norm, const int* n, const double* a, const int* lda, const double* anorm,
                   double* rcond, double* work, int* iwork, int* info, std::size_t);
double scipy_dlange_(const char* norm, const int* m, const int* n, const double* a, const int* lda,
                     double* work, std::size_t);
void scipy_dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
                  const double* alpha, const double* a, const int* lda, const double* b, const int* ldb,
                  const double* beta, double* c, const int* ldc, std::size_t, std::size_t);
void scipy_dgbtrf_(const int* m, const int* n, const int* kl, const int* ku, double* ab, const int* ldab,
                   int* ipiv, int* info);
void scipy_dgbtrs_(const char* trans, const int* n, const int* kl, const int* ku, const int* nrhs,
                   const double* ab, const int* ldab, const int* ipiv, double* b, const int* ldb, int* info,
                   std::size_t);
void scipy_dgees_(const char* jobvs, const char* sort, void* select, const int* n, double* a, const int* lda,
                  int* sdim, double* wr, double* wi, double* vs, const int* ldvs, double* work, const int* lwork,
                  int* bwork, int* info, std::size_t, std::size_t);
void scipy_openblas_set_num_threads(int);
}

namespace orc {

static int as_int(Index v) {
  if (v > 0x7fffffff) invalid("dimension exceeds LP64 LAPACK range");
  return static_cast<int>(v);
}

double dot(const double* x, const double* y, Index n) {
  double s = 0.0;
  for (Index i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

double norm2(const double* x, Index n) {
  // scaled accumulation is unnecessary at these magnitudes; plain sum of squares
  double s = 0.0;
  for (Index i = 0; i < n; ++i) s += x[i] * x[i];
  return std::sqrt(s);
}

bool all_finite(const Vec& x) {
  for (double v : x)
    if (!std::isfinite(v)) return false;
  return true;
}

void gemv_acc(const double* A, Index lda, Index rows, Index cols, const double* x, double* y) {
  Index j = 0;
  for (; j + 4 <= cols; j += 4) {
    const double x0 = x[j], x1 = x[j + 1], x2 = x[j + 2], x3 = x[j + 3];
    const double* a0 = A + j * lda;
    const double* a1 = a0 + lda;
    const double* a2 = a1 + lda;
    const double* a3 = a2 + lda;
    for (Index i = 0; i < rows; ++i) y[i] += a0[i] * x0 + a1[i] * x1 + a2[i] * x2 + a3[i] * x3;
  }
  for (; j < cols; ++j) {
    const double xj = x[j];
    const double* a = A + j * lda;
    for (Index i = 0; i < rows; ++i) y[i] += a[i] * xj;
  }
}

void gemv_t_acc(const double* A, Index lda, Index rows, Index cols, const double* x, double* y) {
  for (Index j = 0; j < cols; ++j) y[j] += dot(A + j * lda, x, rows);
}

Mat matmul(const Mat& A, const Mat& B) {
  if (A.cols != B.rows) invalid("matmul: shape mismatch");
  Mat C(A.rows, B.cols);
  if (A.rows == 0 || B.cols == 0 || A.cols == 0) return C;
  const int m = as_int(A.rows), n = as_int(B.cols), k = as_int(A.cols);
  const double one = 1.0, zero = 0.0;
  scipy_dgemm_("N", "N", &m, &n, &k, &one, A.data(), &m, B.data(), &k, &zero, C.data(), &m, 1, 1);
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.cols, A.rows);
  for (Index j = 0; j < A.cols; ++j)
    for (Index i = 0; i < A.rows; ++i) T(j, i) = A(i, j);
  return T;
}

double frob2(const Mat& A) {
  double s = 0.0;
  for (double v : A.a) s += v * v;
  return s;
}

void LU::compute(const Mat& A) {
  if (A.rows != A.cols) invalid("LU: matrix not square");
  n = A.rows;
  f = A;
  piv.assign(static_cast<std::size_t>(n), 0);
  if (n == 0) {
    rcond_est = 1.0;
    return;
  }
  const int nn = as_int(n);
  std::vector<double> work(static_cast<std::size_t>(4 * n));
  std::vector<int> iwork(static_cast<std::size_t>(n));
  const double anorm = scipy_dlange_("1", &nn, &nn, A.data(), &nn, work.data(), 1);
  int info = 0;
  scipy_dgetrf_(&nn, &nn, f.data(), &nn, piv.data(), &info);
  if (info < 0) runtime("LU: dgetrf argument error");
  if (info > 0) {
    rcond_est = 0.0;  // exactly singular pivot
    return;
  }
  scipy_dgecon_("1", &nn, f.data(), &nn, &anorm, &rcond_est, work.data(), iwork.data(), &info, 1);
}

void LU::solve_inplace(double* x) const {
  for (Index i = 0; i < n; ++i) {
    const Index p = piv[static_cast<std::size_t>(i)] - 1;
    if (p != i) std::swap(x[i], x[p]);
  }
  // L y = b (unit lower), column-oriented
  for (Index j = 0; j < n; ++j) {
    const double xj = x[j];
    if (xj == 0.0) continue;
    const double* c = f.col(j);
    for (Index i = j + 1; i < n; ++i) x[i] -= c[i] * xj;
  }
  // U x = y
  for (Index j = n - 1; j >= 0; --j) {
    const double* c = f.col(j);
    x[j] /= c[j];
    const double xj = x[j];
    if (xj == 0.0) continue;
    for (Index i = 0; i < j; ++i) x[i] -= c[i] * xj;
  }
}

void LU::solve_t_inplace(double* x) const {
  // A = P L U  =>  A^T = U^T L^T P^T
  for (Index i = 0; i < n; ++i) {
    const double* c = f.col(i);
    x[i] = (x[i] - dot(c, x, i)) / c[i];
  }
  for (Index i = n - 1; i >= 0; --i) {
    const double* c = f.col(i);
    x[i] -= dot(c + i + 1, x + i + 1, n - i - 1);
  }
  for (Index i = n - 1; i >= 0; --i) {
    const Index p = piv[static_cast<std::size_t>(i)] - 1;
    if (p != i) std::swap(x[i], x[p]);
  }
}

void LU::solve_cols(Mat& B) const {
  if (B.rows != n) invalid("LU::solve_cols: shape mismatch");
  if (n == 0 || B.cols == 0) return;
  const int nn = as_int(n), nr = as_int(B.cols);
  int info = 0;
  scipy_dgetrs_("N", &nn, &nr, f.data(), &nn, piv.data(), B.data(), &nn, &info, 1);
  if (info != 0) runtime("LU::solve_cols: dgetrs failed");
}

void BandLU::init(Index n_, Index kl_, Index ku_) {
  n = n_;
  kl = kl_;
  ku = ku_;
  ldab = 2 * kl + ku + 1;
  ab.assign(static_cast<std::size_t>(ldab * n), 0.0);
  piv.assign(static_cast<std::size_t>(n), 0);
}

void BandLU::add(Index i, Index j, double v) {
  if (i - j > kl || j - i > ku) invalid("BandLU: entry outside band");
  ab[static_cast<std::size_t>(kl + ku + i - j + j * ldab)] += v;
}

void BandLU::factor() {
  const int nn = as_int(n), l = as_int(kl), u = as_int(ku), ld = as_int(ldab);
  int info = 0;
  scipy_dgbtrf_(&nn, &nn, &l, &u, ab.data(), &ld, piv.data(), &info);
  if (info != 0) singular("BandLU: factorization failed (info " + std::to_string(info) + ")");
}

void BandLU::solve_inplace(double* x) const {
  const int nn = as_int(n), l = as_int(kl), u = as_int(ku), ld = as_int(ldab), one = 1;
  int info = 0;
  scipy_dgbtrs_("N", &nn, &l, &u, &one, ab.data(), &ld, piv.data(), x, &nn, &info, 1);
  if (info != 0) runtime("BandLU: dgbtrs failed");
}

void real_schur(const Mat& A, Mat& U, Mat& T) {
  if (A.rows != A.cols) invalid("real_schur: matrix not square");
  const int n = as_int(A.rows);
  T = A;
  U = Mat(A.rows, A.rows);
  std::vector<double> wr(static_cast<std::size_t>(n)), wi(static_cast<std::size_t>(n));
  int sdim = 0, info = 0, lwork = -1;
  double wq = 0.0;
  scipy_dgees_("V", "N", nullptr, &n, T.data(), &n, &sdim, wr.data(), wi.data(), U.data(), &n, &wq, &lwork,
               nullptr, &info, 1, 1);
  lwork = static_cast<int>(wq);
  std::vector<double> work(static_cast<std::size_t>(std::max(lwork, 1)));
  scipy_dgees_("V", "N", nullptr, &n, T.data(), &n, &sdim, wr.data(), wi.data(), U.data(), &n, work.data(),
               &lwork, nullptr, &info, 1, 1);
  if (info != 0) runtime("real_schur: dgees failed (info " + std::to_string(info) + ")");
}

void set_blas_threads(int n) { scipy_openblas_set_num_threads(n); }

}  // namespace orc
