// ORACLE — TEST INFRASTRUCTURE ONLY. Restates /root/reference/proj/src/nullspace.cpp
// and /root/reference/proj/src/deflation.cpp (coarse space, projections).
#include <algorithm>
#include <cmath>

#include "smpm.hpp"

namespace orc {

namespace {

// largest-magnitude entry made positive (proj/src/nullspace.cpp:13-17);
// first index on ties, as Eigen's maxCoeff
void fix_sign(Vec& v) {
  std::size_t imax = 0;
  double best = -1.0;
  for (std::size_t i = 0; i < v.size(); ++i)
    if (std::abs(v[i]) > best) {
      best = std::abs(v[i]);
      imax = i;
    }
  if (v[imax] < 0.0)
    for (double& x : v) x = -x;
}

void normalize(Vec& v) {
  const double nv = norm2(v);
  for (double& x : v) x /= nv;
}

}  // namespace

// Shifted inverse iteration on S^T - sigma I (proj/src/nullspace.cpp:21-76).
// Beyond dense_limit the reference factors with Eigen::SparseLU; this
// restatement factors the same matrix with banded partial-pivot LU (dgbtrf):
// S is block tridiagonal over interfaces, so its half-bandwidth is < 4w.
Vec left_null_vector_s(const SchurSystem& sys, double sigma, double tol, int max_iter, int* its, double* sigma_out,
                       Index dense_limit) {
  const Index k = sys.k;
  if (sigma == 0.0) sigma = 1e-8 * sys.frob / std::sqrt(static_cast<double>(k));
  if (sigma_out) *sigma_out = sigma;
  Rng rng(0x5eed0001u);
  Vec v(static_cast<std::size_t>(k));
  for (Index i = 0; i < k; ++i) v[i] = rng.uniform() - 0.5;
  normalize(v);

  LU dense;
  BandLU band;
  const bool use_dense = k <= dense_limit;
  if (use_dense) {
    Mat st = transpose(dense_schur(sys));
    for (Index i = 0; i < k; ++i) st(i, i) -= sigma;
    dense.compute(st);
  } else {
    const Index w2 = 2 * sys.w;
    Index kl = 0, ku = 0;
    for (int i = 0; i < sys.d; ++i)
      for (const auto& [start, len] : sys.blocks[i].segs) {
        // S(start+r, i*w2+c) -> S^T(i*w2+c, start+r)
        kl = std::max(kl, (i * w2 + w2 - 1) - start);
        ku = std::max(ku, (start + len - 1) - i * w2);
      }
    band.init(k, kl, ku);
    for (Index i = 0; i < k; ++i) band.add(i, i, 1.0 - sigma);
    for (int i = 0; i < sys.d; ++i) {
      const auto& blk = sys.blocks[i];
      const Mat ent = block_entries(sys, i);
      Index off = 0;
      for (const auto& [start, len] : blk.segs) {
        for (Index c = 0; c < w2; ++c)
          for (Index r = 0; r < len; ++r) {
            const double val = ent(off + r, c);
            if (val != 0.0) band.add(i * w2 + c, start + r, val);
          }
        off += len;
      }
    }
    band.factor();
  }

  double resid = 0.0;
  for (int it = 1; it <= max_iter; ++it) {
    if (use_dense)
      dense.solve_inplace(v.data());
    else
      band.solve_inplace(v.data());
    normalize(v);
    resid = norm2(apply_St(sys, v));
    if (resid <= tol * sys.frob) {
      if (its) *its = it;
      fix_sign(v);
      return v;
    }
  }
  runtime("left_null_vector_s: no convergence, residual " + std::to_string(resid / sys.frob) + " of ||S||_F");
}

// proj/src/nullspace.cpp:78-83
Vec left_null_vector_l(const Operator& op, const Vec& u_S) {
  Vec u = solve_At(op, apply_Bt(op, u_S));
  normalize(u);
  fix_sign(u);
  return u;
}

// proj/src/nullspace.cpp:85-90
NullSpace compute_nullspace(const SchurSystem& sys) {
  NullSpace ns;
  ns.u_S = left_null_vector_s(sys, 0.0, 1e-10, 25, &ns.iterations, &ns.sigma, 3200);
  ns.u_L = left_null_vector_l(*sys.op, ns.u_S);
  return ns;
}

// proj/src/nullspace.cpp:92
Vec project_out(const Vec& v, const Vec& dir) {
  if (v.size() != dir.size()) invalid("project_out: wrong length");
  const double c = dot(dir, v);
  Vec y = v;
  for (std::size_t i = 0; i < y.size(); ++i) y[i] -= dir[i] * c;
  return y;
}

// proj/src/deflation.cpp:8-22
Vec apply_Z(const Decomposition& dec, const Vec& y) {
  if (static_cast<Index>(y.size()) != dec.d) invalid("apply_Z: wrong length");
  Vec v(static_cast<std::size_t>(dec.k));
  const Index w2 = dec.iface();
  for (int i = 0; i < dec.d; ++i) std::fill(v.begin() + i * w2, v.begin() + (i + 1) * w2, y[i]);
  return v;
}

Vec apply_Zt(const Decomposition& dec, const Vec& v) {
  if (static_cast<Index>(v.size()) != dec.k) invalid("apply_Zt: wrong length");
  Vec y(static_cast<std::size_t>(dec.d));
  const Index w2 = dec.iface();
  for (int i = 0; i < dec.d; ++i) {
    double s = 0.0;
    for (Index t = 0; t < w2; ++t) s += v[i * w2 + t];
    y[i] = s;
  }
  return y;
}

// proj/src/deflation.cpp:24-69
CoarseSpace build_coarse(const SchurSystem& sys, const Vec* u_S) {
  const Decomposition& dec = sys.op->dec;
  CoarseSpace cs;
  cs.d = dec.d;
  cs.singular = u_S != nullptr;
  cs.C = Mat(cs.d, cs.d);
  for (int j = 0; j < cs.d; ++j) {
    Vec e(static_cast<std::size_t>(cs.d), 0.0);
    e[j] = 1.0;
    const Vec c = apply_Zt(dec, apply_S(sys, apply_Z(dec, e)));
    std::copy(c.begin(), c.end(), cs.C.col(j));
  }
  const double off_tol = 1e-12 * std::sqrt(frob2(cs.C));
  cs.tridiagonal = true;
  for (int i = 0; i < cs.d && cs.tridiagonal; ++i)
    for (int j = 0; j < cs.d; ++j)
      if (std::abs(i - j) > 1 && std::abs(cs.C(i, j)) > off_tol) {
        cs.tridiagonal = false;
        break;
      }
  if (cs.singular) {
    cs.u_S = *u_S;
    cs.u_C = apply_Zt(dec, *u_S);
    normalize(cs.u_C);
    fix_sign(cs.u_C);
    Mat shifted = cs.C;
    for (int j = 0; j < cs.d; ++j)
      for (int i = 0; i < cs.d; ++i) shifted(i, j) += cs.u_C[i] * cs.u_C[j];
    cs.lu.compute(shifted);
    if (cs.lu.rcond() < 1e-14) singular("build_coarse: rank-one-shifted coarse matrix is singular");
  } else if (cs.tridiagonal) {
    cs.diag.resize(static_cast<std::size_t>(cs.d));
    for (int i = 0; i < cs.d; ++i) cs.diag[i] = cs.C(i, i);
    cs.sub.resize(static_cast<std::size_t>(std::max(cs.d - 1, 0)));
    cs.sup.resize(cs.sub.size());
    for (int i = 0; i + 1 < cs.d; ++i) {
      cs.sub[i] = cs.C(i + 1, i);
      cs.sup[i] = cs.C(i, i + 1);
    }
  } else {
    cs.lu.compute(cs.C);
    if (cs.lu.rcond() < 1e-14) singular("build_coarse: coarse matrix is singular");
  }
  return cs;
}

// proj/src/deflation.cpp:71-92
Vec coarse_solve(const CoarseSpace& cs, const Vec& b) {
  if (static_cast<Index>(b.size()) != cs.d) invalid("coarse_solve: wrong length");
  if (cs.singular) {
    Vec rhs = b;
    const double c = dot(cs.u_C, b);
    for (int i = 0; i < cs.d; ++i) rhs[i] -= cs.u_C[i] * c;
    cs.lu.solve_inplace(rhs.data());
    return rhs;
  }
  if (cs.tridiagonal) {
    const int d = cs.d;
    Vec c(static_cast<std::size_t>(d)), y(static_cast<std::size_t>(d));
    double piv = cs.diag[0];
    y[0] = b[0] / piv;
    for (int i = 1; i < d; ++i) {
      c[i - 1] = cs.sup[i - 1] / piv;
      piv = cs.diag[i] - cs.sub[i - 1] * c[i - 1];
      y[i] = (b[i] - cs.sub[i - 1] * y[i - 1]) / piv;
    }
    for (int i = d - 2; i >= 0; --i) y[i] -= c[i] * y[i + 1];
    return y;
  }
  Vec x = b;
  cs.lu.solve_inplace(x.data());
  return x;
}

// proj/src/deflation.cpp:94-100
Vec apply_P(const CoarseSpace& cs, const SchurSystem& sys, const Vec& v) {
  const Decomposition& dec = sys.op->dec;
  const Vec t = apply_S(sys, apply_Z(dec, coarse_solve(cs, apply_Zt(dec, v))));
  Vec y = v;
  for (std::size_t i = 0; i < y.size(); ++i) y[i] -= t[i];
  return y;
}

Vec apply_Q(const CoarseSpace& cs, const SchurSystem& sys, const Vec& v) {
  const Decomposition& dec = sys.op->dec;
  const Vec t = apply_Z(dec, coarse_solve(cs, apply_Zt(dec, apply_S(sys, v))));
  Vec y = v;
  for (std::size_t i = 0; i < y.size(); ++i) y[i] -= t[i];
  return y;
}

}  // namespace orc
