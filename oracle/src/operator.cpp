// ORACLE — TEST INFRASTRUCTURE ONLY. Restates /root/reference/proj/src/operator.cpp
// (strip operator split L = A + E B), the validate-only monolithic assembly
// (proj/src/bench.cpp:217-277) and the real-Schur shifted solves of
// proj/src/helmholtz.cpp:14-87.
#include <algorithm>
#include <cmath>
#include <map>
#include <thread>

#include "smpm.hpp"

namespace orc {

namespace {

// Every entry of one strip kind's block, emit(row, col, value); duplicates
// accumulate (proj/src/operator.cpp:13-74).
template <class F>
void strip_entries(const Mesh& mesh, double tx, double tz, Operator::Kind kind, F&& emit) {
  const int n = mesh.n, mz = mesh.m_z;
  const Mat& D = mesh.basis.diff;
  const Mat D2 = matmul(D, D);
  const double cx = 2.0 / mesh.h_x, cz = 2.0 / mesh.h_z;
  auto at = [n](int ez, int ix, int iz) { return (static_cast<Index>(ez) * n + ix) * n + iz; };
  for (int ez = 0; ez < mz; ++ez) {
    for (int ix = 0; ix < n; ++ix)
      for (int iz = 0; iz < n; ++iz) {
        const Index row = at(ez, ix, iz);
        for (int m = 0; m < n; ++m) {
          emit(row, at(ez, m, iz), cx * cx * D2(ix, m));
          emit(row, at(ez, ix, m), cz * cz * D2(iz, m));
        }
      }
    for (int iz = 0; iz < n; ++iz) {  // west rows, outward normal -x
      const Index row = at(ez, 0, iz);
      if (kind.west_iface) emit(row, row, tx);
      for (int m = 0; m < n; ++m) emit(row, at(ez, m, iz), -tx * cx * D(0, m));
    }
    for (int iz = 0; iz < n; ++iz) {  // east rows, outward normal +x
      const Index row = at(ez, n - 1, iz);
      if (kind.east_iface) emit(row, row, tx);
      for (int m = 0; m < n; ++m) emit(row, at(ez, m, iz), tx * cx * D(n - 1, m));
    }
    for (int ix = 0; ix < n; ++ix) {  // south rows
      const Index row = at(ez, ix, 0);
      if (ez == 0) {
        for (int m = 0; m < n; ++m) emit(row, at(ez, ix, m), -tz * cz * D(0, m));
      } else {
        emit(row, row, tz);
        for (int m = 0; m < n; ++m) emit(row, at(ez, ix, m), -tz * cz * D(0, m));
        emit(row, at(ez - 1, ix, n - 1), -tz);
        for (int m = 0; m < n; ++m) emit(row, at(ez - 1, ix, m), tz * cz * D(n - 1, m));
      }
    }
    for (int ix = 0; ix < n; ++ix) {  // north rows
      const Index row = at(ez, ix, n - 1);
      if (ez == mz - 1) {
        for (int m = 0; m < n; ++m) emit(row, at(ez, ix, m), tz * cz * D(n - 1, m));
      } else {
        emit(row, row, tz);
        for (int m = 0; m < n; ++m) emit(row, at(ez, ix, m), tz * cz * D(n - 1, m));
        emit(row, at(ez + 1, ix, 0), -tz);
        for (int m = 0; m < n; ++m) emit(row, at(ez + 1, ix, m), -tz * cz * D(0, m));
      }
    }
  }
}

template <class F>
void parallel_for(Index n, F&& body) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const Index nt = std::min<Index>(static_cast<Index>(hw), n);
  if (nt <= 1) {
    for (Index i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> th;
  for (Index t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (Index i = t; i < n; i += nt) body(i);
    });
  for (auto& x : th) x.join();
}

}  // namespace

// proj/src/operator.cpp:78-82
double penalty_tau(int n, double h_x, double h_z, double c_tau) {
  if (n < 2 || h_x <= 0.0 || h_z <= 0.0 || c_tau <= 0.0) invalid("penalty_tau: inputs must be positive");
  return c_tau * n * n / std::min(h_x, h_z);
}

// proj/src/operator.cpp:84-153
Operator assemble_operator(const Mesh& mesh, const Decomposition& dec, double tau) {
  Operator op;
  op.mesh = mesh;
  op.dec = dec;
  op.tau = op.tau_x = op.tau_z = tau;
  op.q = static_cast<Index>(mesh.n) * mesh.n * mesh.m_z;
  op.kind_of.resize(static_cast<std::size_t>(mesh.m_x));
  for (int s = 0; s < mesh.m_x; ++s) {
    const Operator::Kind want{s > 0, s < mesh.m_x - 1};
    int id = -1;
    for (std::size_t i = 0; i < op.kinds.size(); ++i)
      if (op.kinds[i].west_iface == want.west_iface && op.kinds[i].east_iface == want.east_iface)
        id = static_cast<int>(i);
    if (id < 0) {
      op.kinds.push_back(want);
      id = static_cast<int>(op.kinds.size()) - 1;
    }
    op.kind_of[s] = id;
  }
  for (const auto& kind : op.kinds) {
    Mat a(op.q, op.q);
    strip_entries(mesh, op.tau_x, op.tau_z, kind, [&](Index r, Index c, double v) { a(r, c) += v; });
    op.a.push_back(std::move(a));
  }
  if (mesh.m_x >= 2) {
    for (std::size_t i = 0; i < op.kinds.size(); ++i) {
      LU lu;
      lu.compute(op.a[i]);
      if (lu.rcond() < 1e-15) singular("assemble_operator: singular strip block (kind " + std::to_string(i) + ")");
      op.lu.push_back(std::move(lu));
    }
  }
  // B rows: neighbour traces of the horizontal fluxes (proj/src/operator.cpp:127-151)
  const int n = mesh.n;
  const double cx = 2.0 / mesh.h_x;
  const Mat& D = mesh.basis.diff;
  op.brow.assign(static_cast<std::size_t>(dec.k), {});
  auto add = [&](Index p, Index node, double v) {
    auto& row = op.brow[static_cast<std::size_t>(p)];
    for (auto& e : row)
      if (e.first == node) {
        e.second += v;  // duplicate triplets accumulate
        return;
      }
    row.emplace_back(node, v);
  };
  for (int i = 0; i < dec.d; ++i)
    for (int ez = 0; ez < mesh.m_z; ++ez)
      for (int iz = 0; iz < n; ++iz) {
        Index p = 2 * dec.side() * i + static_cast<Index>(ez) * n + iz;
        int e = mesh.elem(i + 1, ez);
        add(p, mesh.node(e, 0, iz), -op.tau_x);
        for (int m = 0; m < n; ++m) add(p, mesh.node(e, m, iz), -op.tau_x * cx * D(0, m));
        p += dec.side();
        e = mesh.elem(i, ez);
        add(p, mesh.node(e, n - 1, iz), -op.tau_x);
        for (int m = 0; m < n; ++m) add(p, mesh.node(e, m, iz), op.tau_x * cx * D(n - 1, m));
      }
  for (auto& row : op.brow) std::sort(row.begin(), row.end());
  return op;
}

// proj/src/operator.cpp:160-167
Vec apply_A(const Operator& op, const Vec& u) {
  if (static_cast<Index>(u.size()) != op.dec.r) invalid("apply_A: wrong length");
  Vec y(u.size(), 0.0);
  for (int s = 0; s < op.mesh.m_x; ++s) {
    const Mat& a = op.a[op.kind_of[s]];
    gemv_acc(a.data(), op.q, op.q, op.q, u.data() + s * op.q, y.data() + s * op.q);
  }
  return y;
}

Vec apply_B(const Operator& op, const Vec& u) {
  if (static_cast<Index>(u.size()) != op.dec.r) invalid("apply_B: wrong length");
  Vec y(static_cast<std::size_t>(op.dec.k), 0.0);
  for (Index p = 0; p < op.dec.k; ++p) {
    double s = 0.0;
    for (const auto& [node, v] : op.brow[p]) s += v * u[node];
    y[p] = s;
  }
  return y;
}

Vec apply_Bt(const Operator& op, const Vec& v) {
  if (static_cast<Index>(v.size()) != op.dec.k) invalid("apply_Bt: wrong length");
  Vec y(static_cast<std::size_t>(op.dec.r), 0.0);
  for (Index p = 0; p < op.dec.k; ++p)
    for (const auto& [node, c] : op.brow[p]) y[node] += c * v[p];
  return y;
}

// proj/src/operator.cpp:179-184
Vec apply_L(const Operator& op, const Vec& u) {
  Vec y = apply_A(op, u);
  const Vec bu = apply_B(op, u);
  for (Index p = 0; p < op.dec.k; ++p) y[op.dec.gamma_to_node[p]] += bu[p];
  return y;
}

// proj/src/operator.cpp:186-204
Vec solve_A(const Operator& op, const Vec& f) {
  if (op.lu.empty()) runtime("solve_A: single-strip operator is not factored");
  if (static_cast<Index>(f.size()) != op.dec.r) invalid("solve_A: wrong length");
  Vec u = f;
  for (int s = 0; s < op.mesh.m_x; ++s) op.lu[op.kind_of[s]].solve_inplace(u.data() + s * op.q);
  return u;
}

Vec solve_At(const Operator& op, const Vec& f) {
  if (op.lu.empty()) runtime("solve_At: single-strip operator is not factored");
  if (static_cast<Index>(f.size()) != op.dec.r) invalid("solve_At: wrong length");
  Vec u = f;
  for (int s = 0; s < op.mesh.m_x; ++s) op.lu[op.kind_of[s]].solve_t_inplace(u.data() + s * op.q);
  return u;
}

// Monolithic per-element assembly, independent of the strip split
// (proj/src/bench.cpp:217-277).
Mat dense_L(const Mesh& mesh, double tau) {
  const int n = mesh.n;
  Mat L(mesh.r, mesh.r);
  const Mat& D = mesh.basis.diff;
  const Mat D2 = matmul(D, D);
  const double cx = 2.0 / mesh.h_x, cz = 2.0 / mesh.h_z;
  for (int ex = 0; ex < mesh.m_x; ++ex)
    for (int ez = 0; ez < mesh.m_z; ++ez) {
      const int e = mesh.elem(ex, ez);
      for (int ix = 0; ix < n; ++ix)
        for (int iz = 0; iz < n; ++iz) {
          const Index row = mesh.node(e, ix, iz);
          for (int m = 0; m < n; ++m) {
            L(row, mesh.node(e, m, iz)) += cx * cx * D2(ix, m);
            L(row, mesh.node(e, ix, m)) += cz * cz * D2(iz, m);
          }
          if (ix == 0) {
            const int nb = mesh.nbr[4 * e + 0];
            for (int m = 0; m < n; ++m) L(row, mesh.node(e, m, iz)) += -tau * cx * D(0, m);
            if (nb >= 0) {
              L(row, row) += tau;
              L(row, mesh.node(nb, n - 1, iz)) -= tau;
              for (int m = 0; m < n; ++m) L(row, mesh.node(nb, m, iz)) += tau * cx * D(n - 1, m);
            }
          }
          if (ix == n - 1) {
            const int nb = mesh.nbr[4 * e + 1];
            for (int m = 0; m < n; ++m) L(row, mesh.node(e, m, iz)) += tau * cx * D(n - 1, m);
            if (nb >= 0) {
              L(row, row) += tau;
              L(row, mesh.node(nb, 0, iz)) -= tau;
              for (int m = 0; m < n; ++m) L(row, mesh.node(nb, m, iz)) += -tau * cx * D(0, m);
            }
          }
          if (iz == 0) {
            const int nb = mesh.nbr[4 * e + 2];
            for (int m = 0; m < n; ++m) L(row, mesh.node(e, ix, m)) += -tau * cz * D(0, m);
            if (nb >= 0) {
              L(row, row) += tau;
              L(row, mesh.node(nb, ix, n - 1)) -= tau;
              for (int m = 0; m < n; ++m) L(row, mesh.node(nb, ix, m)) += tau * cz * D(n - 1, m);
            }
          }
          if (iz == n - 1) {
            const int nb = mesh.nbr[4 * e + 3];
            for (int m = 0; m < n; ++m) L(row, mesh.node(e, ix, m)) += tau * cz * D(n - 1, m);
            if (nb >= 0) {
              L(row, row) += tau;
              L(row, mesh.node(nb, ix, 0)) -= tau;
              for (int m = 0; m < n; ++m) L(row, mesh.node(nb, ix, m)) += -tau * cz * D(0, m);
            }
          }
        }
    }
  return L;
}

// ---- Helmholtz: real Schur factors + quasi-triangular shifted solves ------

// proj/src/helmholtz.cpp:58-70; T is stored transposed so each row of T is
// a contiguous column of schur_t.
void factor_unshifted_blocks(Operator& op) {
  if (!op.schur_u.empty()) return;
  for (std::size_t kind = 0; kind < op.kinds.size(); ++kind) {
    Mat U, T;
    real_schur(op.a[kind], U, T);
    op.schur_u.push_back(std::move(U));
    op.schur_t.push_back(transpose(T));
  }
}

namespace {

// back-substitution of (T - mu I) y = b, T quasi-upper-triangular
// (proj/src/helmholtz.cpp:14-54); tt = T^T
void quasi_tri_solve(const Mat& tt, double mu, double* b) {
  const Index q = tt.rows;
  double tmax = 0.0;
  for (double v : tt.a) tmax = std::max(tmax, std::abs(v));
  const double tiny = 1e-13 * (tmax + std::abs(mu));
  auto T = [&](Index i, Index j) { return tt(j, i); };
  Index i = q - 1;
  while (i >= 0) {
    if (i > 0 && T(i, i - 1) != 0.0) {
      double r1 = b[i - 1], r2 = b[i];
      const Index tail = q - 1 - i;
      if (tail > 0) {
        r1 -= dot(tt.col(i - 1) + i + 1, b + i + 1, tail);
        r2 -= dot(tt.col(i) + i + 1, b + i + 1, tail);
      }
      const double a11 = T(i - 1, i - 1) - mu, a12 = T(i - 1, i);
      const double a21 = T(i, i - 1), a22 = T(i, i) - mu;
      const double det = a11 * a22 - a12 * a21;
      if (std::abs(det) <= tiny * (std::abs(a11) + std::abs(a12) + std::abs(a21) + std::abs(a22)))
        runtime("shifted solve: shift coincides with a block eigenvalue");
      b[i - 1] = (a22 * r1 - a12 * r2) / det;
      b[i] = (-a21 * r1 + a11 * r2) / det;
      i -= 2;
    } else {
      const Index tail = q - 1 - i;
      double r = b[i];
      if (tail > 0) r -= dot(tt.col(i) + i + 1, b + i + 1, tail);
      const double dii = T(i, i) - mu;
      if (std::abs(dii) <= tiny) runtime("shifted solve: shift coincides with a block eigenvalue");
      b[i] = r / dii;
      --i;
    }
  }
}

}  // namespace

// (A_kind - mu I)^{-1} rhs (proj/src/helmholtz.cpp:72-87); columns solved in
// parallel threads (independent, so results are deterministic)
void shifted_solve_kind(const Operator& op, int kind, double mu, Mat& rhs) {
  const Mat& U = op.schur_u[kind];
  Mat y = matmul(transpose(U), rhs);
  const Mat& tt = op.schur_t[kind];
  parallel_for(y.cols, [&](Index c) { quasi_tri_solve(tt, mu, y.col(c)); });
  rhs = matmul(U, y);
}

// proj/src/helmholtz.cpp:89-97
Vec shifted_solve(const Operator& op, double mu, const Vec& b) {
  if (static_cast<Index>(b.size()) != op.dec.r) invalid("shifted_solve: wrong length");
  Mat cols(op.q, 1);
  Vec x(b.size());
  for (int s = 0; s < op.mesh.m_x; ++s) {
    std::copy(b.begin() + s * op.q, b.begin() + (s + 1) * op.q, cols.col(0));
    shifted_solve_kind(op, op.kind_of[s], mu, cols);
    std::copy(cols.col(0), cols.col(0) + op.q, x.begin() + s * op.q);
  }
  return x;
}

}  // namespace orc
