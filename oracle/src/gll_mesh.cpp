// ORACLE — TEST INFRASTRUCTURE ONLY. Restates /root/reference/proj/src/gll.cpp
// and /root/reference/proj/src/mesh.cpp.
#include <cmath>

#include "smpm.hpp"

namespace orc {

namespace {

// three-term recurrence for P_N and P_N' (proj/src/gll.cpp:10-30)
void legendre_pd(int N, double x, double& p, double& dp) {
  double pm = 1.0, dm = 0.0, pc = x, dc = 1.0;
  if (N == 0) {
    p = pm;
    dp = dm;
    return;
  }
  for (int j = 2; j <= N; ++j) {
    const double pn = ((2 * j - 1) * x * pc - (j - 1) * pm) / j;
    const double dn = dm + (2 * j - 1) * pc;
    pm = pc;
    pc = pn;
    dm = dc;
    dc = dn;
  }
  p = pc;
  dp = dc;
}

// Newton on P_N' with P_N'' from the Legendre ODE (proj/src/gll.cpp:33-44)
double newton_root(int N, double x) {
  for (int it = 0; it < 100; ++it) {
    double p, dp;
    legendre_pd(N, x, p, dp);
    const double ddp = (2.0 * x * dp - N * (N + 1) * p) / (1.0 - x * x);
    const double step = dp / ddp;
    x -= step;
    if (std::abs(step) <= 1e-14) return x;
  }
  runtime("gll_basis: Newton iteration failed to converge");
}

}  // namespace

// barycentric weights + negative-sum diagonal (proj/src/gll.cpp:48-68)
Mat lagrange_diff(const Vec& x) {
  const Index n = static_cast<Index>(x.size());
  Vec lam(static_cast<std::size_t>(n), 1.0);
  for (Index j = 0; j < n; ++j)
    for (Index m = 0; m < n; ++m)
      if (m != j) lam[j] /= x[j] - x[m];
  double mx = 0.0;
  for (double v : lam) mx = std::max(mx, std::abs(v));
  for (double& v : lam) v /= mx;
  Mat D(n, n);
  for (Index i = 0; i < n; ++i) {
    double s = 0.0;
    for (Index j = 0; j < n; ++j) {
      if (j == i) continue;
      D(i, j) = (lam[j] / lam[i]) / (x[i] - x[j]);
      s += D(i, j);
    }
    D(i, i) = -s;
  }
  return D;
}

// proj/src/gll.cpp:70-97
Gll gll_basis(int n) {
  if (n < 2) invalid("gll_basis: order must be at least 2");
  const int N = n - 1;
  Gll b;
  b.n = n;
  b.nodes.assign(static_cast<std::size_t>(n), 0.0);
  b.nodes[0] = -1.0;
  b.nodes[N] = 1.0;
  for (int i = 1; i <= (N - 1) / 2; ++i) {
    const double r = newton_root(N, -std::cos(M_PI * i / N));
    b.nodes[i] = r;
    b.nodes[N - i] = -r;
  }
  if (N % 2 == 0 && N >= 2) b.nodes[N / 2] = 0.0;
  b.weights.resize(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    double p, dp;
    legendre_pd(N, b.nodes[i], p, dp);
    b.weights[i] = 2.0 / (N * (N + 1) * p * p);
  }
  b.diff = lagrange_diff(b.nodes);
  return b;
}

// proj/src/mesh.cpp:7-46
Mesh build_mesh(int n, int m_x, int m_z, double l_x, double l_z) {
  if (n < 2 || m_x < 1 || m_z < 1 || l_x <= 0.0 || l_z <= 0.0)
    invalid("build_mesh: counts must be positive and extents > 0");
  Mesh m;
  m.basis = gll_basis(n);
  m.n = n;
  m.m_x = m_x;
  m.m_z = m_z;
  m.l_x = l_x;
  m.l_z = l_z;
  m.h_x = l_x / m_x;
  m.h_z = l_z / m_z;
  m.eta = m.h_x / m.h_z;
  m.r = static_cast<Index>(n) * n * m_x * m_z;
  m.x.resize(static_cast<std::size_t>(m.r));
  m.z.resize(static_cast<std::size_t>(m.r));
  m.nbr.assign(static_cast<std::size_t>(4 * m_x * m_z), -1);
  for (int ex = 0; ex < m_x; ++ex)
    for (int ez = 0; ez < m_z; ++ez) {
      const int e = m.elem(ex, ez);
      m.nbr[4 * e + 0] = ex > 0 ? m.elem(ex - 1, ez) : -1;
      m.nbr[4 * e + 1] = ex < m_x - 1 ? m.elem(ex + 1, ez) : -1;
      m.nbr[4 * e + 2] = ez > 0 ? m.elem(ex, ez - 1) : -1;
      m.nbr[4 * e + 3] = ez < m_z - 1 ? m.elem(ex, ez + 1) : -1;
      for (int ix = 0; ix < n; ++ix) {
        const double xc = -0.5 * l_x + ex * m.h_x + 0.5 * (m.basis.nodes[ix] + 1.0) * m.h_x;
        for (int iz = 0; iz < n; ++iz) {
          const double zc = -0.5 * l_z + ez * m.h_z + 0.5 * (m.basis.nodes[iz] + 1.0) * m.h_z;
          const Index g = m.node(e, ix, iz);
          m.x[g] = xc;
          m.z[g] = zc;
        }
      }
    }
  return m;
}

// interface slot order: left side (east edge of strip i) bottom-to-top, then
// right side (west edge of strip i+1) (proj/src/mesh.cpp:48-80)
Decomposition build_decomposition(const Mesh& mesh) {
  Decomposition dec;
  dec.n = mesh.n;
  dec.m_x = mesh.m_x;
  dec.m_z = mesh.m_z;
  dec.r = mesh.r;
  dec.d = mesh.m_x - 1;
  dec.k = 2 * dec.side() * dec.d;
  dec.gamma_to_node.resize(static_cast<std::size_t>(dec.k));
  Index p = 0;
  for (int i = 0; i < dec.d; ++i) {
    for (int ez = 0; ez < mesh.m_z; ++ez)
      for (int iz = 0; iz < mesh.n; ++iz) dec.gamma_to_node[p++] = mesh.node(mesh.elem(i, ez), mesh.n - 1, iz);
    for (int ez = 0; ez < mesh.m_z; ++ez)
      for (int iz = 0; iz < mesh.n; ++iz) dec.gamma_to_node[p++] = mesh.node(mesh.elem(i + 1, ez), 0, iz);
  }
  return dec;
}

// proj/src/mesh.cpp:82-94
Vec apply_E(const Decomposition& dec, const Vec& v) {
  if (static_cast<Index>(v.size()) != dec.k) invalid("apply_E: interface vector has wrong length");
  Vec u(static_cast<std::size_t>(dec.r), 0.0);
  for (Index p = 0; p < dec.k; ++p) u[dec.gamma_to_node[p]] = v[p];
  return u;
}

Vec apply_Et(const Decomposition& dec, const Vec& u) {
  if (static_cast<Index>(u.size()) != dec.r) invalid("apply_Et: full vector has wrong length");
  Vec v(static_cast<std::size_t>(dec.k));
  for (Index p = 0; p < dec.k; ++p) v[p] = u[dec.gamma_to_node[p]];
  return v;
}

}  // namespace orc
