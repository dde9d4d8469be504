// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product path.
//
// CPU restatement of the reference library `smpm` (/root/reference/proj):
// GLL basis, mesh + strip decomposition, operator split L = A + E B, the
// Schur complement S = I + B A^{-1} E, block-Jacobi, left null vectors,
// deflation coarse space, Householder GMRES and the deflated / two-level
// Schwarz drivers, plus the per-wavenumber Helmholtz systems of the Fourier
// extension. Every function cites the reference file:line it restates.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this code, and only as the checker / CPU
// baseline. The reference itself cannot be compiled here (Eigen3 and CLI11
// are absent), so parity is pinned through the reference's SPEC examples,
// its in-binary `validate` checks and an independent numpy dense solve; see
// DESIGN.md "Oracle and pinning".
#pragma once

#include <atomic>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "la.hpp"

namespace orc {

// /root/reference/proj/include/smpm/rng.hpp:11-32 — splitmix64-scrambled
// mt19937_64, doubles from the top 53 bits, per-trial streams.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : seed_(seed), eng_(mix(seed)) {}
  double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  Rng stream(std::uint64_t i) const { return Rng(seed_ + 0x9e3779b97f4a7c15ull * (i + 1)); }
  // Box-Muller on two consecutive uniforms (cosine branch only); the
  // reference RNG is uniform-only, this is the documented N(0,1) extension
  // (SURVEY.md convention 4).
  double normal() {
    const double u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
  }

 private:
  static std::uint64_t mix(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  }
  std::uint64_t seed_;
  std::mt19937_64 eng_;
};

// /root/reference/proj/include/smpm/gll.hpp:14-19, proj/src/gll.cpp:70-97
struct Gll {
  int n = 0;
  Vec nodes, weights;
  Mat diff;
};
Gll gll_basis(int n);
Mat lagrange_diff(const Vec& nodes);

// /root/reference/proj/include/smpm/mesh.hpp:19-37, proj/src/mesh.cpp:7-46
struct Mesh {
  Gll basis;
  int n = 0, m_x = 0, m_z = 0;
  double l_x = 0, l_z = 0, h_x = 0, h_z = 0, eta = 0;
  Index r = 0;
  Vec x, z;                  // node coordinates (reference frame centred on 0)
  std::vector<int> nbr;      // 4 per element: west, east, south, north (-1 = boundary)
  int elem(int ex, int ez) const { return ex * m_z + ez; }
  Index node(int e, int ix, int iz) const { return (static_cast<Index>(e) * n + ix) * n + iz; }
};
Mesh build_mesh(int n, int m_x, int m_z, double l_x, double l_z);

// /root/reference/proj/include/smpm/mesh.hpp:43-57, proj/src/mesh.cpp:48-80
struct Decomposition {
  int n = 0, m_x = 0, m_z = 0, d = 0;
  Index r = 0, k = 0;
  std::vector<Index> gamma_to_node;
  Index side() const { return static_cast<Index>(n) * m_z; }
  Index iface() const { return 2 * side(); }
};
Decomposition build_decomposition(const Mesh& mesh);
Vec apply_E(const Decomposition& dec, const Vec& v);
Vec apply_Et(const Decomposition& dec, const Vec& u);

// /root/reference/proj/include/smpm/operator.hpp:26-44, proj/src/operator.cpp
struct Operator {
  Mesh mesh;
  Decomposition dec;
  double tau = 0, tau_x = 0, tau_z = 0;
  Index q = 0;  // block_dim = n^2 m_z
  struct Kind {
    bool west_iface = false, east_iface = false;
  };
  std::vector<Kind> kinds;
  std::vector<int> kind_of;  // strip -> kind
  std::vector<Mat> a;        // dense strip matrix per kind
  std::vector<LU> lu;        // per kind (empty when m_x == 1)
  // B as row lists (k rows): (global node, value) pairs in emission order
  std::vector<std::vector<std::pair<Index, double>>> brow;
  // lazily built real Schur factors of each kind (Helmholtz path)
  std::vector<Mat> schur_u, schur_t;
};
double penalty_tau(int n, double h_x, double h_z, double c_tau);
Operator assemble_operator(const Mesh& mesh, const Decomposition& dec, double tau);
Vec apply_A(const Operator& op, const Vec& u);
Vec apply_B(const Operator& op, const Vec& u);
Vec apply_Bt(const Operator& op, const Vec& v);
Vec apply_L(const Operator& op, const Vec& u);
Vec solve_A(const Operator& op, const Vec& f);
Vec solve_At(const Operator& op, const Vec& f);
Mat dense_L(const Mesh& mesh, double tau);  // proj/src/bench.cpp:217-277 (validate oracle)

// Helmholtz shifted solves (proj/src/helmholtz.cpp:14-87)
void factor_unshifted_blocks(Operator& op);
void shifted_solve_kind(const Operator& op, int kind, double mu, Mat& rhs_to_x);
Vec shifted_solve(const Operator& op, double mu, const Vec& b);

// Per-kind coupling G = Btrace A_kind^{-1} E_own (proj/src/schur.cpp:19-69).
struct KindCoupling {
  Mat g;
  Index cols_west = 0, cols_east = 0, rows_west = 0, rows_east = 0;
};

// /root/reference/proj/include/smpm/schur.hpp:26-47
struct SchurSystem {
  std::shared_ptr<const Operator> op;
  Index k = 0, w = 0;
  int d = 0;
  double shift = 0.0;
  std::vector<KindCoupling> kc;  // per strip kind
  // reference per-interface layout (proj/src/schur.cpp:87-124); when
  // `materialized` is false the entries are read from kc on the fly
  // (bitwise-identical values, SURVEY.md §8(d) dedup layout).
  bool materialized = false;
  struct Block {
    Mat entries;  // rows x 2w, structural zeros included (as the reference stores them)
    std::vector<std::pair<Index, Index>> segs;
  };
  std::vector<Block> blocks;
  double frob = 0.0;
  // block-Jacobi (proj/src/schur.cpp:188-216); `jb_lu_id` maps block -> factor
  struct JBlock {
    Index begin = 0, size = 0;
    int factor = 0;
  };
  std::vector<JBlock> jacobi;
  std::vector<LU> jfactors;
  std::shared_ptr<std::atomic<std::uint64_t>> applies = std::make_shared<std::atomic<std::uint64_t>>(0);
};

// Builds per-kind couplings (mu == 0: the strip LU; mu > 0: real-Schur
// shifted solves) and the system; `layout_reference` materializes the
// reference's per-interface blocks.
SchurSystem assemble_schur(std::shared_ptr<Operator> op, double mu, bool layout_reference);
// Same from caller-supplied per-kind couplings in the export layout
// (G_W = west-boundary kind, w x w; G_I = interior kind, 2w x 2w;
// G_E = east-boundary kind, w x w), column-major.
SchurSystem schur_from_kinds(std::shared_ptr<Operator> op, double mu, const double* G_W, const double* G_I,
                             const double* G_E, bool layout_reference);
void export_kinds(const SchurSystem& sys, double* G_W, double* G_I, double* G_E);

Vec apply_S(const SchurSystem& sys, const Vec& v);
Vec apply_St(const SchurSystem& sys, const Vec& v);
Vec apply_S_definition(const SchurSystem& sys, const Vec& v);
Vec schur_rhs(const SchurSystem& sys, const Vec& f);
void build_block_jacobi(SchurSystem& sys, int dedup);
Vec apply_block_jacobi_inv(const SchurSystem& sys, const Vec& v);
Vec recover_solution(const SchurSystem& sys, const Vec& f, const Vec& x_S);
Mat dense_schur(const SchurSystem& sys);
Mat block_entries(const SchurSystem& sys, int i);

// /root/reference/proj/include/smpm/nullspace.hpp:23-36
struct NullSpace {
  Vec u_S, u_L;
  double sigma = 0.0;
  int iterations = 0;
};
Vec left_null_vector_s(const SchurSystem& sys, double sigma, double tol, int max_iter, int* its, double* sigma_out,
                       Index dense_limit);
Vec left_null_vector_l(const Operator& op, const Vec& u_S);
NullSpace compute_nullspace(const SchurSystem& sys);
Vec project_out(const Vec& v, const Vec& dir);

// /root/reference/proj/include/smpm/deflation.hpp:17-28
struct CoarseSpace {
  int d = 0;
  Mat C;
  bool singular = false, tridiagonal = false;
  Vec u_C, u_S;
  LU lu;
  Vec sub, diag, sup;
};
Vec apply_Z(const Decomposition& dec, const Vec& y);
Vec apply_Zt(const Decomposition& dec, const Vec& v);
CoarseSpace build_coarse(const SchurSystem& sys, const Vec* u_S);
Vec coarse_solve(const CoarseSpace& cs, const Vec& b);
Vec apply_P(const CoarseSpace& cs, const SchurSystem& sys, const Vec& v);
Vec apply_Q(const CoarseSpace& cs, const SchurSystem& sys, const Vec& v);

// /root/reference/proj/include/smpm/gmres.hpp:10-33
struct KrylovReport {
  int iterations = 0;
  Vec history;
  bool converged = false;
  double final_rel_residual = 0.0;
  bool mismatch = false;
  long operator_applies = 0;
  double wall_time_s = 0.0;
};
struct GmresOptions {
  double rel_tol = 1e-10;
  double abs_tol = 0.0;
  int max_iter = 2000;
  bool final_residual_check = true;
  // restart length; 0 = never restart (the reference's behaviour). The
  // restart extension is this repo's, documented in DESIGN.md.
  int restart = 0;
};
using LinOp = std::function<Vec(const Vec&)>;
Vec gmres(const LinOp& op, const Vec& b, const GmresOptions& opt, KrylovReport& rep);

struct SchurSolveResult {
  Vec x_S;
  KrylovReport report;
  std::uint64_t krylov_s_applies = 0;
};
SchurSolveResult deflated_solve(const SchurSystem& sys, const CoarseSpace& cs, const Vec& b_S, double tol,
                                int max_iter, int restart);
SchurSolveResult two_level_schwarz_solve(const SchurSystem& sys, const CoarseSpace& cs, const Vec& b_S, double tol,
                                         int max_iter, int restart);
// 'schur' and 'bj' methods of solve_poisson (proj/src/solver.cpp:56-75)
SchurSolveResult plain_solve(const SchurSystem& sys, const Vec& b_S, double tol, int max_iter, int restart);
SchurSolveResult bj_solve(const SchurSystem& sys, const Vec& b_S, double tol, int max_iter, int restart);

}  // namespace orc
