// ORACLE — TEST INFRASTRUCTURE ONLY. Restates /root/reference/proj/src/schur.cpp.
#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>

#include "smpm.hpp"

namespace orc {

namespace {

// G = Btrace * A_kind^{-1} * E_own, rows [west-readers; east-readers],
// cols [west-own; east-own] (proj/src/schur.cpp:19-69)
KindCoupling build_kind_coupling(const Operator& op, int kind_id, double mu) {
  const Mesh& mesh = op.mesh;
  const int n = mesh.n, mz = mesh.m_z;
  const Index w = static_cast<Index>(n) * mz;
  const Operator::Kind kind = op.kinds[kind_id];
  auto at = [n](int ez, int ix, int iz) { return (static_cast<Index>(ez) * n + ix) * n + iz; };
  KindCoupling kc;
  kc.cols_west = kc.rows_west = kind.west_iface ? w : 0;
  kc.cols_east = kc.rows_east = kind.east_iface ? w : 0;
  const Index ncols = kc.cols_west + kc.cols_east;
  Mat x(op.q, ncols);
  Index c = 0;
  if (kind.west_iface)
    for (int ez = 0; ez < mz; ++ez)
      for (int iz = 0; iz < n; ++iz) x(at(ez, 0, iz), c++) = 1.0;
  if (kind.east_iface)
    for (int ez = 0; ez < mz; ++ez)
      for (int iz = 0; iz < n; ++iz) x(at(ez, n - 1, iz), c++) = 1.0;
  if (mu == 0.0)
    op.lu[kind_id].solve_cols(x);  // PartialPivLU solve (proj/src/schur.cpp:135,225)
  else
    shifted_solve_kind(op, kind_id, mu, x);  // proj/src/helmholtz.cpp:131-134

  const Mat& D = mesh.basis.diff;
  const double cx = 2.0 / mesh.h_x, tau = op.tau_x;
  kc.g = Mat(kc.rows_west + kc.rows_east, ncols);
  Vec acc(static_cast<std::size_t>(ncols));
  Index row = 0;
  auto emit_row = [&](int ez, int iz, int edge, double sign, int drow) {
    for (Index j = 0; j < ncols; ++j) acc[j] = x(at(ez, edge, iz), j);
    for (int m = 0; m < n; ++m) {
      const double coef = cx * D(drow, m);
      for (Index j = 0; j < ncols; ++j) acc[j] += sign * coef * x(at(ez, m, iz), j);
    }
    for (Index j = 0; j < ncols; ++j) kc.g(row, j) = -tau * acc[j];
    ++row;
  };
  // readers across the west interface: -tau (u + du/dx) on the west edge
  if (kind.west_iface)
    for (int ez = 0; ez < mz; ++ez)
      for (int iz = 0; iz < n; ++iz) emit_row(ez, iz, 0, +1.0, 0);
  // readers across the east interface: -tau (u - du/dx) on the east edge
  if (kind.east_iface)
    for (int ez = 0; ez < mz; ++ez)
      for (int iz = 0; iz < n; ++iz) emit_row(ez, iz, n - 1, -1.0, n - 1);
  return kc;
}

// sub-block of a kind coupling: X in {W,E} readers, Y in {W,E} own columns
const double* sub(const KindCoupling& kc, bool east_rows, bool east_cols, Index w, Index& ld) {
  ld = kc.g.rows;
  const Index r0 = east_rows ? kc.rows_west : 0;
  const Index c0 = east_cols ? kc.cols_west : 0;
  return kc.g.data() + c0 * ld + r0;
}

// y += G_sub x, x/y of length w (the ld is taken from the coupling itself)
void gemv_sub(const KindCoupling& kc, bool er, bool ec, Index w, Index rows, Index cols, const double* x, double* y) {
  Index ld = 0;
  const double* p = sub(kc, er, ec, w, ld);
  gemv_acc(p, ld, rows, cols, x, y);
}
void gemv_t_sub(const KindCoupling& kc, bool er, bool ec, Index w, Index rows, Index cols, const double* x, double* y) {
  Index ld = 0;
  const double* p = sub(kc, er, ec, w, ld);
  gemv_t_acc(p, ld, rows, cols, x, y);
}

void finish_system(SchurSystem& sys, bool layout_reference) {
  const Operator& op = *sys.op;
  const Index w = sys.w;
  const int d = sys.d;
  double frob2 = static_cast<double>(sys.k);
  sys.materialized = layout_reference;
  sys.blocks.assign(static_cast<std::size_t>(d), {});
  // per-interface blocks (proj/src/schur.cpp:87-124)
  for (int i = 0; i < d; ++i) {
    auto& blk = sys.blocks[i];
    const bool has_a = i >= 1, has_d = i <= d - 2;
    const Index rows = (has_a ? w : 0) + 2 * w + (has_d ? w : 0);
    Index off = 0, sa = -1, sb, sc, sd = -1;
    if (has_a) {
      sa = off;
      blk.segs.emplace_back((i - 1) * 2 * w, w);
      off += w;
    }
    sb = off;
    blk.segs.emplace_back(i * 2 * w, w);
    off += w;
    sc = off;
    blk.segs.emplace_back(i * 2 * w + w, w);
    off += w;
    if (has_d) {
      sd = off;
      blk.segs.emplace_back((i + 1) * 2 * w + w, w);
    }
    const KindCoupling& gl = sys.kc[op.kind_of[i]];
    const KindCoupling& gr = sys.kc[op.kind_of[i + 1]];
    Mat e(rows, 2 * w);
    auto put = [&](Index r0, Index c0, const KindCoupling& kc, bool er, bool ec) {
      Index ld;
      const double* p = sub(kc, er, ec, w, ld);
      for (Index c = 0; c < w; ++c)
        for (Index r = 0; r < w; ++r) e(r0 + r, c0 + c) = p[c * ld + r];
    };
    if (has_a) put(sa, 0, gl, false, true);
    put(sc, 0, gl, true, true);
    put(sb, w, gr, false, false);
    if (has_d) put(sd, w, gr, true, false);
    frob2 += orc::frob2(e);
    if (layout_reference) blk.entries = std::move(e);
  }
  sys.frob = std::sqrt(frob2);
}

}  // namespace

// entries of interface block i (rows x 2w, structural zeros included), read
// from the materialized reference layout or rebuilt from the kind couplings
Mat block_entries(const SchurSystem& sys, int i) {
  const auto& blk = sys.blocks[i];
  if (sys.materialized) return blk.entries;
  const Operator& op = *sys.op;
  const Index w = sys.w;
  const KindCoupling& gl = sys.kc[op.kind_of[i]];
  const KindCoupling& gr = sys.kc[op.kind_of[i + 1]];
  Index rows = 0;
  for (const auto& s : blk.segs) rows += s.second;
  Mat ent(rows, 2 * w);
  Index off = 0, ld = 0;
  auto put = [&](Index r0, Index c0, const KindCoupling& kc, bool er, bool ec) {
    const double* p = sub(kc, er, ec, w, ld);
    for (Index c = 0; c < w; ++c)
      for (Index r = 0; r < w; ++r) ent(r0 + r, c0 + c) = p[c * ld + r];
  };
  if (i >= 1) {
    put(off, 0, gl, false, true);
    off += w;
  }
  put(off, w, gr, false, false);
  off += w;
  put(off, 0, gl, true, true);
  off += w;
  if (i <= sys.d - 2) put(off, w, gr, true, false);
  return ent;
}

SchurSystem assemble_schur(std::shared_ptr<Operator> op, double mu, bool layout_reference) {
  if (op->mesh.m_x < 2) invalid("assemble_schur: need m_x >= 2");
  if (mu != 0.0) factor_unshifted_blocks(*op);
  SchurSystem sys;
  sys.op = op;
  sys.k = op->dec.k;
  sys.d = op->dec.d;
  sys.w = op->dec.side();
  sys.shift = mu;
  for (std::size_t i = 0; i < op->kinds.size(); ++i) sys.kc.push_back(build_kind_coupling(*op, static_cast<int>(i), mu));
  finish_system(sys, layout_reference);
  return sys;
}

namespace {
int kind_with(const Operator& op, bool west, bool east) {
  for (std::size_t i = 0; i < op.kinds.size(); ++i)
    if (op.kinds[i].west_iface == west && op.kinds[i].east_iface == east) return static_cast<int>(i);
  return -1;
}
}  // namespace

SchurSystem schur_from_kinds(std::shared_ptr<Operator> op, double mu, const double* G_W, const double* G_I,
                             const double* G_E, bool layout_reference) {
  if (op->mesh.m_x < 2) invalid("schur_from_kinds: need m_x >= 2");
  SchurSystem sys;
  sys.op = op;
  sys.k = op->dec.k;
  sys.d = op->dec.d;
  sys.w = op->dec.side();
  sys.shift = mu;
  const Index w = sys.w;
  sys.kc.resize(op->kinds.size());
  for (std::size_t i = 0; i < op->kinds.size(); ++i) {
    KindCoupling& kc = sys.kc[i];
    const auto kd = op->kinds[i];
    kc.cols_west = kc.rows_west = kd.west_iface ? w : 0;
    kc.cols_east = kc.rows_east = kd.east_iface ? w : 0;
    const Index m = kc.rows_west + kc.rows_east;
    kc.g = Mat(m, m);
    const double* src = (kd.west_iface && kd.east_iface) ? G_I : (kd.east_iface ? G_W : G_E);
    std::copy(src, src + m * m, kc.g.data());
  }
  finish_system(sys, layout_reference);
  return sys;
}

void export_kinds(const SchurSystem& sys, double* G_W, double* G_I, double* G_E) {
  const Operator& op = *sys.op;
  const Index w = sys.w;
  const int kw = kind_with(op, false, true), ki = kind_with(op, true, true), ke = kind_with(op, true, false);
  auto copy = [](const KindCoupling& kc, double* dst) { std::copy(kc.g.a.begin(), kc.g.a.end(), dst); };
  if (G_W) copy(sys.kc[kw], G_W);
  if (G_E) copy(sys.kc[ke], G_E);
  if (G_I) {
    if (ki >= 0)
      copy(sys.kc[ki], G_I);
    else
      std::fill(G_I, G_I + 4 * w * w, 0.0);
  }
}

// proj/src/schur.cpp:143-158
Vec apply_S(const SchurSystem& sys, const Vec& v) {
  if (static_cast<Index>(v.size()) != sys.k) invalid("apply_S: wrong length");
  sys.applies->fetch_add(1, std::memory_order_relaxed);
  const Index w = sys.w, w2 = 2 * w;
  const Operator& op = *sys.op;
  Vec y = v;
  Vec prod(static_cast<std::size_t>(4 * w));
  for (int i = 0; i < sys.d; ++i) {
    const auto& blk = sys.blocks[i];
    if (sys.materialized) {
      std::fill(prod.begin(), prod.begin() + blk.entries.rows, 0.0);
      gemv_acc(blk.entries.data(), blk.entries.rows, blk.entries.rows, w2, v.data() + i * w2, prod.data());
    } else {
      // same per-segment products read from the per-kind couplings
      const KindCoupling& gl = sys.kc[op.kind_of[i]];
      const KindCoupling& gr = sys.kc[op.kind_of[i + 1]];
      const double* vl = v.data() + i * w2;  // east-own of strip i
      const double* vr = vl + w;             // west-own of strip i+1
      Index off = 0;
      std::fill(prod.begin(), prod.end(), 0.0);
      if (i >= 1) {
        gemv_sub(gl, false, true, w, w, w, vl, prod.data() + off);
        off += w;
      }
      gemv_sub(gr, false, false, w, w, w, vr, prod.data() + off);
      off += w;
      gemv_sub(gl, true, true, w, w, w, vl, prod.data() + off);
      off += w;
      if (i <= sys.d - 2) gemv_sub(gr, true, false, w, w, w, vr, prod.data() + off);
    }
    Index off = 0;
    for (const auto& [start, len] : blk.segs) {
      for (Index t = 0; t < len; ++t) y[start + t] += prod[off + t];
      off += len;
    }
  }
  return y;
}

// proj/src/schur.cpp:160-175
Vec apply_St(const SchurSystem& sys, const Vec& v) {
  if (static_cast<Index>(v.size()) != sys.k) invalid("apply_St: wrong length");
  const Index w = sys.w, w2 = 2 * w;
  const Operator& op = *sys.op;
  Vec y = v;
  Vec g(static_cast<std::size_t>(4 * w));
  for (int i = 0; i < sys.d; ++i) {
    const auto& blk = sys.blocks[i];
    Index off = 0;
    for (const auto& [start, len] : blk.segs) {
      std::copy(v.begin() + start, v.begin() + start + len, g.begin() + off);
      off += len;
    }
    if (sys.materialized) {
      gemv_t_acc(blk.entries.data(), blk.entries.rows, blk.entries.rows, w2, g.data(), y.data() + i * w2);
    } else {
      const KindCoupling& gl = sys.kc[op.kind_of[i]];
      const KindCoupling& gr = sys.kc[op.kind_of[i + 1]];
      Index o = 0;
      double* yl = y.data() + i * w2;
      double* yr = yl + w;
      Vec tl(static_cast<std::size_t>(w), 0.0), tr(static_cast<std::size_t>(w), 0.0);
      if (i >= 1) {
        gemv_t_sub(gl, false, true, w, w, w, g.data() + o, tl.data());
        o += w;
      }
      gemv_t_sub(gr, false, false, w, w, w, g.data() + o, tr.data());
      o += w;
      gemv_t_sub(gl, true, true, w, w, w, g.data() + o, tl.data());
      o += w;
      if (i <= sys.d - 2) gemv_t_sub(gr, true, false, w, w, w, g.data() + o, tr.data());
      for (Index t = 0; t < w; ++t) {
        yl[t] += tl[t];
        yr[t] += tr[t];
      }
    }
  }
  return y;
}

// proj/src/schur.cpp:177-180
Vec apply_S_definition(const SchurSystem& sys, const Vec& v) {
  const Operator& op = *sys.op;
  const Vec t = apply_B(op, solve_A(op, apply_E(op.dec, v)));
  Vec y = v;
  for (std::size_t i = 0; i < y.size(); ++i) y[i] += t[i];
  return y;
}

// proj/src/schur.cpp:182-186
Vec schur_rhs(const SchurSystem& sys, const Vec& f) {
  const Operator& op = *sys.op;
  if (static_cast<Index>(f.size()) != op.dec.r) invalid("schur_rhs: wrong length");
  return apply_B(op, solve_A(op, f));
}

// proj/src/schur.cpp:188-216; identical blocks (same strip kinds and size)
// share one factor when dedup is set — their LU factors are bitwise equal.
void build_block_jacobi(SchurSystem& sys, int dedup) {
  const Index w = sys.w, w2 = 2 * w;
  const Operator& op = *sys.op;
  sys.jacobi.clear();
  sys.jfactors.clear();
  std::map<std::tuple<Index, int, int, int>, int> seen;
  for (int b = 0; 2 * b < sys.d; ++b) {
    const int i0 = 2 * b, i1 = std::min(2 * b + 1, sys.d - 1);
    SchurSystem::JBlock jb;
    jb.begin = i0 * w2;
    jb.size = (i1 - i0 + 1) * w2;
    const auto key = std::make_tuple(jb.size, op.kind_of[i0], op.kind_of[i0 + 1], op.kind_of[i1 + 1]);
    if (dedup) {
      auto it = seen.find(key);
      if (it != seen.end()) {
        if (dedup == 2) {
          // bitwise copy of the identical factor in its own storage: the
          // reference keeps one LU per block (memory traffic as the reference)
          jb.factor = static_cast<int>(sys.jfactors.size());
          sys.jfactors.push_back(sys.jfactors[it->second]);
        } else {
          jb.factor = it->second;
        }
        sys.jacobi.push_back(jb);
        continue;
      }
    }
    Mat m = Mat::identity(jb.size);
    // M entries = S entries inside the block (proj/src/schur.cpp:197-206)
    for (int i = i0; i <= i1; ++i) {
      const auto& blk = sys.blocks[i];
      const Mat ent = block_entries(sys, i);
      Index off = 0;
      for (const auto& [start, len] : blk.segs) {
        if (start >= jb.begin && start + len <= jb.begin + jb.size)
          for (Index c = 0; c < w2; ++c)
            for (Index r = 0; r < len; ++r) m(start - jb.begin + r, i * w2 - jb.begin + c) += ent(off + r, c);
        off += len;
      }
    }
    LU lu;
    lu.compute(m);
    if (lu.rcond() < 1e-16) singular("build_block_jacobi: singular preconditioner block " + std::to_string(b));
    jb.factor = static_cast<int>(sys.jfactors.size());
    sys.jfactors.push_back(std::move(lu));
    seen[key] = jb.factor;
    sys.jacobi.push_back(jb);
  }
}

// proj/src/schur.cpp:218-225
Vec apply_block_jacobi_inv(const SchurSystem& sys, const Vec& v) {
  if (sys.jacobi.empty()) runtime("apply_block_jacobi_inv: not built");
  if (static_cast<Index>(v.size()) != sys.k) invalid("apply_block_jacobi_inv: wrong length");
  Vec y = v;
  for (const auto& jb : sys.jacobi) sys.jfactors[jb.factor].solve_inplace(y.data() + jb.begin);
  return y;
}

// proj/src/schur.cpp:227-230
Vec recover_solution(const SchurSystem& sys, const Vec& f, const Vec& x_S) {
  const Operator& op = *sys.op;
  const Vec e = apply_E(op.dec, x_S);
  Vec g = f;
  for (std::size_t i = 0; i < g.size(); ++i) g[i] -= e[i];
  return solve_A(op, g);
}

// proj/src/schur.cpp:232-244 (built column-wise through apply_S)
Mat dense_schur(const SchurSystem& sys) {
  Mat s(sys.k, sys.k);
  Vec e(static_cast<std::size_t>(sys.k), 0.0);
  for (Index j = 0; j < sys.k; ++j) {
    e[j] = 1.0;
    const Vec c = apply_S(sys, e);
    std::copy(c.begin(), c.end(), s.col(j));
    e[j] = 0.0;
  }
  sys.applies->fetch_sub(static_cast<std::uint64_t>(sys.k), std::memory_order_relaxed);
  return s;
}

}  // namespace orc
