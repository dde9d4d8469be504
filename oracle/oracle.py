"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/build/liboracle.so``, the C++ restatement of
the reference library (``/root/reference/proj``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this
module, and only as the checker / CPU baseline — never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")

METHODS = {"schur": 0, "bj": 1, "dbj": 2, "2las": 3}


def build() -> str:
    """Compile the oracle (make in oracle/)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True, stdout=subprocess.DEVNULL)
    return LIB_PATH


_lib = None


class OracleError(RuntimeError):
    pass


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("mismatch", C.c_int),
        ("history_len", C.c_int),
        ("operator_applies", C.c_longlong),
        ("krylov_s_applies", C.c_longlong),
        ("final_rel_residual", C.c_double),
        ("wall_time_s", C.c_double),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_problem_create.restype = vp
        L.orc_problem_create.argtypes = [ip, ip, ip, C.c_double, C.c_double, C.c_double]
        for f in ("orc_system_create",):
            getattr(L, f).restype = vp
            getattr(L, f).argtypes = [vp, C.c_double, ip]
        L.orc_system_from_kinds.restype = vp
        L.orc_system_from_kinds.argtypes = [vp, C.c_double, dp, dp, dp, ip]
        L.orc_coarse_create.restype = vp
        L.orc_coarse_create.argtypes = [vp, dp]
        L.orc_applies.restype = C.c_ulonglong
        L.orc_applies.argtypes = [vp]
        for f in ("orc_problem_free", "orc_system_free", "orc_coarse_free"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = None
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise OracleError(f"oracle error {rc}: {lib().orc_last_error().decode()}")


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _vec(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise ValueError(f"expected length {n}, got {a.size}")
    return a


def set_threads(n: int):
    _chk(lib().orc_set_threads(int(n)))


def rng_uniforms(seed: int, stream: int, n: int):
    """Rng(seed).stream(stream) uniforms from the C++ engine (stream < 0: Rng(seed))."""
    out = np.zeros(n)
    _chk(lib().orc_rng_uniforms(C.c_ulonglong(seed), C.c_longlong(stream), int(n), _p(out)))
    return out


def gll(n: int):
    nodes, weights, diff = np.zeros(n), np.zeros(n), np.zeros((n, n), order="F")
    _chk(lib().orc_gll(n, _p(nodes), _p(weights), _p(diff)))
    return nodes, weights, np.asfortranarray(diff)


class Problem:
    """Mesh + strip decomposition + operator split (proj/src/mesh.cpp, proj/src/operator.cpp)."""

    def __init__(self, n, m_x, m_z, l_x, l_z, c_tau=2.0):
        L = lib()
        self.h = L.orc_problem_create(n, m_x, m_z, float(l_x), float(l_z), float(c_tau))
        if not self.h:
            raise OracleError(L.orc_last_error().decode())
        self.n, self.m_x, self.m_z, self.l_x, self.l_z, self.c_tau = n, m_x, m_z, l_x, l_z, c_tau
        info = (C.c_longlong * 6)()
        dinfo = (C.c_double * 4)()
        _chk(L.orc_problem_info(C.c_void_p(self.h), info, dinfo))
        self.r, self.k, self.d, self.w, self.q, self.nkinds = [int(v) for v in info]
        self.tau, self.h_x, self.h_z, self.eta = list(dinfo)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and C is not None:  # not at interpreter exit
            try:
                lib().orc_problem_free(C.c_void_p(self.h))
            except Exception:
                pass
            self.h = None

    def coords(self):
        x, z = np.zeros(self.r), np.zeros(self.r)
        _chk(lib().orc_problem_coords(C.c_void_p(self.h), _p(x), _p(z)))
        return x, z

    def gamma_to_node(self):
        out = np.zeros(self.k, dtype=np.int64)
        _chk(lib().orc_gamma_to_node(C.c_void_p(self.h), out.ctypes.data_as(C.POINTER(C.c_longlong))))
        return out

    def strip_matrix(self, s):
        out = np.zeros((self.q, self.q), order="F")
        _chk(lib().orc_strip_matrix(C.c_void_p(self.h), int(s), _p(out)))
        return out

    def _op(self, name, v, nin, nout):
        v = _vec(v, nin)
        out = np.zeros(nout)
        _chk(getattr(lib(), name)(C.c_void_p(self.h), _p(v), _p(out)))
        return out

    def apply_A(self, u): return self._op("orc_apply_A", u, self.r, self.r)
    def apply_B(self, u): return self._op("orc_apply_B", u, self.r, self.k)
    def apply_Bt(self, v): return self._op("orc_apply_Bt", v, self.k, self.r)
    def apply_L(self, u): return self._op("orc_apply_L", u, self.r, self.r)
    def solve_A(self, f): return self._op("orc_solve_A", f, self.r, self.r)
    def solve_At(self, f): return self._op("orc_solve_At", f, self.r, self.r)
    def apply_E(self, v): return self._op("orc_apply_E", v, self.k, self.r)
    def apply_Et(self, u): return self._op("orc_apply_Et", u, self.r, self.k)
    def apply_Z(self, y): return self._op("orc_apply_Z", y, self.d, self.k)
    def apply_Zt(self, v): return self._op("orc_apply_Zt", v, self.k, self.d)

    def dense_L(self):
        out = np.zeros((self.r, self.r), order="F")
        _chk(lib().orc_dense_L(C.c_void_p(self.h), _p(out)))
        return out

    def shifted_solve(self, mu, b):
        b = _vec(b, self.r)
        x = np.zeros(self.r)
        _chk(lib().orc_shifted_solve(C.c_void_p(self.h), C.c_double(mu), _p(b), _p(x)))
        return x

    def manufactured(self, kmax, decay, seed=1234, stream=0, forcing_only=False, mu=0.0):
        """Seeded cosine field u and f = (Lap - mu) u (or f = u when forcing_only)."""
        f, u = np.zeros(self.r), np.zeros(self.r)
        _chk(lib().orc_manufactured(C.c_void_p(self.h), int(kmax), int(bool(decay)), C.c_ulonglong(seed),
                                    C.c_ulonglong(stream), int(bool(forcing_only)), C.c_double(mu), _p(f), _p(u)))
        return f, u


@dataclass
class SolveResult:
    x_S: np.ndarray
    iterations: int
    converged: bool
    mismatch: bool
    final_rel_residual: float
    operator_applies: int
    krylov_s_applies: int
    wall_time_s: float
    history: np.ndarray = field(repr=False)


def _result(x, rep, hist):
    return SolveResult(x, rep.iterations, bool(rep.converged), bool(rep.mismatch), rep.final_rel_residual,
                       rep.operator_applies, rep.krylov_s_applies, rep.wall_time_s,
                       hist[: rep.history_len].copy())


class System:
    """Schur system (proj/src/schur.cpp) for wavenumber shift mu (0 = Poisson)."""

    def __init__(self, prob: Problem, mu=0.0, layout_reference=True, kinds=None):
        L = lib()
        self.prob = prob
        self.mu = float(mu)
        if kinds is None:
            self.h = L.orc_system_create(C.c_void_p(prob.h), C.c_double(mu), int(layout_reference))
        else:
            gw, gi, ge = [np.asfortranarray(g, dtype=np.float64) for g in kinds]
            self.h = L.orc_system_from_kinds(C.c_void_p(prob.h), C.c_double(mu), _p(gw), _p(gi), _p(ge),
                                             int(layout_reference))
        if not self.h:
            raise OracleError(L.orc_last_error().decode())
        self.k, self.w, self.d = prob.k, prob.w, prob.d
        self.coarse = None

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and C is not None:  # not at interpreter exit
            try:
                lib().orc_system_free(C.c_void_p(self.h))
            except Exception:
                pass
            self.h = None

    @property
    def frob(self):
        v = C.c_double()
        _chk(lib().orc_system_frob(C.c_void_p(self.h), C.byref(v)))
        return v.value

    @property
    def applies(self):
        return int(lib().orc_applies(C.c_void_p(self.h)))

    def kinds(self):
        w = self.w
        gw, gi, ge = np.zeros((w, w), order="F"), np.zeros((2 * w, 2 * w), order="F"), np.zeros((w, w), order="F")
        _chk(lib().orc_export_kinds(C.c_void_p(self.h), _p(gw), _p(gi), _p(ge)))
        return gw, gi, ge

    def build_bj(self, dedup=True):
        _chk(lib().orc_build_bj(C.c_void_p(self.h), int(dedup)))

    def _op(self, name, v, nin, nout):
        v = _vec(v, nin)
        out = np.zeros(nout)
        _chk(getattr(lib(), name)(C.c_void_p(self.h), _p(v), _p(out)))
        return out

    def apply_S(self, v): return self._op("orc_apply_S", v, self.k, self.k)
    def apply_St(self, v): return self._op("orc_apply_St", v, self.k, self.k)
    def apply_S_definition(self, v): return self._op("orc_apply_S_definition", v, self.k, self.k)
    def bj_inv(self, v): return self._op("orc_bj_inv", v, self.k, self.k)
    def schur_rhs(self, f): return self._op("orc_schur_rhs", f, self.prob.r, self.k)

    def recover(self, f, x_S):
        f, x_S = _vec(f, self.prob.r), _vec(x_S, self.k)
        u = np.zeros(self.prob.r)
        _chk(lib().orc_recover(C.c_void_p(self.h), _p(f), _p(x_S), _p(u)))
        return u

    def dump_blocks(self, path):
        """The reference's binary block file (proj/src/schur.cpp:246-264); needs layout_reference."""
        _chk(lib().orc_dump_schur_blocks(C.c_void_p(self.h), str(path).encode()))

    def dense_S(self):
        out = np.zeros((self.k, self.k), order="F")
        _chk(lib().orc_dense_S(C.c_void_p(self.h), _p(out)))
        return out

    def nullspace(self, dense_limit=3200):
        u_S, u_L = np.zeros(self.k), np.zeros(self.prob.r)
        its, sigma = C.c_int(), C.c_double()
        _chk(lib().orc_nullspace(C.c_void_p(self.h), _p(u_S), _p(u_L), C.byref(its), C.byref(sigma),
                                 C.c_longlong(dense_limit)))
        return u_S, u_L, its.value, sigma.value

    def build_coarse(self, u_S=None):
        L = lib()
        if u_S is not None:
            u_S = _vec(u_S, self.k)
            self._u_S = u_S
        h = L.orc_coarse_create(C.c_void_p(self.h), _p(u_S) if u_S is not None else None)
        if not h:
            raise OracleError(L.orc_last_error().decode())
        self.coarse = Coarse(h, self.d)
        return self.coarse

    def apply_P(self, v):
        v = _vec(v, self.k)
        y = np.zeros(self.k)
        _chk(lib().orc_apply_P(C.c_void_p(self.coarse.h), C.c_void_p(self.h), _p(v), _p(y)))
        return y

    def apply_Q(self, v):
        v = _vec(v, self.k)
        y = np.zeros(self.k)
        _chk(lib().orc_apply_Q(C.c_void_p(self.coarse.h), C.c_void_p(self.h), _p(v), _p(y)))
        return y

    def solve(self, b_S, method="dbj", tol=1e-10, max_iter=2000, restart=0) -> SolveResult:
        b_S = _vec(b_S, self.k)
        x = np.zeros(self.k)
        rep = Report()
        cap = max(max_iter, 1) + 2
        hist = np.zeros(cap)
        cs = C.c_void_p(self.coarse.h) if self.coarse is not None else None
        _chk(lib().orc_solve(C.c_void_p(self.h), cs, METHODS[method], _p(b_S), C.c_double(tol), int(max_iter),
                             int(restart), _p(x), C.byref(rep), _p(hist), cap))
        return _result(x, rep, hist)


class Coarse:
    def __init__(self, h, d):
        self.h, self.d = h, d

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and C is not None:  # not at interpreter exit
            try:
                lib().orc_coarse_free(C.c_void_p(self.h))
            except Exception:
                pass
            self.h = None

    def info(self):
        s, t = C.c_int(), C.c_int()
        Cm = np.zeros((self.d, self.d), order="F")
        u_C = np.zeros(self.d)
        _chk(lib().orc_coarse_info(C.c_void_p(self.h), C.byref(s), C.byref(t), _p(Cm), _p(u_C)))
        return bool(s.value), bool(t.value), Cm, (u_C if s.value else None)

    def solve(self, b):
        b = _vec(b, self.d)
        x = np.zeros(self.d)
        _chk(lib().orc_coarse_solve(C.c_void_p(self.h), _p(b), _p(x)))
        return x


def project_out(v, direction):
    v = _vec(v)
    direction = _vec(direction, v.size)
    out = np.zeros(v.size)
    _chk(lib().orc_project_out(C.c_longlong(v.size), _p(v), _p(direction), _p(out)))
    return out


def solve_many(systems, b, method="dbj", tol=1e-10, max_iter=100, restart=0, threads=1):
    """Independent solves across host threads (parallel_trials analogue)."""
    n = len(systems)
    k = systems[0].k
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(n, k)
    x = np.zeros((n, k))
    reps = (Report * n)()
    sys_arr = (C.c_void_p * n)(*[s.h for s in systems])
    cs_arr = (C.c_void_p * n)(*[s.coarse.h for s in systems])
    _chk(lib().orc_solve_many(sys_arr, cs_arr, n, METHODS[method], _p(b), C.c_double(tol), int(max_iter),
                              int(restart), _p(x), reps, int(threads)))
    return x, [reps[i] for i in range(n)]


def solve_stacked(systems, b, method="dbj", tol=1e-10, max_iter=100, restart=0):
    """Stacked solve of proj/src/helmholtz.cpp:187-246: one GMRES over every
    system's (deflated) right-hand side with the block-diagonal operator."""
    n = len(systems)
    k = systems[0].k
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(n, k)
    x = np.zeros((n, k))
    rep = Report()
    cap = max_iter + 2
    hist = np.zeros(cap)
    sys_arr = (C.c_void_p * n)(*[s.h for s in systems])
    cs_arr = (C.c_void_p * n)(*[s.coarse.h for s in systems])
    _chk(lib().orc_solve_stacked(sys_arr, cs_arr, n, METHODS[method], _p(b), C.c_double(tol), int(max_iter),
                                 int(restart), _p(x), C.byref(rep), _p(hist), cap))
    return _result(x, rep, hist)


def gmres_dense(A, b, tol=1e-10, max_iter=200, restart=0):
    A = np.asfortranarray(A, dtype=np.float64)
    b = _vec(b, A.shape[0])
    x = np.zeros(A.shape[0])
    rep = Report()
    hist = np.zeros(max_iter + 2)
    _chk(lib().orc_gmres_dense(C.c_longlong(A.shape[0]), _p(A), _p(b), C.c_double(tol), int(max_iter),
                               int(restart), _p(x), C.byref(rep), _p(hist), max_iter + 2))
    return _result(x, rep, hist)


@dataclass
class PoissonSetup:
    """proj/include/smpm/solver.hpp:18-24 / proj/src/solver.cpp:26-39."""
    prob: Problem
    sys: System
    u_S: np.ndarray
    u_L: np.ndarray


def build_poisson_setup(n, m_x, m_z, l_x, l_z, c_tau=2.0, layout_reference=True, dense_limit=3200):
    prob = Problem(n, m_x, m_z, l_x, l_z, c_tau)
    sys = System(prob, 0.0, layout_reference)
    sys.build_bj()
    u_S, u_L, _, _ = sys.nullspace(dense_limit)
    sys.build_coarse(u_S)
    return PoissonSetup(prob, sys, u_S, u_L)


def solve_poisson(setup: PoissonSetup, f, method="dbj", tol=1e-10, max_iter=2000, restart=0, with_checks=False):
    """Algorithm 1 (proj/src/solver.cpp:41-104)."""
    sys = setup.sys
    f_t = project_out(f, setup.u_L)
    b_S = project_out(sys.schur_rhs(f_t), setup.u_S)
    res = sys.solve(b_S, method, tol, max_iter, restart)
    bn = np.linalg.norm(b_S)
    sr = sys.apply_S(res.x_S) - b_S
    out = {"b_S": b_S, "f_tilde": f_t, "res": res,
           "schur_rel_residual": np.linalg.norm(sr) / bn if bn > 0 else np.linalg.norm(sr)}
    out["u"] = sys.recover(f_t, res.x_S)
    if with_checks:
        out["residual_bound_lhs"] = np.linalg.norm(setup.prob.apply_L(out["u"]) - f_t)
        out["residual_bound_rhs"] = np.linalg.norm(sr)
    return out
