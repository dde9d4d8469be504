"""Host-side mirror of the reference operator/solver API over the C ABI.

Names follow the reference library (``/root/reference/proj/include/smpm``):
``apply_S``, ``apply_St``, ``apply_block_jacobi_inv``, ``apply_Z``,
``apply_Zt``, ``coarse_solve``, ``apply_P``, ``apply_Q``, ``project_out``,
``deflated_solve``, ``two_level_schwarz_solve``.  Vectors are torch CUDA
tensors of shape (nsys, k) (coarse vectors (nsys, d)); matrices are host
arrays.  Everything runs in ``lib/libsmpm_b200.so`` — there is no Python or
CPU compute path here, only plumbing.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import METHODS, ORTH, Report, SmpmError, SolveOptions, StripFactors, check, lib


def _torch():
    import torch

    return torch


def _dptr(t):
    return C.c_void_p(t.data_ptr())


def _hptr(a):
    return C.c_void_p(a.ctypes.data)


class Context:
    """One per device (``smpm_ctx``)."""

    def __init__(self, device: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise SmpmError(5, "no CUDA device visible (the B200 path has no CPU fallback)")
        torch.cuda.init()
        self.device = device
        h = C.c_void_p()
        check(lib().smpm_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().smpm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


@dataclass
class SolveResult:
    x_S: object  # torch tensor (nsys, k) or numpy for solve_host
    iterations: list
    converged: list
    final_rel_residual: list
    operator_applies: list
    krylov_s_applies: list
    mismatch_warning: list
    wall_time_s: float
    histories: list = field(repr=False, default_factory=list)


class SchurBatch:
    """``nsys`` Schur systems of one geometry on one device (``smpm_batch``)."""

    def __init__(self, ctx: Context, n: int, m_x: int, m_z: int, nsys: int = 1):
        self.ctx = ctx
        h = C.c_void_p()
        check(lib().smpm_batch_create(ctx.h, n, m_x, m_z, nsys, C.byref(h)))
        self.h = h
        k, d, w = C.c_longlong(), C.c_int(), C.c_int()
        check(lib().smpm_batch_dims(h, C.byref(k), C.byref(d), C.byref(w)))
        self.n, self.m_x, self.m_z, self.nsys = n, m_x, m_z, nsys
        self.k, self.d, self.w = k.value, d.value, w.value
        self.spectral = False
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            lib().smpm_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # ---- setup ----------------------------------------------------------
    def set_couplings(self, sys: int, G_W, G_I, G_E):
        w = self.w
        gw = np.asfortranarray(G_W, dtype=np.float64)
        ge = np.asfortranarray(G_E, dtype=np.float64)
        if gw.shape != (w, w) or ge.shape != (w, w):
            raise SmpmError(1, "G_W/G_E must be w x w")
        gi = None
        if G_I is not None:
            gi = np.asfortranarray(G_I, dtype=np.float64)
            if gi.shape != (2 * w, 2 * w):
                raise SmpmError(1, "G_I must be 2w x 2w")
        check(lib().smpm_batch_set_couplings(self.h, sys, _hptr(gw), _hptr(gi) if gi is not None else None, _hptr(ge)))

    def set_spectral(self, npairs: int, T, T_inv, gamma):
        """Spectral factors of the couplings (smpm_batch_set_spectral): T, T_inv
        w x w; gamma (nsys, 6, w - npairs) complex."""
        w = self.w
        t = np.asfortranarray(T, dtype=np.float64)
        ti = np.asfortranarray(T_inv, dtype=np.float64)
        g = np.ascontiguousarray(np.asarray(gamma, dtype=np.complex128))
        if t.shape != (w, w) or ti.shape != (w, w):
            raise SmpmError(1, "T/T_inv must be w x w")
        if g.shape != (self.nsys, 6, w - npairs):
            raise SmpmError(1, "gamma must be (nsys, 6, w - npairs)")
        gv = g.view(np.float64)
        check(lib().smpm_batch_set_spectral(self.h, int(npairs), _hptr(t), _hptr(ti), _hptr(gv)))
        self.spectral = True

    def set_interface_blocks(self, sys: int, blocks):
        """blocks: list of (entries[rows x 2w], [(start, len), ...]) in the
        reference's InterfaceBlock layout (proj/include/smpm/schur.hpp:32-36)."""
        d = len(blocks)
        ents = [np.asfortranarray(e, dtype=np.float64) for e, _ in blocks]
        starts = [np.array([s for s, _ in segs], dtype=np.int64) for _, segs in blocks]
        lens = [np.array([l for _, l in segs], dtype=np.int64) for _, segs in blocks]
        ep = (C.c_void_p * d)(*[e.ctypes.data for e in ents])
        rows = (C.c_longlong * d)(*[e.shape[0] for e in ents])
        sp = (C.c_void_p * d)(*[s.ctypes.data for s in starts])
        lp = (C.c_void_p * d)(*[l.ctypes.data for l in lens])
        ns = (C.c_int * d)(*[len(s) for s in starts])
        check(lib().smpm_batch_set_interface_blocks(self.h, sys, ep, rows, sp, lp, ns))

    def load_schur_blocks(self, sys: int, path):
        """The reference's dump_schur_blocks file (proj/src/schur.cpp:246-297) for system `sys`."""
        check(lib().smpm_batch_load_schur_blocks(self.h, sys, str(path).encode()))

    def set_nullspace(self, sys: int, u_S):
        u = np.ascontiguousarray(u_S, dtype=np.float64)
        if u.size != self.k:
            raise SmpmError(1, "u_S must have length k")
        check(lib().smpm_batch_set_nullspace(self.h, sys, _hptr(u)))

    def set_fdm(self, npairs: int, T, T_inv, fac: dict):
        """Device-side setup (smpm_batch_set_fdm): the shared z eigenbasis and the
        strip factors (StripFDM.strip_factors(mus)); finalize() then builds every
        system's spectral diagonals, dense couplings, block-Jacobi inverses, row
        sums and coarse matrix on the device.  Replaces set_couplings +
        set_spectral (+ set_strip_factors)."""
        w = self.w
        t = np.asfortranarray(T, dtype=np.float64)
        ti = np.asfortranarray(T_inv, dtype=np.float64)
        if t.shape != (w, w) or ti.shape != (w, w):
            raise SmpmError(1, "T/T_inv must be w x w")
        sf, keep = self._strip_struct(fac)
        check(lib().smpm_batch_set_fdm(self.h, int(npairs), _hptr(t), _hptr(ti), C.byref(sf)))
        self.spectral = True
        del keep

    def set_strip_factors(self, fac: dict):
        """Fast-diagonalisation factors of the strip operator (smpm_batch_set_strip_factors):
        fac from StripFDM.strip_factors(mus) — Vx, Vx_inv, lx (3 kinds each, complex),
        lz (nmode complex), tW, tE (n), tau, mu (nsys)."""
        sf, keep = self._strip_struct(fac)
        check(lib().smpm_batch_set_strip_factors(self.h, C.byref(sf)))
        del keep

    def _strip_struct(self, fac: dict):
        keep = []

        def cplx(a):
            a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128).reshape(-1, order="F"))
            keep.append(a)
            return a.ctypes.data

        def real(a):
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
            keep.append(a)
            return a.ctypes.data

        sf = StripFactors()
        for i in range(3):
            sf.Vx[i] = cplx(fac["Vx"][i])
            sf.Vx_inv[i] = cplx(fac["Vx_inv"][i])
            sf.lx[i] = cplx(fac["lx"][i])
        sf.lz = cplx(fac["lz"])
        sf.tW = real(fac["tW"])
        sf.tE = real(fac["tE"])
        sf.tau = float(fac["tau"])
        mu = np.asarray(fac["mu"], dtype=np.float64)
        if mu.size != self.nsys:
            raise SmpmError(1, "mu must have one shift per system")
        sf.mu = real(mu)
        return sf, keep

    def finalize(self):
        check(lib().smpm_batch_finalize(self.h))
        return self

    def coarse_info(self):
        Cm = np.zeros((self.nsys, self.d, self.d))
        tri = (C.c_int * self.nsys)()
        sing = (C.c_int * self.nsys)()
        check(lib().smpm_batch_coarse_info(self.h, _hptr(Cm), tri, sing))
        return np.transpose(Cm, (0, 2, 1)).copy(), list(tri), list(sing)

    # ---- operators --------------------------------------------------------
    def _stream(self):
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def _vec(self, v, n):
        torch = _torch()
        if not (isinstance(v, torch.Tensor) and v.is_cuda and v.dtype == torch.float64):
            raise SmpmError(1, "expected a float64 CUDA tensor")
        v = v.contiguous()
        if v.numel() != self.nsys * n:
            raise SmpmError(1, f"expected {self.nsys} x {n} elements, got {v.numel()}")
        return v.view(self.nsys, n)

    def _op(self, fn, v, nin, nout):
        torch = _torch()
        v = self._vec(v, nin)
        y = torch.empty((self.nsys, nout), dtype=torch.float64, device=v.device)
        check(getattr(lib(), fn)(self.h, _dptr(v), _dptr(y), self._stream()))
        return y

    def apply_S(self, v):  # proj/src/schur.cpp:143-158
        return self._op("smpm_apply_S", v, self.k, self.k)

    def apply_St(self, v):  # proj/src/schur.cpp:160-175
        return self._op("smpm_apply_St", v, self.k, self.k)

    def apply_block_jacobi_inv(self, v):  # proj/src/schur.cpp:218-225
        return self._op("smpm_apply_block_jacobi_inv", v, self.k, self.k)

    def apply_Z(self, y):  # proj/src/deflation.cpp:8-14
        return self._op("smpm_apply_Z", y, self.d, self.k)

    def apply_Zt(self, v):  # proj/src/deflation.cpp:16-22
        return self._op("smpm_apply_Zt", v, self.k, self.d)

    def coarse_solve(self, b):  # proj/src/deflation.cpp:71-92
        return self._op("smpm_coarse_solve", b, self.d, self.d)

    def apply_Q(self, v):  # proj/src/deflation.cpp:98-100
        return self._op("smpm_apply_Q", v, self.k, self.k)

    def apply_P(self, v, fused: bool = False):  # proj/src/deflation.cpp:94-96
        torch = _torch()
        v = self._vec(v, self.k)
        y = torch.empty_like(v)
        check(lib().smpm_apply_P(self.h, _dptr(v), _dptr(y), int(bool(fused)), self._stream()))
        return y

    def project_out(self, v, direction):  # proj/src/nullspace.cpp:92
        """v - dir (dir . v) per system; any per-system length (k for u_S on b_S,
        r for u_L on f).  A zero direction row leaves that system's row unchanged."""
        torch = _torch()
        n = v.numel() // self.nsys if isinstance(v, torch.Tensor) else -1
        v = self._vec(v, n)
        dr = self._vec(direction, n)
        y = torch.empty_like(v)
        check(lib().smpm_project_out(self.h, C.c_longlong(n), _dptr(v), _dptr(dr), _dptr(y), self._stream()))
        return y

    # ---- strip solves -------------------------------------
    @property
    def r(self):
        return self.m_x * self.m_z * self.n * self.n

    def schur_rhs(self, f):  # proj/src/schur.cpp:182-186
        torch = _torch()
        f = self._vec(f, self.r)
        y = torch.empty((self.nsys, self.k), dtype=torch.float64, device=f.device)
        check(lib().smpm_schur_rhs(self.h, _dptr(f), _dptr(y), self._stream()))
        return y

    def recover_solution(self, f, x_S):  # proj/src/schur.cpp:227-230
        torch = _torch()
        f = self._vec(f, self.r)
        x = self._vec(x_S, self.k)
        u = torch.empty((self.nsys, self.r), dtype=torch.float64, device=f.device)
        check(lib().smpm_recover_solution(self.h, _dptr(f), _dptr(x), _dptr(u), self._stream()))
        return u

    # ---- solves -----------------------------------------------------------
    @staticmethod
    def options(tol=1e-10, max_iter=100, restart=0, orth="cgs2", fuse_deflation=True, final_residual_check=True):
        o = SolveOptions()
        o.tol = tol
        o.max_iter = max_iter
        o.restart = restart
        o.orth = ORTH[orth]
        o.fuse_deflation = int(bool(fuse_deflation))
        o.final_residual_check = int(bool(final_residual_check))
        return o

    def _collect(self, x, reps, hist, cap):
        its = [reps[i].iterations for i in range(self.nsys)]
        hs = [hist[i, : reps[i].history_len].copy() for i in range(self.nsys)] if hist is not None else []
        return SolveResult(
            x, its, [bool(reps[i].converged) for i in range(self.nsys)],
            [reps[i].final_rel_residual for i in range(self.nsys)],
            [reps[i].operator_applies for i in range(self.nsys)],
            [reps[i].krylov_s_applies for i in range(self.nsys)],
            [bool(reps[i].mismatch_warning) for i in range(self.nsys)],
            reps[0].wall_time_s if self.nsys else 0.0, hs)

    def solve(self, b_S, method="dbj", tol=1e-10, max_iter=100, restart=0, orth="cgs2", fuse_deflation=True,
              history=True):
        torch = _torch()
        b = self._vec(b_S, self.k)
        x = torch.empty_like(b)
        o = self.options(tol, max_iter, restart, orth, fuse_deflation)
        reps = (Report * self.nsys)()
        cap = min(max_iter, self.k) + 2
        hist = np.zeros((self.nsys, cap)) if history else None
        check(lib().smpm_solve(self.h, METHODS[method], _dptr(b), _dptr(x), C.byref(o), reps,
                               _hptr(hist) if hist is not None else None, self._stream()))
        return self._collect(x, reps, hist, cap)

    def solve_stacked(self, b_S, method="dbj", tol=1e-10, max_iter=100, restart=0, history=True):
        """One GMRES over all systems stacked (proj/src/helmholtz.cpp:187-246); one report."""
        torch = _torch()
        b = self._vec(b_S, self.k)
        x = torch.empty_like(b)
        o = self.options(tol, max_iter, restart, "cgs2", True)
        rep = Report()
        cap = min(max_iter, self.k) + 2
        hist = np.zeros(cap) if history else None
        check(lib().smpm_solve_stacked(self.h, METHODS[method], _dptr(b), _dptr(x), C.byref(o), C.byref(rep),
                                       _hptr(hist) if hist is not None else None, self._stream()))
        return SolveResult(x, [rep.iterations], [bool(rep.converged)], [rep.final_rel_residual],
                           [rep.operator_applies], [rep.krylov_s_applies], [bool(rep.mismatch_warning)],
                           rep.wall_time_s, [hist[: rep.history_len].copy()] if hist is not None else [])

    def deflated_solve(self, b_S, tol=1e-10, max_iter=100, **kw):  # proj/src/deflation.cpp:102-122
        return self.solve(b_S, "dbj", tol, max_iter, **kw)

    def two_level_schwarz_solve(self, b_S, tol=1e-10, max_iter=100, **kw):  # proj/src/deflation.cpp:124-143
        return self.solve(b_S, "2las", tol, max_iter, **kw)

    def solve_host(self, b_S_host, method="dbj", tol=1e-10, max_iter=100, restart=0, orth="cgs2",
                   fuse_deflation=True, out=None):
        """End-to-end: host b_S in, host x_S out (copies inside the call)."""
        b = np.ascontiguousarray(b_S_host, dtype=np.float64).reshape(self.nsys, self.k)
        x = out if out is not None else np.empty_like(b)
        o = self.options(tol, max_iter, restart, orth, fuse_deflation)
        reps = (Report * self.nsys)()
        check(lib().smpm_solve_host(self.h, METHODS[method], _hptr(b), _hptr(x), C.byref(o), reps, None))
        return self._collect(x, reps, None, 0)

    def prefetch_rhs(self, b_S_host):
        """Start the upload of a host right-hand-side array ahead of its solve_host
        (smpm_prefetch_rhs); the array must be the very object later passed to
        solve_host (same memory) and stay unchanged until then."""
        b = np.ascontiguousarray(b_S_host, dtype=np.float64).reshape(self.nsys, self.k)
        if b.ctypes.data != np.asarray(b_S_host).ctypes.data:
            raise SmpmError(1, "prefetch_rhs needs a C-contiguous float64 array (no copy)")
        check(lib().smpm_prefetch_rhs(self.h, _hptr(b)))

    def tune(self, **knobs):
        """Performance knobs (smpm_batch_set_tuning), e.g. tune(grid_max=4, pdl=0)."""
        for k, v in knobs.items():
            check(lib().smpm_batch_set_tuning(self.h, k.encode(), int(v)))
        return self

    def set_allreduce(self, fn):
        """Stacked solve across ranks (smpm_batch_set_allreduce): fn(ptr, count,
        stream) sums `count` doubles at device pointer `ptr` in place over the
        ranks, ordered on CUDA stream `stream`; None: single rank.  See
        dist.nccl_allreduce_hook."""
        from ._lib import ALLREDUCE_FN

        if fn is None:
            self._ar = None
            check(lib().smpm_batch_set_allreduce(self.h, C.cast(None, ALLREDUCE_FN), None))
            return self

        def thunk(_user, ptr, count, stream):
            try:
                fn(int(ptr), int(count), int(stream or 0))
                return 0
            except Exception:  # the C side turns a non-zero return into SMPM_ERUNTIME
                import traceback

                traceback.print_exc()
                return 1

        self._ar = ALLREDUCE_FN(thunk)  # keep the callback alive
        check(lib().smpm_batch_set_allreduce(self.h, self._ar, None))
        return self

    def query(self, key: str) -> int:
        """Which kernels this batch runs (smpm_batch_query), e.g. query("xform_parity")."""
        v = C.c_longlong()
        check(lib().smpm_batch_query(self.h, key.encode(), C.byref(v)))
        return int(v.value)

    def trace(self, which: int, path):
        """Grid-tail phase trace into `path` (smpm_batch_set_trace); None: off."""
        check(lib().smpm_batch_set_trace(self.h, int(which), path.encode() if path else None))

    def tune_from_env(self):
        """Tools only: SMPM_<KNOB>=<int> environment variables -> tune(); the
        library itself reads no environment."""
        import os

        from ._lib import TUNING_KEYS

        for k in TUNING_KEYS:
            v = os.environ.get("SMPM_" + k.upper())
            if v is not None:
                self.tune(**{k: int(v)})
        for which, name in ((0, "SMPM_GT_TRACE"), (1, "SMPM_GT_TRACE2")):
            if os.environ.get(name):
                self.trace(which, os.environ[name])
        return self

    def profile(self, enable=None):
        """Per-kernel-class device time (ms) and launch counts accumulated since
        the last reset; enable=True/False resets and switches timing."""
        from ._lib import PROFILE_CLASSES

        n = len(PROFILE_CLASSES)
        ms = (C.c_double * n)()
        cnt = (C.c_longlong * n)()
        flag = -1 if enable is None else int(bool(enable))
        check(lib().smpm_batch_profile(self.h, flag, ms, cnt, n))
        return {name: (ms[i], cnt[i]) for i, name in enumerate(PROFILE_CLASSES)}

    @property
    def launch_count(self) -> int:
        return int(lib().smpm_batch_launch_count(self.h))
