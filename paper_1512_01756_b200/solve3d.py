"""The 3D Fourier-extended solve on the device (``solve_3d``,
/root/reference/proj/src/helmholtz.cpp:150-297): transverse FFT, per-wavenumber
right-hand sides, the Schur solves of every (mode, real / imaginary part)
system in one batch (independent GMRES, or the stacked branch), per-mode
recovery and the inverse FFT — each step one call into the C ABI
(``smpm_fourier_y``, ``smpm_schur_rhs``, ``smpm_solve`` / ``smpm_solve_stacked``,
``smpm_recover_solution``, ``smpm_inverse_fourier_y``). Python only orders the
calls and applies the two rank-one null-space projections of the j = 0 mode.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

from ._lib import check, lib
from .fdm import Geometry, StripFDM
from .schur import SchurBatch


def _torch():
    import torch

    return torch


def fourier_y(field, m_y):
    """(m_y, r) plane-major field -> (m_y, r) coefficients, system 2 j + part
    (proj/src/fourier.cpp:47-62)."""
    torch = _torch()
    field = field.contiguous()
    r = field.shape[1]
    out = torch.empty((m_y, r), dtype=torch.float64, device=field.device)
    check(lib().smpm_fourier_y(r, m_y, C.c_void_p(field.data_ptr()), C.c_void_p(out.data_ptr()),
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def inverse_fourier_y(coeff, m_y):
    """(m_y, r) coefficients (system 2 j + part) -> (m_y, r) field (proj/src/fourier.cpp:64-86)."""
    torch = _torch()
    coeff = coeff.contiguous()
    r = coeff.shape[1]
    out = torch.empty((m_y, r), dtype=torch.float64, device=coeff.device)
    check(lib().smpm_inverse_fourier_y(r, m_y, C.c_void_p(coeff.data_ptr()), C.c_void_p(out.data_ptr()),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


@dataclass
class Solve3dResult:
    u: object                 # (m_y, r) torch tensor
    iterations: list          # per system (2 j + part), or [stacked count]
    converged: list
    rel_residual: float       # stacked Schur relative residual (proj/src/helmholtz.cpp:276-281)


class Fourier3D:
    """FourierContext (proj/src/helmholtz.cpp:112-147) on one device: the m_y / 2
    wavenumber systems, each twice (real and imaginary part), k_j = 2 pi j / l_y."""

    def __init__(self, ctx, n, m_x, m_z, l_x, l_z, m_y, l_y, c_tau=2.0):
        if m_y < 2 or m_y & (m_y - 1):
            raise ValueError("m_y must be a power of two >= 2")
        self.m_y, self.half = m_y, m_y // 2
        self.geo = Geometry(n, m_x, m_z, l_x, l_z, c_tau)
        F = StripFDM(self.geo, "cuda")
        self.mus = [(2.0 * math.pi * j / l_y) ** 2 for j in range(self.half)]
        sys_mus = [mu for mu in self.mus for _ in range(2)]
        GW, GI, GE = F.couplings(self.mus)
        self.u_S, self.u_L = F.nullspace()
        b = SchurBatch(ctx, n, m_x, m_z, 2 * self.half)
        for j in range(self.half):
            for p in range(2):
                b.set_couplings(2 * j + p, GW[j], GI[j] if m_x > 2 else None, GE[j])
                if j == 0:
                    b.set_nullspace(2 * j + p, self.u_S)
        b.set_spectral(*F.spectral(sys_mus))
        b.finalize()
        b.set_strip_factors(F.strip_factors(sys_mus))
        self.batch = b

    def solve(self, f, method="dbj", tol=1e-10, max_iter=100, restart=0, stacked=False):
        """f: (m_y, r) torch CUDA tensor (the reference's r x m_y matrix, column-major)."""
        torch = _torch()
        b = self.batch
        fh = fourier_y(f, self.m_y)
        uL = torch.tensor(self.u_L, device=fh.device)
        uS = torch.tensor(self.u_S, device=fh.device)
        # j = 0 consistency projections (proj/src/helmholtz.cpp:159-160, 168-169)
        dl = torch.zeros_like(fh)
        dl[0:2] = uL
        fh = b.project_out(fh, dl)
        bS = b.schur_rhs(fh)
        dirs = torch.zeros_like(bS)
        dirs[0:2] = uS
        bS = b.project_out(bS, dirs)
        if stacked:
            res = b.solve_stacked(bS, method, tol, max_iter, restart, history=False)
        else:
            res = b.solve(bS, method, tol, max_iter, restart, history=False)
        uh = b.recover_solution(fh, res.x_S)
        u = inverse_fourier_y(uh, self.m_y)
        # residual accounting (proj/src/helmholtz.cpp:272-281)
        r = b.apply_S(res.x_S) - bS
        rel = float(torch.sqrt((r * r).sum() / (bS * bS).sum()))
        return Solve3dResult(u, list(res.iterations), list(res.converged), rel)
