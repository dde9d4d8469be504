"""Seeded synthetic inputs for the BASELINE configurations and the product
setup that turns them into Schur systems (couplings, null vectors, b_S).

Inputs follow SURVEY.md §8(d): seed 1234, per-trial / per-mode streams of the
reference RNG (splitmix64-scrambled mt19937_64, 53-bit uniforms,
/root/reference/proj/include/smpm/rng.hpp:11-32), N(0,1) by Box-Muller on two
consecutive uniforms (cosine branch), cosine modes evaluated at the
reference's centred node coordinates shifted by (+l_x/2, +l_z/2).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .configs import Config
from .fdm import Geometry, StripFDM, gll_nodes, project_out

_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (standard-defined, so bit-identical to the C++ engine)."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _M64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt, self.i = mt, 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= 312:
            self._twist()
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64


class Rng:
    """proj/include/smpm/rng.hpp:11-32."""

    def __init__(self, seed: int):
        self.seed = seed & _M64
        self.eng = MT19937_64(self._mix(self.seed))

    @staticmethod
    def _mix(x):
        x = (x + 0x9E3779B97F4A7C15) & _M64
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
        return x ^ (x >> 31)

    def uniform(self) -> float:
        return float(self.eng() >> 11) * 2.0 ** -53

    def stream(self, i: int) -> "Rng":
        return Rng((self.seed + 0x9E3779B97F4A7C15 * (i + 1)) & _M64)

    def normal(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(1.0 - u1)) * math.cos(2.0 * math.pi * u2)


def node_coords(geo: Geometry):
    """Node coordinates in the reference numbering g = ((ex*m_z+ez)*n+ix)*n+iz,
    shifted to [0, l_x] x [0, l_z] (proj/src/mesh.cpp:27-40 + l/2)."""
    xi, _, _ = gll_nodes(geo.n)
    n, mx, mz = geo.n, geo.m_x, geo.m_z
    ex = np.arange(mx)[:, None, None, None]
    ez = np.arange(mz)[None, :, None, None]
    ix = np.arange(n)[None, None, :, None]
    iz = np.arange(n)[None, None, None, :]
    x = -0.5 * geo.l_x + ex * geo.h_x + 0.5 * (xi[ix] + 1.0) * geo.h_x + 0.5 * geo.l_x
    z = -0.5 * geo.l_z + ez * geo.h_z + 0.5 * (xi[iz] + 1.0) * geo.h_z + 0.5 * geo.l_z
    shape = (mx, mz, n, n)
    return np.broadcast_to(x, shape).reshape(-1), np.broadcast_to(z, shape).reshape(-1)


def manufactured(geo: Geometry, kmax: int, decay: bool, seed: int = 1234, stream: int = 0,
                 forcing_only: bool = False, mu: float = 0.0):
    """u = sum a_kl cos(k pi x/l_x) cos(l pi z/l_z); returns (f, u) with
    f = (Lap - mu) u (g = 0 exactly; mu = k_y^2 gives the manufactured per-mode
    Helmholtz right-hand side) or f = the series itself when forcing_only."""
    rng = Rng(seed).stream(stream)
    a = np.zeros((kmax + 1, kmax + 1))
    for k in range(kmax + 1):
        for l in range(kmax + 1):
            c = rng.normal()
            if decay:
                c /= 1.0 + k * k + l * l
            a[k, l] = c
    x, z = node_coords(geo)
    kk = np.arange(kmax + 1) * math.pi / geo.l_x
    ll = np.arange(kmax + 1) * math.pi / geo.l_z
    cx = np.cos(np.outer(x, kk))  # (r, K)
    cz = np.cos(np.outer(z, ll))
    u = np.einsum("rk,kl,rl->r", cx, a, cz)
    if forcing_only:
        return u.copy(), u
    lap = -(kk[:, None] ** 2 + ll[None, :] ** 2 + mu) * a
    f = np.einsum("rk,kl,rl->r", cx, lap, cz)
    return f, u


def manufactured_batch(geo: Geometry, kmax: int, decay: bool, seed: int, streams, mus, device):
    """f = (Lap - mu) u of `manufactured` for several (stream, mu) at once, on
    `device` (torch, nsys x r): the same seeded coefficients and formula."""
    import torch

    x, z = node_coords(geo)
    kk = np.arange(kmax + 1) * math.pi / geo.l_x
    ll = np.arange(kmax + 1) * math.pi / geo.l_z
    cx = torch.cos(torch.outer(torch.tensor(x, device=device), torch.tensor(kk, device=device)))  # (r, K)
    cz = torch.cos(torch.outer(torch.tensor(z, device=device), torch.tensor(ll, device=device)))
    out = torch.empty((len(streams), x.size), dtype=torch.float64, device=device)
    for i, (st, mu) in enumerate(zip(streams, mus)):
        rng = Rng(seed).stream(st)
        a = np.zeros((kmax + 1, kmax + 1))
        for k in range(kmax + 1):
            for l in range(kmax + 1):
                c = rng.normal()
                if decay:
                    c /= 1.0 + k * k + l * l
                a[k, l] = c
        lap = -(kk[:, None] ** 2 + ll[None, :] ** 2 + mu) * a
        out[i] = ((cx @ torch.tensor(lap, device=device)) * cz).sum(dim=1)
    return out


@dataclass
class ProblemSet:
    """Everything a SchurBatch needs for a set of systems of one config."""
    cfg: Config
    modes: list
    mus: list
    GW: np.ndarray
    GI: np.ndarray
    GE: np.ndarray
    u_S: np.ndarray | None
    u_L: np.ndarray | None
    b_S: np.ndarray  # (nsys, k); None until load_batch computes it on the device (device_rhs)
    fdm: StripFDM
    f: object = None  # device_rhs: torch (nsys, r) forcing (mode 0 projected with u_L in load_batch)

    def kinds(self, i):
        """(G_W, G_I, G_E) of system i: the stored dense couplings, or (device_setup
        problems, which never build them) the host/torch FDM product for that system."""
        if self.GW is not None:
            return self.GW[i], self.GI[i], self.GE[i]
        gw, gi, ge = self.fdm.couplings([self.mus[i]])
        return gw[0], gi[0], ge[0]


def build_problem(cfg: Config, modes=None, device=None, device_rhs=False, device_setup=False) -> ProblemSet:
    """Product setup for `modes` of a 3D config (all modes by default) or the
    single system of a 2D config.  device_rhs: the seeded forcings are built on
    the device and b_S = B (A - mu)^{-1} f is left to load_batch, which runs it
    through the C ABI's schur_rhs (strip.cuh) instead of the host FDM.
    device_setup: no dense couplings are built here; load_batch hands the
    geometry-level factors to smpm_batch_set_fdm and the library builds every
    system's couplings, block inverses and coarse data with its own kernels."""
    geo = Geometry(cfg.n, cfg.m_x, cfg.m_z, cfg.l_x, cfg.l_z, cfg.c_tau)
    F = StripFDM(geo, device)
    mus_all = cfg.mus()
    if modes is None:
        modes = list(range(len(mus_all)))
    mus = [mus_all[m] for m in modes]
    if device_setup and geo.w % 16 == 0:
        GW = GI = GE = None
    else:
        GW, GI, GE = F.couplings(mus)
    u_S = u_L = None
    if any(mu == 0.0 for mu in mus):
        u_S, u_L = F.nullspace()
    if device_rhs:
        import torch

        # the mode-0 u_L projection of f runs in load_batch (smpm_project_out)
        f = manufactured_batch(geo, cfg.kmax, cfg.decay, cfg.seed, modes, mus, device)
        return ProblemSet(cfg, list(modes), mus, GW, GI, GE, u_S, u_L, None, F, f)
    bs = []
    for m, mu in zip(modes, mus):
        f, _ = manufactured(geo, cfg.kmax, cfg.decay, cfg.seed, m, mu=mu)
        if mu == 0.0:
            f = project_out(f, u_L)
            b = project_out(F.schur_rhs(f, 0.0), u_S)
        else:
            b = F.schur_rhs(f, mu)
        bs.append(b)
    return ProblemSet(cfg, list(modes), mus, GW, GI, GE, u_S, u_L, np.array(bs), F)


def load_batch(ctx, ps: ProblemSet, spectral: bool = True):
    """SchurBatch with the couplings / null vector of a ProblemSet (and, by
    default, the spectral factors of the couplings)."""
    from .schur import SchurBatch

    cfg = ps.cfg
    b = SchurBatch(ctx, cfg.n, cfg.m_x, cfg.m_z, len(ps.modes))
    if ps.GW is None:
        # device-side setup: geometry-level factors only (smpm_batch_set_fdm)
        npairs, T, Ti, _ = ps.fdm.real_basis()
        b.set_fdm(npairs, T, Ti, ps.fdm.strip_factors(ps.mus))
        for i in range(len(ps.modes)):
            if ps.mus[i] == 0.0:
                b.set_nullspace(i, ps.u_S)
        b.finalize()
    else:
        for i in range(len(ps.modes)):
            b.set_couplings(i, ps.GW[i], ps.GI[i] if cfg.m_x > 2 else None, ps.GE[i])
            if ps.mus[i] == 0.0:
                b.set_nullspace(i, ps.u_S)
        if spectral:
            npairs, T, Ti, gam = ps.fdm.spectral(ps.mus)
            b.set_spectral(npairs, T, Ti, gam)
        b.finalize()
        if spectral and b.m_x >= 3 and 4 <= b.n <= 17:
            b.set_strip_factors(ps.fdm.strip_factors(ps.mus))
    if ps.b_S is None:
        # device b_S = B (A - mu)^{-1} f, then the mode-0 projection with u_S
        # (proj/src/helmholtz.cpp:159-176)
        import torch

        f = ps.f
        if ps.u_L is not None:
            sing = torch.tensor([mu == 0.0 for mu in ps.mus], device=f.device)
            uL = torch.tensor(ps.u_L, device=f.device)
            dl = torch.where(sing[:, None], uL[None, :], torch.zeros_like(uL)[None, :]).contiguous()
            f = b.project_out(f, dl)
            ps.f = f
        bS = b.schur_rhs(f)
        if ps.u_S is not None:
            sing = torch.tensor([mu == 0.0 for mu in ps.mus], device=bS.device)
            uS = torch.tensor(ps.u_S, device=bS.device)
            dirs = torch.where(sing[:, None], uS[None, :], torch.zeros_like(uS)[None, :]).contiguous()
            bS = b.project_out(bS, dirs)
        torch.cuda.synchronize()
        ps.b_S = bS.cpu().numpy()
    return b
