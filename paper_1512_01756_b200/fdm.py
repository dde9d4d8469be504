"""Product-side setup of the Schur systems by fast diagonalization.

The reference builds every strip-kind coupling G = Btrace A_kind^{-1} E_own
with a dense LU of A_kind (q = n^2 m_z) and, per Fourier wavenumber, with
real-Schur shifted solves (/root/reference/proj/src/schur.cpp:19-69,
proj/src/helmholtz.cpp:58-87).  On a uniform rectangular mesh each strip
block is an exact Kronecker sum

    A_kind = Ax_kind (x) I_z  +  I_x (x) Az          (index order (ez, ix, iz)),

Ax_kind (n x n) carrying the x-collocation, the west/east flux rows and the
Robin self-terms (proj/src/operator.cpp:37-48), Az (n m_z x n m_z) the
z-collocation and the vertical penalty coupling (proj/src/operator.cpp:49-72).
Diagonalising both factors gives, for any shift mu,

    G_kind[X,Y](mu) = Vz diag_q( -tau sum_p a^{XY}_p / (lx_p + lz_q - mu) ) Vz^{-1},

so every w x w block of every mode's coupling is one w^3 product instead of a
q^3 factorization.  The same structure yields the left null vector u_S of the
singular (mu = 0) system from one 2d x 2d singular vector, and the Schur
right-hand sides B (A - mu)^{-1} f.  The eigenvector matrices are
well-conditioned here (cond(Vx) ~ 5, cond(Vz) ~ 20-100), and the tests hold
these couplings to the oracle's LU / real-Schur ones.

This is setup (outside the timed hot path); it runs on the
GPU through torch when one is present, on the CPU otherwise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def gll_nodes(n: int):
    """GLL nodes/weights and barycentric differentiation matrix
    (/root/reference/proj/src/gll.cpp:10-97): Newton on P'_{n-1} from
    Chebyshev-Lobatto guesses, mirrored for symmetry, negative-sum diagonal."""
    if n < 2:
        raise ValueError("order must be at least 2")
    N = n - 1

    def leg(x):
        p0, d0, p1, d1 = 1.0, 0.0, x, 1.0
        if N == 0:
            return p0, d0
        for j in range(2, N + 1):
            p2 = ((2 * j - 1) * x * p1 - (j - 1) * p0) / j
            d2 = d0 + (2 * j - 1) * p1
            p0, p1, d0, d1 = p1, p2, d1, d2
        return p1, d1

    x = np.zeros(n)
    x[0], x[N] = -1.0, 1.0
    for i in range(1, (N - 1) // 2 + 1):
        g = -math.cos(math.pi * i / N)
        for _ in range(100):
            p, dp = leg(g)
            step = dp / ((2.0 * g * dp - N * (N + 1) * p) / (1.0 - g * g))
            g -= step
            if abs(step) <= 1e-14:
                break
        else:
            raise RuntimeError("GLL Newton iteration failed")
        x[i], x[N - i] = g, -g
    if N % 2 == 0 and N >= 2:
        x[N // 2] = 0.0
    wts = np.array([2.0 / (N * (N + 1) * leg(xi)[0] ** 2) for xi in x])
    lam = np.ones(n)
    for j in range(n):
        for m in range(n):
            if m != j:
                lam[j] /= x[j] - x[m]
    lam /= np.abs(lam).max()
    D = np.zeros((n, n))
    for i in range(n):
        s = 0.0
        for j in range(n):
            if j != i:
                D[i, j] = (lam[j] / lam[i]) / (x[i] - x[j])
                s += D[i, j]
        D[i, i] = -s
    return x, wts, D


@dataclass
class Geometry:
    n: int
    m_x: int
    m_z: int
    l_x: float
    l_z: float
    c_tau: float = 2.0

    @property
    def w(self):
        return self.n * self.m_z

    @property
    def d(self):
        return self.m_x - 1

    @property
    def k(self):
        return 2 * self.w * self.d

    @property
    def q(self):
        return self.n * self.n * self.m_z

    @property
    def r(self):
        return self.q * self.m_x

    @property
    def h_x(self):
        return self.l_x / self.m_x

    @property
    def h_z(self):
        return self.l_z / self.m_z

    @property
    def tau(self):  # proj/src/operator.cpp:78-82
        return self.c_tau * self.n * self.n / min(self.h_x, self.h_z)


class StripFDM:
    """Fast-diagonalization factors of the strip operator of one geometry."""

    def __init__(self, geo: Geometry, device: str | None = None):
        import torch

        self.torch = torch
        self.geo = geo
        if device is None:
            device = "cuda" if torch.cuda.is_available() else "cpu"
        self.device = device
        n, mz = geo.n, geo.m_z
        _, _, D = gll_nodes(n)
        self.D = D
        tau = geo.tau
        cx, cz = 2.0 / geo.h_x, 2.0 / geo.h_z
        self.cx, self.cz, self.tau = cx, cz, tau
        D2 = D @ D
        # ---- x factor per strip kind (west_iface, east_iface)
        self.kinds = {}
        for key in ((False, True), (True, True), (True, False)):
            Ax = cx * cx * D2
            Ax[0, :] += -tau * cx * D[0, :]
            Ax[n - 1, :] += tau * cx * D[n - 1, :]
            if key[0]:
                Ax[0, 0] += tau
            if key[1]:
                Ax[n - 1, n - 1] += tau
            lx, Vx = np.linalg.eig(Ax)
            Vxi = np.linalg.inv(Vx)
            tW = np.zeros(n)
            tW[0] = 1.0
            tW += cx * D[0, :]
            tE = np.zeros(n)
            tE[n - 1] = 1.0
            tE -= cx * D[n - 1, :]
            # a[X][Y][p] = (t_X . Vx[:, p]) * Vxi[p, y_Y]
            tv = {"W": tW @ Vx, "E": tE @ Vx}
            yv = {"W": Vxi[:, 0], "E": Vxi[:, n - 1]}
            a = {X + Y: tv[X] * yv[Y] for X in "WE" for Y in "WE"}
            self.kinds[key] = dict(Ax=Ax, lx=lx, Vx=Vx, Vxi=Vxi, a=a, tW=tW, tE=tE)
        # ---- z factor (shared by all kinds), index Z = ez*n + iz
        w = n * mz
        Az = np.zeros((w, w))
        for ez in range(mz):
            o = ez * n
            Az[o:o + n, o:o + n] += cz * cz * D2
            Az[o, o:o + n] += -tau * cz * D[0, :]
            if ez > 0:
                Az[o, o] += tau
                Az[o, o - 1] += -tau
                Az[o, o - n:o] += tau * cz * D[n - 1, :]
            Az[o + n - 1, o:o + n] += tau * cz * D[n - 1, :]
            if ez < mz - 1:
                Az[o + n - 1, o + n - 1] += tau
                Az[o + n - 1, o + n] += -tau
                Az[o + n - 1, o + n:o + 2 * n] += -tau * cz * D[0, :]
        self.Az = Az
        # Az commutes with the reflection z -> l_z - z (uniform elements, symmetric
        # GLL nodes, the same penalty at both ends), so its eigenvectors are even or
        # odd.  Diagonalising the even and the odd block separately makes every
        # eigenvector exactly parity-pure (a plain eig mixes the nearly degenerate
        # even/odd eigenvalue pairs, gaps ~1e-8) and lets the transform kernels run
        # two half-size contractions (csrc/xformp.cuh).
        hE, hO = (w + 1) // 2, w // 2
        Re, Ro = np.zeros((w, hE)), np.zeros((w, hO))
        for kk in range(hO):
            Re[kk, kk] = Re[w - 1 - kk, kk] = math.sqrt(0.5)
            Ro[kk, kk], Ro[w - 1 - kk, kk] = math.sqrt(0.5), -math.sqrt(0.5)
        if w % 2:
            Re[hO, hO] = 1.0
        le, Ve = np.linalg.eig(Re.T @ Az @ Re)
        lo, Vo = np.linalg.eig(Ro.T @ Az @ Ro)
        lz = np.concatenate([le, lo])
        Vz = np.concatenate([Re @ Ve, Ro @ Vo], axis=1)
        Vzi = np.concatenate([np.linalg.inv(Ve) @ Re.T, np.linalg.inv(Vo) @ Ro.T], axis=0)
        self.parity = np.concatenate([np.ones(hE, dtype=int), -np.ones(hO, dtype=int)])
        self.lz, self.Vz, self.Vzi = lz, Vz, Vzi
        self.cond = (max(np.linalg.cond(v["Vx"]) for v in self.kinds.values()), np.linalg.cond(Vz))
        t = torch
        self.tVz = t.tensor(Vz, dtype=t.complex128, device=device)
        self.tVzi = t.tensor(self.Vzi, dtype=t.complex128, device=device)
        self.tlz = t.tensor(lz, dtype=t.complex128, device=device)

    # ---- couplings ---------------------------------------------------------
    def gamma(self, key, XY, mus):
        """diag of G_kind[X,Y] in the z-eigenbasis, shape (len(mus), w)."""
        t = self.torch
        kd = self.kinds[key]
        a = t.tensor(kd["a"][XY], dtype=t.complex128, device=self.device)
        lx = t.tensor(kd["lx"], dtype=t.complex128, device=self.device)
        mu = t.as_tensor(np.asarray(mus, dtype=np.float64), device=self.device).to(t.complex128)
        den = lx[None, :, None] + self.tlz[None, None, :] - mu[:, None, None]  # (M, p, q)
        return -self.tau * (a[None, :, None] / den).sum(dim=1)

    def real_basis(self):
        """Real eigenbasis T of the z factor for the spectral operator form:
        complex-conjugate pairs first (columns Re v, Im v of the member with
        Im(lambda) > 0), then the real modes.  Returns (npairs, T, T^{-1},
        representative eigen-indices)."""
        if getattr(self, "_rb", None) is None:
            lz, Vz = self.lz, np.asarray(self.Vz)
            tol = 1e-9 * np.abs(lz).max()
            # even modes before odd ones inside the pairs and inside the real modes
            # (the order the parity-split transform kernels expect)
            order = sorted(range(len(lz)), key=lambda q: (-self.parity[q], q))
            pairs = [q for q in order if lz[q].imag > tol]
            reals = [q for q in order if abs(lz[q].imag) <= tol]
            if 2 * len(pairs) + len(reals) != len(lz):
                raise RuntimeError("z eigenvalues are not in conjugate pairs")
            cols = []
            for q in pairs:
                cols += [Vz[:, q].real, Vz[:, q].imag]
            for q in reals:
                cols.append(Vz[:, q].real)
            T = np.ascontiguousarray(np.stack(cols, 1))
            # T^{-1} from the complex left eigenvectors (rows of Vz^{-1}, exactly
            # parity-pure like the columns of T): for a pair v = a + i b with left
            # row l, the rows of T^{-1} for (a, b) are 2 Re l and -2 Im l
            Vzi = np.asarray(self.Vzi)
            rows = []
            for q in pairs:
                rows += [2.0 * Vzi[q].real, -2.0 * Vzi[q].imag]
            for q in reals:
                rows.append(Vzi[q].real)
            Ti = np.ascontiguousarray(np.stack(rows, 0))
            if np.abs(Ti @ T - np.eye(len(lz))).max() > 1e-8:
                Ti = np.linalg.inv(T)
            self._rb = (len(pairs), T, Ti, pairs + reals)
        return self._rb

    def spectral(self, mus):
        """(npairs, T, T^{-1}, gamma) for smpm_batch_set_spectral: gamma is
        (len(mus), 6, nmode) complex in kind order W_EE, I_WW, I_WE, I_EW,
        I_EE, E_WW at the representative eigen-indices (G = T diag T^{-1})."""
        npairs, T, Ti, rep = self.real_basis()
        mus = np.atleast_1d(np.asarray(mus, dtype=np.float64))
        out = np.empty((len(mus), 6, len(rep)), dtype=np.complex128)
        kinds = (((False, True), "EE"), ((True, True), "WW"), ((True, True), "WE"), ((True, True), "EW"),
                 ((True, True), "EE"), ((True, False), "WW"))
        for i, (key, XY) in enumerate(kinds):
            out[:, i, :] = self.gamma(key, XY, mus).cpu().numpy()[:, rep]
        return npairs, T, Ti, out

    def strip_factors(self, mus):
        """smpm_strip_factors of this geometry for shifts `mus`: x factors per strip
        kind (west-boundary, interior, east-boundary), z eigenvalues in the
        spectral basis order, trace weights, tau."""
        _, _, _, rep = self.real_basis()
        keys = ((False, True), (True, True), (True, False))
        kd = [self.kinds[k] for k in keys]
        return dict(Vx=[k["Vx"] for k in kd], Vx_inv=[k["Vxi"] for k in kd], lx=[k["lx"] for k in kd],
                    lz=np.asarray(self.lz)[rep], tW=self.kinds[(True, True)]["tW"],
                    tE=self.kinds[(True, True)]["tE"], tau=self.tau,
                    mu=np.atleast_1d(np.asarray(mus, dtype=np.float64)))

    def _block(self, gam):
        # Vz diag(gam) Vz^{-1} for a batch of diagonals -> real (M, w, w)
        t = self.torch
        out = t.matmul(self.tVz[None] * gam[:, None, :], self.tVzi[None])
        return out

    def couplings(self, mus, chunk: int = 16):
        """G_W (M,w,w), G_I (M,2w,2w), G_E (M,w,w) as float64 numpy (column-major
        semantics are the caller's: these are plain matrices)."""
        t = self.torch
        w = self.geo.w
        mus = np.atleast_1d(np.asarray(mus, dtype=np.float64))
        M = len(mus)
        GW = np.empty((M, w, w))
        GI = np.empty((M, 2 * w, 2 * w))
        GE = np.empty((M, w, w))
        self.max_imag = 0.0
        for c0 in range(0, M, chunk):
            mc = mus[c0:c0 + chunk]
            blk = {}
            for key, XYs in (((False, True), ["EE"]), ((True, True), ["WW", "WE", "EW", "EE"]), ((True, False), ["WW"])):
                for XY in XYs:
                    g = self._block(self.gamma(key, XY, mc))
                    self.max_imag = max(self.max_imag, float(g.imag.abs().max()))
                    blk[(key, XY)] = g.real.cpu().numpy()
            sl = slice(c0, c0 + len(mc))
            GW[sl] = blk[((False, True), "EE")]
            GE[sl] = blk[((True, False), "WW")]
            GI[sl, :w, :w] = blk[((True, True), "WW")]
            GI[sl, :w, w:] = blk[((True, True), "WE")]
            GI[sl, w:, :w] = blk[((True, True), "EW")]
            GI[sl, w:, w:] = blk[((True, True), "EE")]
        return GW, GI, GE

    # ---- strip solves (A - mu)^{-1} and B ----------------------------------
    def _kind_of(self, s):
        return (s > 0, s < self.geo.m_x - 1)

    def solve_A(self, f, mu=0.0, transpose=False):
        """(A - mu I)^{-1} f  (or A^{-T}) for a full-grid vector f (r,)."""
        g = self.geo
        n, mz, w = g.n, g.m_z, g.w
        F = np.asarray(f, dtype=np.float64).reshape(g.m_x, mz, n, n)  # (s, ez, ix, iz)
        out = np.empty_like(F)
        Vz, Vzi = (self.Vzi.T, self.Vz.T) if transpose else (self.Vz, self.Vzi)
        for s in range(g.m_x):
            kd = self.kinds[self._kind_of(s)]
            Vx, Vxi = (kd["Vxi"].T, kd["Vx"].T) if transpose else (kd["Vx"], kd["Vxi"])
            X = F[s].transpose(1, 0, 2).reshape(n, w)  # (ix, Z)
            T = Vxi @ X @ Vzi.T  # (p, q)
            T = T / (kd["lx"][:, None] + self.lz[None, :] - mu)
            Y = (Vx @ T @ Vz.T).real
            out[s] = Y.reshape(n, mz, n).transpose(1, 0, 2)
        return out.reshape(-1)

    def apply_B(self, u):
        """B u: neighbour traces -tau t_X . u (proj/src/operator.cpp:127-151)."""
        g = self.geo
        n, mz, w = g.n, g.m_z, g.w
        U = np.asarray(u, dtype=np.float64).reshape(g.m_x, mz, n, n)  # (s, ez, ix, iz)
        kd = self.kinds[(True, True)]
        tW, tE = kd["tW"], kd["tE"]
        b = np.empty((g.d, 2, w))
        for i in range(g.d):
            b[i, 0] = -self.tau * np.einsum("m,emz->ez", tW, U[i + 1]).reshape(w)
            b[i, 1] = -self.tau * np.einsum("m,emz->ez", tE, U[i]).reshape(w)
        return b.reshape(-1)

    def apply_Bt(self, v):
        g = self.geo
        n, mz, w = g.n, g.m_z, g.w
        V = np.asarray(v, dtype=np.float64).reshape(g.d, 2, mz, n)
        kd = self.kinds[(True, True)]
        tW, tE = kd["tW"], kd["tE"]
        U = np.zeros((g.m_x, mz, n, n))
        for i in range(g.d):
            U[i + 1] += -self.tau * np.einsum("m,ez->emz", tW, V[i, 0])
            U[i] += -self.tau * np.einsum("m,ez->emz", tE, V[i, 1])
        return U.reshape(-1)

    def schur_rhs(self, f, mu=0.0):
        """b_S = B (A - mu I)^{-1} f (proj/src/schur.cpp:182-186, proj/src/helmholtz.cpp:172-176)."""
        return self.apply_B(self.solve_A(f, mu))

    # ---- left null vectors of the mu = 0 system ----------------------------
    def nullspace(self):
        """u_S (left null vector of S) and u_L = normalize(A^{-T} B^T u_S),
        signs fixed as proj/src/nullspace.cpp:13-17."""
        g = self.geo
        d, w = g.d, g.w
        gam = {}
        for key, XYs in (((False, True), ["EE"]), ((True, True), ["WW", "WE", "EW", "EE"]), ((True, False), ["WW"])):
            for XY in XYs:
                gam[(key, XY)] = self.gamma(key, XY, [0.0])[0].cpu().numpy()
        q = int(np.argmin(np.abs(self.lz)))
        St = np.eye(2 * d, dtype=complex)
        # strip s reads blocks 2s-1 (W-own), 2s (E-own); writes 2s-2 (W-readers), 2s+1 (E-readers)
        for s in range(g.m_x):
            key = self._kind_of(s)
            for X, row in (("W", 2 * s - 2), ("E", 2 * s + 1)):
                if row < 0 or row >= 2 * d:
                    continue
                for Y, col in (("W", 2 * s - 1), ("E", 2 * s)):
                    if col < 0 or col >= 2 * d:
                        continue
                    St[row, col] += gam[(key, X + Y)][q]
        U_, sv, _ = np.linalg.svd(St)
        phi = U_[:, -1]
        uS = (phi[:, None] * self.Vzi[q][None, :]).reshape(-1)
        uS = uS * np.exp(-1j * np.angle(uS[np.argmax(np.abs(uS))]))
        uS = uS.real
        uS /= np.linalg.norm(uS)
        if uS[np.argmax(np.abs(uS))] < 0:
            uS = -uS
        uL = self.solve_A(self.apply_Bt(uS), 0.0, transpose=True)
        uL /= np.linalg.norm(uL)
        if uL[np.argmax(np.abs(uL))] < 0:
            uL = -uL
        self.null_sigma_ratio = sv[-1] / sv[-2]
        return uS, uL


def project_out(v, direction):
    """v - dir (dir . v) (proj/src/nullspace.cpp:92) — host helper for setup data."""
    return v - direction * float(direction @ v)
