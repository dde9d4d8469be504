"""The five BASELINE.json configurations, n = p + 1 GLL
points, c_tau = 2, seed 1234.  Domains [0,L] are evaluated at the reference's
centred coordinates shifted by (+l_x/2, +l_z/2)."""
from __future__ import annotations

import math
from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    m_x: int
    m_z: int
    l_x: float
    l_z: float
    kmax: int           # cosine modes k,l <= kmax in the seeded manufactured field
    decay: bool         # a_kl ~ N(0,1)/(1+k^2+l^2) when True
    max_iter: int       # GMRES(m): cycle length and iteration cap
    methods: tuple = ("dbj",)
    modes: int = 0      # Fourier modes (3D); 0 = 2D Poisson
    l_y: float = 0.0
    c_tau: float = 2.0
    seed: int = 1234

    @property
    def w(self):
        return self.n * self.m_z

    @property
    def d(self):
        return self.m_x - 1

    @property
    def k(self):
        return 2 * self.w * self.d

    def mus(self):
        """Helmholtz shifts k_j^2, k_j = 2 pi j / l_y (proj/src/helmholtz.cpp:126)."""
        if not self.modes:
            return [0.0]
        return [(2.0 * math.pi * j / self.l_y) ** 2 for j in range(self.modes)]


C1 = Config("C1", 9, 4, 4, 1.0, 1.0, 4, False, 50)
C2 = Config("C2", 13, 32, 32, 8.0, 1.0, 8, True, 50)
C3 = Config("C3", 17, 128, 16, 100.0, 1.0, 8, True, 100, methods=("dbj", "2las"))
C4 = Config("C4", 11, 64, 16, 16.0, 1.0, 8, True, 100, modes=128, l_y=16.0)
# BASELINE gives no L_y for C5; L_y = l_x = 64 as in C4
C5 = Config("C5", 17, 256, 32, 64.0, 1.0, 16, True, 100, modes=256, l_y=64.0)

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
