"""B200-native (sm_100a, fp64) deflated block-Jacobi Schur-GMRES for the SMPM
Poisson-Neumann / per-Fourier-mode Helmholtz problems (arXiv:1512.01756 path).

The compute path lives in ``lib/libsmpm_b200.so`` (C ABI: include/smpm_b200.h).
"""
from ._lib import SmpmError, lib  # noqa: F401
from .schur import Context, SchurBatch, SolveResult  # noqa: F401
from .fdm import Geometry, StripFDM, gll_nodes, project_out  # noqa: F401
