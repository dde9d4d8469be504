"""Device time of the 3D-extension steps at C4-3D size (m_y = 256, 256 systems):
transverse FFT / inverse (HBM roofline: 2 x r x m_y x 8 bytes), schur_rhs and
recover_solution (strip solves), with CUDA events, warm."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.solve3d import Fourier3D, fourier_y, inverse_fourier_y  # noqa: E402


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cfg = CONFIGS["C4"]
m_y = 2 * cfg.modes
s = Fourier3D(Context(0), cfg.n, cfg.m_x, cfg.m_z, cfg.l_x, cfg.l_z, m_y, cfg.l_y)
b = s.batch
r = b.r
f = torch.randn(m_y, r, dtype=torch.float64, device="cuda")
c = fourier_y(f, m_y)
x = torch.randn(b.nsys, b.k, dtype=torch.float64, device="cuda")
try:
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    hbm = 6539.2
out = {}
for name, fn, by in (("fourier_y", lambda: fourier_y(f, m_y), 2 * m_y * r * 8),
                     ("inverse_fourier_y", lambda: inverse_fourier_y(c, m_y), 2 * m_y * r * 8),
                     ("schur_rhs", lambda: b.schur_rhs(c), None),
                     ("recover_solution", lambda: b.recover_solution(c, x), None)):
    ms = t(fn)
    row = {"ms": ms}
    if by:
        row["gbs"] = by / (ms * 1e-3) / 1e9
        row["frac_hbm"] = row["gbs"] / hbm
    out[name] = row
    print(name, json.dumps(row), flush=True)
