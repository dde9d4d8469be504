"""Early epilogue check: device solve and end-to-end solve_host of C4 with and
without SMPM_NO_EARLY (x_S bit-compared, times per solve)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

cfg = CONFIGS[os.environ.get("SWEEP_CONFIG", "C4")]
ps = build_problem(cfg, device="cuda")
ctx = Context(0)
bS = torch.tensor(ps.b_S, device="cuda")
hb = torch.tensor(ps.b_S).pin_memory()
hx = torch.empty_like(hb).pin_memory()
out = {}
for setting in ["", "SMPM_EARLY=0"]:
    os.environ.pop("SMPM_EARLY", None)
    if setting:
        os.environ["SMPM_EARLY"] = "0"
    b = load_batch(ctx, ps).tune_from_env()
    args = ("dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True)
    for _ in range(3):
        r = b.solve(bS, *args, history=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = b.solve(bS, *args, history=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    xd = r.x_S.cpu().numpy().copy()
    th = []
    for _ in range(10):
        t0 = time.perf_counter()
        b.solve_host(hb.numpy(), *args, out=hx.numpy())
        th.append((time.perf_counter() - t0) * 1e3)
    xh = hx.numpy().copy()
    out[setting or "default"] = (xd, xh)
    print(f"{setting or 'default':20s} device {np.median(ts):.3f} ms  host e2e {np.median(th):.3f} ms  "
          f"host==device {np.array_equal(xd, xh)}", flush=True)
a, c = out["default"], out["SMPM_EARLY=0"]
print("early vs no-early: device bit-equal", np.array_equal(a[0], c[0]), "max abs diff", float(np.abs(a[0] - c[0]).max()))
