"""Per-mode convergence of a 3D config on a mode subset: GMRES(m) with restarts
vs unrestarted GMRES (the reference never restarts)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--modes", default="0,1,2,3,4,6,8,12,16,24,32,64,128,255")
ap.add_argument("--max-iter", type=int, default=1000)
a = ap.parse_args()
cfg = CONFIGS[a.config]
modes = [int(m) for m in a.modes.split(",")]
t0 = time.time()
ps = build_problem(cfg, modes, device="cuda", device_rhs=True)
print(f"setup {time.time() - t0:.1f}s for {len(modes)} modes", flush=True)
b = load_batch(Context(0), ps).tune_from_env()
bS = torch.tensor(ps.b_S, device="cuda")
for restart in (cfg.max_iter, 0):
    t0 = time.time()
    r = b.solve(bS, "dbj", 1e-10, a.max_iter, restart, "cgs2", True, history=True)
    torch.cuda.synchronize()
    print(f"restart {restart}: {time.time() - t0:.2f}s", flush=True)
    for i, m in enumerate(modes):
        h = r.histories[i]
        print(f"  mode {m:4d} its {r.iterations[i]:5d} conv {int(r.converged[i])} final {r.final_rel_residual[i]:.2e} "
              f"hist[100] {h[min(100, len(h) - 1)]:.2e} hist[-1] {h[-1]:.2e}", flush=True)
