"""Generates tests/golden/*.npz from the CPU oracle (the restatement of the
reference) — small fixtures that pin the oracle (regression) and serve as
GPU parity targets on the box, where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def rng_streams():
    # uniforms of Rng(1234).stream(t), t = 0..3, and of the null-space start
    # Rng(0x5eed0001) (proj/include/smpm/rng.hpp, proj/src/nullspace.cpp:28-31),
    # drawn by the oracle's C++ std::mt19937_64 engine
    out = {f"uniform_{t}": O.rng_uniforms(1234, t, 8) for t in range(4)}
    out["nullspace_start"] = O.rng_uniforms(0x5EED0001, -1, 8) - 0.5
    return out


def c1_case():
    # C1: n=9, 4x4, unit square, a_kl ~ N(0,1), k,l <= 4, dbj GMRES(50)
    setup = O.build_poisson_setup(9, 4, 4, 1.0, 1.0, 2.0)
    f, u = setup.prob.manufactured(4, False, 1234, 0)
    out = O.solve_poisson(setup, f, "dbj", 1e-10, 50, 50)
    gw, gi, ge = setup.sys.kinds()
    r = out["res"]
    return dict(f=f, u_exact=u, b_S=out["b_S"], x_S=r.x_S, u=out["u"], history=r.history,
                iterations=np.array(r.iterations), G_W=gw, G_I=gi, G_E=ge, u_S=setup.u_S, u_L=setup.u_L)


def helmholtz_case():
    # 3 Fourier modes of a small grid (mode 0 singular), manufactured per-mode RHS
    prob = O.Problem(7, 6, 4, 6.0, 1.0, 2.0)
    mus = [0.0, (2 * np.pi / 6.0) ** 2, (2 * np.pi * 5 / 6.0) ** 2]
    d = {}
    for j, mu in enumerate(mus):
        s = O.System(prob, mu, False)
        s.build_bj()
        f, _ = prob.manufactured(4, True, 1234, j, mu=mu)
        if mu == 0.0:
            u_S, u_L, _, _ = s.nullspace()
            s.build_coarse(u_S)
            b = O.project_out(s.schur_rhs(O.project_out(f, u_L)), u_S)
            d["u_S"] = u_S
        else:
            s.build_coarse(None)
            b = prob.apply_B(prob.shifted_solve(mu, f))
        r = s.solve(b, "dbj", 1e-10, 100, 100)
        gw, gi, ge = s.kinds()
        d[f"G_W_{j}"], d[f"G_I_{j}"], d[f"G_E_{j}"] = gw, gi, ge
        d[f"b_S_{j}"], d[f"x_S_{j}"] = b, r.x_S
        d[f"iterations_{j}"] = np.array(r.iterations)
        d[f"history_{j}"] = r.history
    d["mus"] = np.array(mus)
    return d


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng_streams())
    np.savez_compressed(os.path.join(HERE, "c1_dbj.npz"), **c1_case())
    np.savez_compressed(os.path.join(HERE, "helmholtz3.npz"), **helmholtz_case())
    print("written", sorted(os.listdir(HERE)))
