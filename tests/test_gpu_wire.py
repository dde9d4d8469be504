"""The reference's wire format for Schur systems (dump_schur_blocks / read_schur_blocks,
/root/reference/proj/src/schur.cpp:246-297) through smpm_batch_load_schur_blocks: the
oracle's reference-layout system dumped by the restated writer, imported (verified and
deduplicated into the strip-kind couplings), then apply_S and a deflated solve against
the oracle; malformed files are rejected with SMPM_EINVAL."""
import numpy as np
import pytest

from oracle import oracle as O
from tests._cases import rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mu", [0.0, (2 * np.pi) ** 2])
def test_load_dumped_blocks(ctx, tmp_path, mu):
    import torch

    from paper_1512_01756_b200 import SchurBatch

    prob = O.Problem(9, 4, 4, 1.0, 1.0, 2.0)
    s = O.System(prob, mu, True)  # reference per-interface layout
    s.build_bj()
    f, _ = prob.manufactured(4, False, 1234, 0, mu=mu)
    if mu == 0.0:
        u_S, u_L, _, _ = s.nullspace()
        s.build_coarse(u_S)
        bS = O.project_out(s.schur_rhs(O.project_out(f, u_L)), u_S)
    else:
        s.build_coarse(None)
        bS = prob.apply_B(prob.shifted_solve(mu, f))
    path = tmp_path / "schur.bin"
    s.dump_blocks(path)
    b = SchurBatch(ctx, 9, 4, 4, 1)
    b.load_schur_blocks(0, path)
    if mu == 0.0:
        b.set_nullspace(0, u_S)
    b.finalize()
    v = np.random.default_rng(2).standard_normal(s.k)
    Sv = b.apply_S(torch.tensor(v[None], device="cuda"))[0].cpu().numpy()
    assert rel(Sv, s.apply_S(v)) < 1e-13
    res = b.solve(torch.tensor(bS[None], device="cuda"), "dbj", 1e-10, 50, 50)
    ref = s.solve(bS, "dbj", 1e-10, 50, 50)
    assert abs(res.iterations[0] - ref.iterations) <= 1
    x, xr = res.x_S[0].cpu().numpy(), ref.x_S
    if mu == 0.0:
        x, xr = x - x.mean(), xr - xr.mean()
    assert rel(x, xr) < 1e-10


def test_malformed_files_rejected(ctx, tmp_path):
    from paper_1512_01756_b200 import SchurBatch, SmpmError

    prob = O.Problem(9, 4, 4, 1.0, 1.0, 2.0)
    s = O.System(prob, 0.0, True)
    path = tmp_path / "schur.bin"
    s.dump_blocks(path)
    raw = path.read_bytes()
    (tmp_path / "short.bin").write_bytes(raw[: len(raw) // 2])
    b = SchurBatch(ctx, 9, 4, 4, 1)
    with pytest.raises(SmpmError):
        b.load_schur_blocks(0, tmp_path / "short.bin")
    other = SchurBatch(ctx, 9, 5, 4, 1)  # geometry mismatch
    with pytest.raises(SmpmError):
        other.load_schur_blocks(0, path)
    with pytest.raises(SmpmError):
        b.load_schur_blocks(0, tmp_path / "missing.bin")
