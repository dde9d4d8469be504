"""The reference-shaped C++ API (include/smpm_b200.hpp) compiled by the host
compiler against the C ABI library and run on the GPU."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1512_01756_b200", "lib")


def _compile(out):
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "shim_solve.cpp"), "-o", out, "-L", LIBDIR, "-lsmpm_b200",
           f"-Wl,-rpath,{LIBDIR}", "-L", "/usr/local/cuda/lib64", "-lcudart"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_shim_compiles(tmp_path):
    _compile(str(tmp_path / "shim_solve"))


@pytest.mark.gpu
def test_shim_solve_matches_golden(tmp_path):
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_dbj.npz"))
    for name in ("G_W", "G_I", "G_E"):
        np.asfortranarray(g[name]).ravel(order="F").tofile(tmp_path / f"{name}.bin")
    g["u_S"].tofile(tmp_path / "u_S.bin")
    g["b_S"].tofile(tmp_path / "b_S.bin")
    exe = str(tmp_path / "shim_solve")
    _compile(exe)
    out = subprocess.run([exe, str(tmp_path), "9", "4", "4"], check=True, capture_output=True, text=True).stdout.split()
    its, conv = int(out[0]), int(out[1])
    assert abs(its - int(g["iterations"])) <= 1 and conv == 1
    x = np.fromfile(tmp_path / "x_S.bin")
    xr = g["x_S"]
    assert np.linalg.norm((x - x.mean()) - (xr - xr.mean())) / np.linalg.norm(xr - xr.mean()) < 1e-10
