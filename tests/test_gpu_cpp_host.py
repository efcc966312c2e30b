"""The C++ host API (include/rte_b200.hpp) end to end: compile
tests/cpp/host_api_demo.cpp against librte_b200.so, run the C1 config
(BASELINE configs[0]) with SI-DSA and compare with the oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import homog, rel_l2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_demo():
    from paper_2402_10488_b200 import build
    build.build()
    exe = os.path.join(ROOT, "paper_2402_10488_b200", "_build", "host_api_demo")
    src = os.path.join(ROOT, "tests", "cpp", "host_api_demo.cpp")
    lib_dir = os.path.join(ROOT, "paper_2402_10488_b200")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                           src, "-o", exe, "-L" + lib_dir, "-lrte_b200", "-Xlinker", "-rpath=" + lib_dir])
    return exe


def test_cpp_host_api_compiles():
    assert os.path.exists(build_demo())


@pytest.mark.gpu
def test_cpp_host_api_c1_parity():
    exe = build_demo()
    out = subprocess.run([exe, "1e-10"], capture_output=True, text=True, check=True).stdout
    r = json.loads(out)
    mesh = ro.Mesh.slab_uniform(0.0, 1.0, 256)
    sys_ = ro.TransportSystem(homog(ro, ro.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0), mesh,
                              ro.build_dg_space(mesh), ro.gauss_legendre(16), [])
    rho, rep = ro.sisa_solve(sys_, ro.DsaStrategy(ro.build_dsa(sys_)), ro.SolveConfig(eps_sisa=1e-10))
    assert r["converged"] == 1 and r["iterations"] == rep.iterations and r["n_sweep"] == rep.n_sweep
    assert r["log"] == rep.correction_log
    assert rel_l2(np.array(r["rho"]), rho) < 1e-8
    grho, grep_ = ro.gmres_solve(sys_, ro.build_dsa(sys_), ro.SolveConfig(gmres_rel_tol=1e-11))
    assert r["pgmres_converged"] == 1 and r["pgmres_iterations"] == grep_.iterations
    assert r["pgmres_n_sweep"] == grep_.n_sweep
    assert rel_l2(np.array(r["pgmres_rho"]), grho) < 1e-8
