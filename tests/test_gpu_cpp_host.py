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


def build_demo(name="host_api_demo"):
    from paper_2402_10488_b200 import build
    build.build()
    exe = os.path.join(ROOT, "paper_2402_10488_b200", "_build", name)
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    lib_dir = os.path.join(ROOT, "paper_2402_10488_b200")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                           src, "-o", exe, "-L" + lib_dir, "-lrte_b200", "-Xlinker", "-rpath=" + lib_dir])
    return exe


def test_cpp_host_api_compiles():
    assert os.path.exists(build_demo())
    assert os.path.exists(build_demo("rom_pipeline_demo"))


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


@pytest.mark.gpu
def test_cpp_rom_pipeline_matches_the_python_mirror():
    """The C++ wrapper's offline stage (collect_snapshots, snapshot_matrix,
    pod, build_reduced_model) and ROMSAD solve (tests/cpp/rom_pipeline_demo.cpp)
    reproduce the Python host mirror's pipeline on the same inputs: same POD
    spectrum, iteration counts, correction logs and switch iterations, and
    the oracle's ROMSAD with the same reduced model."""
    from paper_2402_10488_b200 import rte
    exe = build_demo("rom_pipeline_demo")
    r = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)

    def problem(mod):
        t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.2, scattering_weight=lambda x, y: 0.5)
        t1 = mod.CoefficientTerm(psi=lambda mu: mu[0], scattering_weight=lambda x, y: 0.3)
        return mod.ProblemDefinition(mod.SLAB1D, [t0, t1], lambda x, y: 1.0, inflow_left=0.3, n_params=1,
                                     param_ranges=[(0.0, 1.0)])
    mesh = rte.Mesh.slab_uniform(0.0, 1.0, 64)
    quad = rte.gauss_legendre(8)
    tb = rte.TransportBatch(problem(rte), mesh, quad, [[m] for m in (0.1, 0.3, 0.5, 0.7, 0.9)])
    snaps = rte.collect_snapshots(tb, 3, 1e-10)
    F = rte.snapshot_matrix(tb, snaps, "correction")
    U, sv = rte.pod(F, 4)
    assert F.shape[0] == r["n_cols"]
    np.testing.assert_allclose(sv, r["sigma"], rtol=1e-12, atol=1e-14 * sv[0])
    eps_pod = float(np.sum(sv[4:]) / np.sum(sv))
    model = rte.build_reduced_model(tb, U, sv, eps_pod, 1e-10, "c")
    test = [[0.2], [0.45], [0.8]]
    b = rte.TransportBatch(problem(rte), mesh, quad, test)
    rte.load_rom(b, 1, model)
    cfg = rte.SolveConfig(eps_sisa=1e-10, theta=3, eps_romsad=rte.romsad_tolerance(1e-10, eps_pod))
    rho, reps = rte.sisa_solve(b, "ROMSAD", cfg)
    rho = rho.cpu().numpy()
    om = ro.Mesh.slab_uniform(0.0, 1.0, 64)
    ocm = ro.ReducedModel(0, 8, b.n_dof(), 4, 2, "c", eps_pod, 1e-10, model.u_rho, model.u_iso, model.a_r,
                          model.singular_values, model.discarded_fraction, model.b_r)
    for s, (c, p) in enumerate(zip(r["samples"], reps)):
        assert c["converged"] == 1 and c["iterations"] == p.iterations and c["log"] == p.correction_log
        assert c["switch_iter"] == p.switch_iter
        assert rel_l2(np.array(c["rho"]), rho[s]) < 1e-12
        o = ro.TransportSystem(problem(ro), om, ro.build_dg_space(om), ro.gauss_legendre(8), test[s])
        o_rho, o_rep = ro.sisa_solve(o, ro.RomsadStrategy(ocm, ro.build_dsa(o), 3, cfg.eps_romsad),
                                     ro.SolveConfig(eps_sisa=1e-10))
        assert o_rep.iterations == p.iterations and o_rep.correction_log == p.correction_log
        assert rel_l2(rho[s], o_rho) < 1e-8
    assert r["zero_strategy_equals_si"] and r["si_iterations"] > 1  # the C++ CorrectionStrategy plugin point


def test_cpp_pin_cell_compiles():
    assert os.path.exists(build_demo("pin_cell_demo"))


@pytest.mark.gpu
def test_cpp_problem_setup_c4_pin_cell(tmp_path):
    """BASELINE configs[3] (C4, 128^2 pin cell, CL(16,8), all 64 test samples)
    set up in C++ from a ProblemDefinition (tests/cpp/pin_cell_demo.cpp:
    closures, psi, weighted_mass, project, build_masses combination) and
    solved with SI-DSA: bitwise equal to the Python host mirror's solve of the
    same parameters, identical iteration counts / logs to the oracle
    (SuperLU DSA) on the first and last sample with flux within 1e-8; then the
    offline stage and ROMSAD run in C++ reproduce the Python mirror's
    iteration counts, logs and switch iterations with fluxes to 1e-12."""
    from paper_2402_10488_b200 import configs, rte
    from tests.tools import parity_workers as pw
    exe = build_demo("pin_cell_demo")
    out = tmp_path / "rho.bin"
    eps = 1e-8
    r = json.loads(subprocess.run([exe, "128", "64", repr(eps), str(out), "0", "40"], capture_output=True, text=True,
                                  check=True).stdout)
    mus = [s["mu"] for s in r["samples"]]
    assert len(mus) == 64 and r["k_terms"] == 5
    rho_cpp = np.fromfile(str(out)).reshape(64, -1)
    _, test = configs.c4_params(40, 64)
    np.testing.assert_allclose(np.array(mus), np.array(test), rtol=1e-15, atol=0)
    mesh = rte.Mesh.rect_uniform(0, 1, 128, 0, 1, 128)
    b = rte.TransportBatch(configs.pin_cell(rte)(128), mesh, rte.chebyshev_legendre(16, 8), mus)
    rho_py, reps = rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=eps, norm="abs", max_iters=500))
    rho_py = rho_py.cpu().numpy()
    for s, (c, p) in enumerate(zip(r["samples"], reps)):
        assert c["converged"] == 1 and c["iterations"] == p.iterations and c["log"] == p.correction_log, s
    assert np.array_equal(rho_cpp, rho_py)
    for s in (0, 63):
        o = pw.solve_sample(("c4", mus[s], ["DSA"], eps, "abs", 3, 0.0, None, None, True))["DSA"]
        assert r["samples"][s]["iterations"] == o["iterations"] and r["samples"][s]["log"] == o["log"]
        assert rel_l2(rho_cpp[s], o["rho"]) < 1e-8
    # the offline stage (40 training samples, correction POD rank 20) and ROMSAD(theta = 5) in C++ against the
    # Python mirror's same pipeline
    train, _ = configs.c4_params(40, 64)
    tb = rte.TransportBatch(configs.pin_cell(rte)(128), mesh, rte.chebyshev_legendre(16, 8), train)
    snaps = rte.collect_snapshots(tb, 3, 1e-8)
    U, sv = rte.pod(rte.snapshot_matrix(tb, snaps, "correction"), 20)
    cm = rte.build_reduced_model(tb, U, sv, float(np.sum(sv[20:]) / np.sum(sv)), 1e-8, "c")
    assert r["pod_cols"] == len(sv)
    np.testing.assert_allclose(r["discarded_fraction"], cm.discarded_fraction, rtol=1e-12)
    rte.load_rom(b, 1, cm)
    cfg = rte.SolveConfig(eps_sisa=eps, norm="abs", theta=5, max_iters=500,
                          eps_romsad=rte.romsad_tolerance(1e-8, cm.discarded_fraction))
    rho_r, reps_r = rte.sisa_solve(b, "ROMSAD", cfg)
    rho_r = rho_r.cpu().numpy()
    rho_rc = np.fromfile(str(out) + ".romsad").reshape(64, -1)
    for s, (c, p) in enumerate(zip(r["romsad"], reps_r)):
        assert (c["converged"], c["iterations"], c["switch_iter"], c["log"]) == \
            (int(p.converged), p.iterations, p.switch_iter, p.correction_log), s
    assert max(rel_l2(rho_rc[s], rho_r[s]) for s in range(64)) < 1e-12
