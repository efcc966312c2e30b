"""Committed golden fixtures (tests/golden/, made by tests/tools/make_golden.py
from the oracle): the oracle must keep reproducing them (CPU), and the B200
path must match them within the north_star tolerances (GPU)."""
import os

import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import homog, prob2d_const, rel_l2, two_region_slab

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def c1_sys(mod):
    mesh = mod.Mesh.slab_uniform(0.0, 1.0, 256)
    return mesh, homog(mod, mod.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0)


def box_problem(mod):
    return prob2d_const(mod, 0.4, 0.8, lambda x, y: 1.0 + x + 0.5 * y, inflow_left=1.0, inflow_bottom=0.7,
                        inflow_right=0.2, inflow_top=0.3)


def test_oracle_reproduces_golden():
    g = load("c1_slab_si_dsa.npz")
    mesh, p = c1_sys(ro)
    s = ro.TransportSystem(p, mesh, ro.build_dg_space(mesh), ro.gauss_legendre(16), [])
    assert rel_l2(s.apply_L(g["probe"]), g["L_probe"]) < 1e-13
    assert rel_l2(s.assemble_rhs(), g["bbar"]) < 1e-13
    rho, rep = ro.sisa_solve(s, ro.DsaStrategy(ro.build_dsa(s)), ro.SolveConfig(eps_sisa=1e-10))
    assert rep.iterations == int(g["iterations"]) and rel_l2(rho, g["rho"]) < 1e-12
    g2 = load("box2d_inflow.npz")
    mesh = ro.Mesh.rect_uniform(0.0, 1.2, 9, -0.5, 1.0, 7)
    s2 = ro.TransportSystem(box_problem(ro), mesh, ro.build_dg_space(mesh), ro.chebyshev_legendre(8, 4), [])
    assert rel_l2(s2.apply_L(g2["probe"]), g2["L_probe"]) < 1e-13
    assert rel_l2(s2.sweep_direction(0, g2["probe"]), g2["f0"]) < 1e-13


@pytest.mark.gpu
def test_device_matches_golden():
    from paper_2402_10488_b200 import rte
    g = load("c1_slab_si_dsa.npz")
    mesh, p = c1_sys(rte)
    b = rte.TransportBatch(p, mesh, rte.gauss_legendre(16), [[]])
    assert rel_l2(b.apply_L(g["probe"][None]).cpu().numpy()[0], g["L_probe"]) < 1e-10
    assert rel_l2(b.assemble_rhs().cpu().numpy()[0], g["bbar"]) < 1e-10
    rho, reps = rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-10))
    assert reps[0].iterations == int(g["iterations"]) and rel_l2(rho.cpu().numpy()[0], g["rho"]) < 1e-8
    g2 = load("box2d_inflow.npz")
    mesh = rte.Mesh.rect_uniform(0.0, 1.2, 9, -0.5, 1.0, 7)
    b2 = rte.TransportBatch(box_problem(rte), mesh, rte.chebyshev_legendre(8, 4), [[]])
    assert rel_l2(b2.apply_L(g2["probe"][None]).cpu().numpy()[0], g2["L_probe"]) < 1e-10
    rho2, reps2 = rte.sisa_solve(b2, "DSA", rte.SolveConfig(eps_sisa=1e-10))
    assert reps2[0].iterations == int(g2["iterations"]) and rel_l2(rho2.cpu().numpy()[0], g2["rho"]) < 1e-8
    g3 = load("c2_small_romsad.npz")
    train, test = [list(x) for x in g3["train"]], [list(x) for x in g3["test"]]
    pm = rte.Mesh.slab_uniform(0.0, 1.0, 64)
    tb = rte.TransportBatch(two_region_slab(rte), pm, rte.gauss_legendre(16), train)
    snaps = rte.collect_snapshots(tb, 3, 1e-8)
    assert list(snaps.n_iter) == list(g3["n_conv"])
    F = rte.snapshot_matrix(tb, snaps, "correction")
    r = int(g3["rank"])
    U, sig = rte.pod(F, r)
    big = g3["sigma"] > 1e-7 * g3["sigma"][0]
    np.testing.assert_allclose(sig[big], g3["sigma"][big], rtol=1e-6)
    model = rte.build_reduced_model(tb, U, sig, float(g3["eps_pod"]), 1e-8, "c")
    b3 = rte.TransportBatch(two_region_slab(rte), pm, rte.gauss_legendre(16), test)
    rte.load_rom(b3, 1, model)
    eps_r = rte.romsad_tolerance(1e-8, float(g3["eps_pod"]))
    rho3, reps3 = rte.sisa_solve(b3, "ROMSAD", rte.SolveConfig(eps_sisa=1e-8, theta=3, eps_romsad=eps_r))
    rho3 = rho3.cpu().numpy()
    for s in range(len(test)):
        assert reps3[s].iterations == int(g3["iterations"][s])
        assert reps3[s].correction_log == str(g3["logs"][s])
        assert rel_l2(rho3[s], g3["rho"][s]) < 1e-8
