"""GPU parity of the online ROM stage (ROMIG, ROMSA, ROMSAD) on the
BASELINE configs[1] slab (two-region, eps log-uniform, c uniform) against the
oracle, with reduced models built offline by the oracle (collect_snapshots ->
POD (LAPACK dgesdd) -> build_reduced_model, reduced_model.cpp:106-199).

Checks per sample: identical iteration counts, correction logs and ROMSAD
switch iteration; scalar flux within 1e-8 at convergence; ROMIG guess within
1e-10 of the oracle's.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import rel_l2, two_region_slab, parametric_slab

pytestmark = pytest.mark.gpu

EPS_TRAIN = 1e-8
EPS_SISA = 1e-8
WINDOW = 3


def c2_params(n_train, n_test):
    from paper_2402_10488_b200 import configs
    return configs.c2_params(n_train, n_test)


@pytest.fixture(scope="module")
def c2_offline():
    """Oracle offline stage on a C2-shaped problem (128 cells to keep it quick)."""
    train, test = c2_params(16, 12)
    mesh = ro.Mesh.slab_uniform(0.0, 1.0, 128)
    space = ro.build_dg_space(mesh)
    quad = ro.gauss_legendre(16)
    prob = two_region_slab(ro)
    snaps = []
    for mu in train:
        sys_ = ro.TransportSystem(prob, mesh, space, quad, mu)
        snaps.append(ro.collect_snapshots(sys_, ro.build_dsa(sys_), window=WINDOW, eps_train=EPS_TRAIN))
    prim = ro.pod_truncate(ro.primary_matrix(snaps), 1e-16)
    corr = ro.pod_truncate(ro.correction_matrix(snaps, WINDOW), 1e-16)
    rp, rc = min(prim.rank, 12), min(corr.rank, 16)
    eps_p = float(np.sum(prim.singular_values[rp:]) / np.sum(prim.singular_values))
    eps_c = float(np.sum(corr.singular_values[rc:]) / np.sum(corr.singular_values))
    repr_sys = ro.TransportSystem(prob, mesh, space, quad, train[0])
    pm = ro.build_reduced_model(repr_sys, prim.u[:, :rp], prim.singular_values, eps_p, EPS_TRAIN, "p")
    cm = ro.build_reduced_model(repr_sys, corr.u[:, :rc], corr.singular_values, eps_c, EPS_TRAIN, "c")
    return dict(mesh=mesh, quad=quad, prob=prob, test=test, primary=pm, correction=cm)


def device_batch(off):
    from paper_2402_10488_b200 import rte
    pm = rte.Mesh.slab(off["mesh"].boundaries)
    b = rte.TransportBatch(two_region_slab(rte), pm, rte.gauss_legendre(16), off["test"])
    rte.load_rom(b, 0, off["primary"])
    rte.load_rom(b, 1, off["correction"])
    return b


def oracle_sys(off, mu):
    return ro.TransportSystem(off["prob"], off["mesh"], ro.build_dg_space(off["mesh"]), off["quad"], mu)


def test_romig_guess_parity(c2_offline):
    from paper_2402_10488_b200 import rte
    b = device_batch(c2_offline)
    rho0, status = rte.romig(b)
    rho0 = rho0.cpu().numpy()
    assert np.all(status == 0)
    for s, mu in enumerate(c2_offline["test"]):
        ref = ro.romig(c2_offline["primary"], oracle_sys(c2_offline, mu))
        assert rel_l2(rho0[s], ref) < 1e-10


@pytest.mark.parametrize("method,theta", [("ROMIG", 0), ("ROMSA", 0), ("ROMSAD", 3)])
def test_rom_solve_parity(c2_offline, method, theta):
    from paper_2402_10488_b200 import rte
    b = device_batch(c2_offline)
    cm = c2_offline["correction"]
    eps_r = ro.romsad_tolerance(EPS_TRAIN, cm.eps_pod)
    cfg = rte.SolveConfig(eps_sisa=EPS_SISA, max_iters=400, theta=theta, eps_romsad=eps_r)
    rho, reps = rte.sisa_solve(b, method, cfg)
    rho = rho.cpu().numpy()
    for s, mu in enumerate(c2_offline["test"]):
        sys_ = oracle_sys(c2_offline, mu)
        dsa = ro.build_dsa(sys_)
        if method == "ROMIG":
            o_rho, o_rep = ro.sisa_solve(sys_, ro.DsaStrategy(dsa),
                                         ro.SolveConfig(eps_sisa=EPS_SISA, max_iters=400,
                                                        initial_guess=ro.romig(c2_offline["primary"], sys_)))
        elif method == "ROMSA":
            o_rho, o_rep = ro.sisa_solve(sys_, ro.RomsaStrategy(cm), ro.SolveConfig(eps_sisa=EPS_SISA, max_iters=400))
        else:
            o_rho, o_rep = ro.sisa_solve(sys_, ro.RomsadStrategy(cm, dsa, theta, eps_r),
                                         ro.SolveConfig(eps_sisa=EPS_SISA, max_iters=400))
        r = reps[s]
        assert r.converged == o_rep.converged
        assert r.iterations == o_rep.iterations, (s, r.iterations, o_rep.iterations)
        assert r.correction_log == o_rep.correction_log, (s, r.correction_log, o_rep.correction_log)
        if method == "ROMSAD":
            o_switch = o_rep.correction_log.find("D")
            assert r.switch_iter == (o_switch + 1 if o_switch >= 0 else -1)
        if o_rep.converged:
            assert rel_l2(rho[s], o_rho) < 1e-8


def test_singular_reduced_model_degrades_gracefully():
    """test_rom.cpp:169-193 through the device path: ROMSA gives 'S' (zero
    correction), ROMSAD switches to DSA at once, ROMIG raises."""
    from paper_2402_10488_b200 import capi, rte
    mesh = rte.Mesh.slab_uniform(0.0, 2.0, 8)
    b = rte.TransportBatch(parametric_slab(rte), mesh, rte.gauss_legendre(4), [[0.4], [0.6]])
    broken = rte.ReducedModel(0, 4, b.n_dof(), 1, 2, "c", 1e-9, 1e-11, np.zeros((b.n_dof(), 1)),
                              np.zeros((b.n_dof(), 1)), [np.zeros((1, 1)), np.zeros((1, 1))], np.ones(1), 0.0,
                              np.zeros(1))
    rte.load_rom(b, 0, broken)
    rte.load_rom(b, 1, broken)
    _, reps = rte.sisa_solve(b, "ROMSA", rte.SolveConfig(eps_sisa=1e-10, max_iters=500))
    assert all(r.singular and set(r.correction_log) <= {"S"} for r in reps)
    _, reps = rte.sisa_solve(b, "ROMSAD", rte.SolveConfig(eps_sisa=1e-10, max_iters=500, theta=3, eps_romsad=1e-10))
    assert all(r.correction_log and set(r.correction_log) == {"D"} and r.switch_iter == 1 for r in reps)
    with pytest.raises(capi.RteError):
        rte.sisa_solve(b, "ROMIG", rte.SolveConfig(eps_sisa=1e-10))
