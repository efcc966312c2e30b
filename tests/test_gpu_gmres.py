"""GPU parity of batched (P)GMRES (gmres.cpp:15-124) against the oracle's
gmres_solve on the same inputs: identical inner-iteration counts, sweep
counts and history lengths; history values within 1e-6 relative (the
Arnoldi sums are reduced in a different fixed order); scalar flux within
1e-8 at convergence.  Cases follow the reference's own GMRES tests
(test_solvers.cpp:101-121 restarts, test_dsa.cpp:85-93 n_sweep = it + 3,
test_dsa.cpp:147-163 pure absorber) plus a parametric batch, PGMRES-ROMIG
and an XY problem.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import homog, parametric_slab, prob2d_const, rel_l2, two_region_slab
from tests.test_gpu_parity import pair_1d, pair_2d

pytestmark = pytest.mark.gpu

CONV_TOL = 1e-8


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def check(osys, batch, pre, m, tol, max_iters=2000, guess=None, romig_models=None, dsa=None):
    R = rte()
    cfg = R.SolveConfig(gmres_restart=m, gmres_rel_tol=tol, max_iters=max_iters, initial_guess=guess)
    if pre and dsa is None:
        dsa = R.DsaOperator(batch)
    rho, reps = R.gmres_solve(batch, dsa, cfg, romig_guess=romig_models is not None)
    rho = rho.cpu().numpy()
    for s, o in enumerate(osys):
        g0 = None
        if romig_models is not None:
            g0 = ro.romig(romig_models, o)
        elif guess is not None:
            g0 = np.asarray(guess)[s]
        ocfg = ro.SolveConfig(gmres_restart=m, gmres_rel_tol=tol, max_iters=max_iters, initial_guess=g0)
        orho, orep = ro.gmres_solve(o, ro.build_dsa(o) if pre else None, ocfg)
        r = reps[s]
        assert r.converged == orep.converged
        assert r.iterations == orep.iterations, (s, r.iterations, orep.iterations)
        assert r.n_sweep == orep.n_sweep
        assert len(r.change_history) == len(orep.change_history)
        h, ho = np.array(r.change_history), np.array(orep.change_history)
        assert np.all(np.abs(h - ho) <= 1e-6 * np.maximum(ho, 1e-14) + 1e-13)
        assert r.strategy == orep.strategy and r.initial_guess == orep.initial_guess
        if orep.converged:
            assert rel_l2(rho[s], orho) < CONV_TOL
            assert r.final_residual == pytest.approx(orep.final_residual, rel=1e-6, abs=1e-14)
    return reps


def test_gmres_restarts_match_oracle():
    """test_solvers.cpp:101-121: plain GMRES with restart 5, tol 1e-12."""
    osys, batch = pair_1d(parametric_slab, np.linspace(0, 2, 9), 4, [[0.4]])
    reps = check(osys, batch, False, 5, 1e-12)
    assert reps[0].converged and len(reps[0].change_history) > reps[0].iterations
    assert reps[0].change_history[-1] <= 1e-12


def test_pgmres_sweep_accounting():
    """test_dsa.cpp:85-93: preconditioned GMRES converges in one cycle; n_sweep = iterations + 3."""
    osys, batch = pair_1d(lambda m: homog(m, m.SLAB1D, 1.0, 0.99, 1.0), np.linspace(0, 10, 101), 8, [[]])
    reps = check(osys, batch, True, 25, 1e-11)
    assert reps[0].n_sweep == reps[0].iterations + 3


def test_pgmres_pure_absorber_identity():
    """test_dsa.cpp:147-163: P A = I for sigma_s = 0 -> one iteration, four sweeps."""
    osys, batch = pair_1d(lambda m: homog(m, m.SLAB1D, 1.0, 0.0, 1.0), np.linspace(0, 1, 9), 4, [[]])
    reps = check(osys, batch, True, 25, 1e-11)
    assert reps[0].iterations == 1 and reps[0].n_sweep == 4


def test_gmres_batch_masks_samples():
    """Samples of a parametric batch converge at different cycles/steps."""
    mus = [[1e-3, 0.95], [0.2, 0.9999], [1.0, 0.9], [0.05, 0.99]]
    osys, batch = pair_1d(two_region_slab, np.linspace(0, 1, 129), 16, mus)
    check(osys, batch, True, 25, 1e-11)
    check(osys, batch, False, 10, 1e-10, max_iters=60)


def test_gmres_iteration_cap_reports_nonconvergence():
    osys, batch = pair_1d(lambda m: homog(m, m.SLAB1D, 1.0, 0.999, 1.0), np.linspace(0, 20, 81), 8, [[]])
    reps = check(osys, batch, False, 4, 1e-13, max_iters=6)
    assert not reps[0].converged and reps[0].iterations == 6 and reps[0].final_residual > 0


def test_gmres_supplied_guess():
    osys, batch = pair_1d(parametric_slab, np.linspace(0, 2, 9), 4, [[0.1], [0.77]])
    rng = np.random.default_rng(3)
    guess = rng.uniform(0, 1, (2, osys[0].n_dof()))
    check(osys, batch, True, 25, 1e-11, guess=guess)


def test_pgmres_romig_parity():
    """PGMRES-ROMIG (runner.cpp:202-205) with an oracle-built primary model."""
    train_mesh = ro.Mesh.slab_uniform(0.0, 1.0, 64)
    space = ro.build_dg_space(train_mesh)
    quad = ro.gauss_legendre(8)
    prob = two_region_slab(ro)
    from paper_2402_10488_b200 import configs
    train, test = configs.c2_params(8, 4)
    snaps = [ro.collect_snapshots(ro.TransportSystem(prob, train_mesh, space, quad, mu),
                                  ro.build_dsa(ro.TransportSystem(prob, train_mesh, space, quad, mu)),
                                  window=3, eps_train=1e-8) for mu in train]
    prim = ro.pod_truncate(ro.primary_matrix(snaps), 1e-16)
    rp = min(prim.rank, 6)
    eps_p = float(np.sum(prim.singular_values[rp:]) / np.sum(prim.singular_values))
    pm = ro.build_reduced_model(ro.TransportSystem(prob, train_mesh, space, quad, train[0]), prim.u[:, :rp],
                                prim.singular_values, eps_p, 1e-8, "p")
    R = rte()
    batch = R.TransportBatch(two_region_slab(R), R.Mesh.slab(train_mesh.boundaries), R.gauss_legendre(8), test)
    R.load_rom(batch, 0, pm)
    osys = [ro.TransportSystem(prob, train_mesh, space, quad, mu) for mu in test]
    check(osys, batch, True, 25, 1e-11, romig_models=pm)


def test_pgmres_xy():
    osys, batch = pair_2d(lambda m: prob2d_const(m, 2.0, 1.8, lambda x, y: 1.0 + x, inflow_left=0.5), 12, 10,
                          (8, 4), [[]])
    dsa = rte().DsaOperator(batch)
    dsa.set_tolerance(1e-13, 2000)
    check(osys, batch, True, 25, 1e-10, dsa=dsa)
