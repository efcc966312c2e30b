"""XY problems with intra-cell-varying coefficients: the
reference assembles full 4x4 per-cell mass blocks by 6x6 Gauss quadrature
(transport_system.cpp:17-55, 111-140); the device path then uses the general
cell solve in the sweep, full blocks in Ms/Mt, and stored Schur factors on
the finest DSA level.  Parity against the oracle (1e-10 per sweep, 1e-8 at
convergence, identical iteration counts), plus: forcing the full-block path
on a cell-constant problem reproduces the sigma-I path.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import rel_l2
from tests.test_gpu_parity import pair_2d

pytestmark = pytest.mark.gpu


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def varying(mod):
    """sigma_a, sigma_s vary inside every cell; left inflow; smooth source."""
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.3 + 0.4 * x * y,
                             scattering_weight=lambda x, y: 1.5 + 0.8 * np.sin(3.0 * x) + 0.3 * y)
    return mod.ProblemDefinition(mod.XY2D, [t0], lambda x, y: 1.0 + x - 0.5 * y, inflow_left=0.7, inflow_bottom=0.2)


def tiny_param(mod):  # acceptance.cpp:100-116 (intra-cell-varying scattering in term 1)
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.25, scattering_weight=lambda x, y: 0.6)
    t1 = mod.CoefficientTerm(psi=lambda mu: mu[0], scattering_weight=lambda x, y: 0.2 + 0.1 * x)
    return mod.ProblemDefinition(mod.XY2D, [t0, t1], lambda x, y: 1.0 + 0.3 * x + 0.1 * y, inflow_left=0.4,
                                 n_params=1, param_ranges=[(0.0, 1.0)])


def test_full_block_operator_parity():
    osys, batch = pair_2d(varying, 13, 9, (8, 4), [[]])
    assert batch._keep[0].shape[-1] == 16  # full blocks selected
    o = osys[0]
    rng = np.random.default_rng(4)
    rho = rng.uniform(-1, 1, (1, o.n_dof()))
    assert rel_l2(batch.apply_L(rho).cpu().numpy()[0], o.apply_L(rho[0])) < 1e-10
    assert rel_l2(batch.assemble_rhs().cpu().numpy()[0], o.assemble_rhs()) < 1e-10
    assert rel_l2(batch.apply_Ms(rho).cpu().numpy()[0], o.apply_Ms(rho[0])) < 1e-14
    assert rel_l2(batch.apply_Mt(rho).cpu().numpy()[0], o.apply_Mt(rho[0])) < 1e-14
    for j in (0, 5, o.quad.n() - 1):
        assert rel_l2(batch.sweep_direction(j, rho).cpu().numpy()[0], o.sweep_direction(j, rho[0])) < 1e-10
    f = batch.kinetic_sweep(rho).cpu().numpy()[0]
    assert rel_l2(f, o.kinetic_sweep(rho[0])) < 1e-10


def test_full_block_dsa_and_solvers_parity():
    R = rte()
    osys, batch = pair_2d(varying, 16, 16, (8, 4), [[]])
    o = osys[0]
    d = R.DsaOperator(batch)
    d.set_tolerance(1e-13, 2000)
    rng = np.random.default_rng(5)
    rhs = rng.uniform(-1, 1, (1, o.n_dof()))
    od = ro.build_dsa(o)
    assert rel_l2(d.solve_density(rhs).cpu().numpy()[0], od.solve_density(rhs[0])) < 1e-9
    assert rel_l2(d.correct(rhs).cpu().numpy()[0], od.correct(rhs[0])) < 1e-9
    for method, strat in (("SI", None), ("DSA", ro.DsaStrategy(od))):
        rho, reps = R.sisa_solve(batch, method, R.SolveConfig(eps_sisa=1e-10, max_iters=5000))
        orho, orep = ro.sisa_solve(o, strat, ro.SolveConfig(eps_sisa=1e-10, max_iters=5000))
        assert reps[0].iterations == orep.iterations and reps[0].correction_log == orep.correction_log
        assert rel_l2(rho.cpu().numpy()[0], orho) < 1e-8
    grho, greps = R.gmres_solve(batch, d, R.SolveConfig(gmres_rel_tol=1e-11))
    gorho, gorep = ro.gmres_solve(o, od, ro.SolveConfig(gmres_rel_tol=1e-11))
    assert greps[0].iterations == gorep.iterations and greps[0].n_sweep == gorep.n_sweep
    assert rel_l2(grho.cpu().numpy()[0], gorho) < 1e-8


def test_full_block_path_matches_sigma_path():
    """A cell-constant problem forced onto the full-block path gives the sigma-I answers."""
    R = rte()
    from tests.problems import prob2d_const
    prob = lambda m: prob2d_const(m, 0.4, 2.0, lambda x, y: 1.0 + x, inflow_left=1.0)
    mesh = R.Mesh.rect_uniform(0, 1, 24, 0, 1, 20)
    quad = R.chebyshev_legendre(8, 4)
    b1 = R.TransportBatch(prob(R), mesh, quad, [[]])
    b16 = R.TransportBatch(prob(R), mesh, quad, [[]], force_full_blocks=True)
    assert b1._keep[0].ndim == 2 and b16._keep[0].shape[-1] == 16
    rho = np.random.default_rng(6).uniform(0, 1, (1, b1.n_dof()))
    assert rel_l2(b16.apply_L(rho).cpu().numpy(), b1.apply_L(rho).cpu().numpy()) < 1e-13
    cfg = R.SolveConfig(eps_sisa=1e-10)
    r1, p1 = R.sisa_solve(b1, "DSA", cfg)
    r16, p16 = R.sisa_solve(b16, "DSA", cfg)
    assert p1[0].iterations == p16[0].iterations
    assert rel_l2(r16.cpu().numpy(), r1.cpu().numpy()) < 1e-9


def test_full_block_parametric_rom_parity():
    """acceptance.cpp tiny XY instance (intra-cell-varying affine term):
    ROMIG guess and ROMSAD with an oracle-built correction model."""
    R = rte()
    om = ro.Mesh.rect_uniform(0.0, 1.0, 8, 0.0, 1.0, 8)
    sp = ro.build_dg_space(om)
    quad = ro.chebyshev_legendre(4, 2)
    prob = tiny_param(ro)
    snaps = []
    for m in (0.2, 0.5, 0.8):
        s_ = ro.TransportSystem(prob, om, sp, quad, [m])
        snaps.append(ro.collect_snapshots(s_, ro.build_dsa(s_), window=3, eps_train=1e-12))
    pod = ro.pod_truncate(ro.correction_matrix(snaps, 3), 1e-12)
    cm = ro.build_reduced_model(ro.TransportSystem(prob, om, sp, quad, [0.2]), pod.u, pod.singular_values,
                                1e-12, 1e-12, "c")
    prim = ro.pod_truncate(ro.primary_matrix(snaps), 1e-14)
    pm = ro.build_reduced_model(ro.TransportSystem(prob, om, sp, quad, [0.2]), prim.u, prim.singular_values,
                                1e-14, 1e-12, "p")
    mus = [[0.35], [0.65]]
    batch = R.TransportBatch(tiny_param(R), R.Mesh.rect_uniform(0.0, 1.0, 8, 0.0, 1.0, 8),
                             R.chebyshev_legendre(4, 2), mus)
    assert batch._keep[0].shape[-1] == 16
    R.load_rom(batch, 0, pm)
    R.load_rom(batch, 1, cm)
    dsa = R.DsaOperator(batch)
    dsa.set_tolerance(1e-13, 2000)
    g, st = R.romig(batch)
    eps_r = ro.romsad_tolerance(1e-12, 1e-12)
    rho, reps = R.sisa_solve(batch, "ROMSAD", R.SolveConfig(eps_sisa=1e-11, theta=3, eps_romsad=eps_r))
    for s, mu in enumerate(mus):
        o = ro.TransportSystem(prob, om, sp, quad, mu)
        assert rel_l2(g.cpu().numpy()[s], ro.romig(pm, o)) < 1e-10
        orho, orep = ro.sisa_solve(o, ro.RomsadStrategy(cm, ro.build_dsa(o), 3, eps_r),
                                   ro.SolveConfig(eps_sisa=1e-11))
        assert reps[s].iterations == orep.iterations and reps[s].correction_log == orep.correction_log
        assert rel_l2(rho.cpu().numpy()[s], orho) < 1e-8
