"""GPU parity of the kinetic-space operators: kinetic_sweep / density_of
(transport_system.cpp:420-441) in 1D and 2D (all original directions, ±vz
copies included) and the affine term operators apply_term_kinetic
(transport_system.cpp:560-596), plus a 2D pin-cell offline + ROMSAD check."""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import pin_cell, prob2d_const, rel_l2

pytestmark = pytest.mark.gpu


def affine_1d(mod):  # test_assembly.cpp:40-55 with cell-wise (not intra-cell) weights kept general
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.3, scattering_weight=lambda x, y: 0.6 + 0.1 * x)
    t1 = mod.CoefficientTerm(psi=lambda mu: mu[0], absorption_weight=lambda x, y: 0.05 + 0.02 * x)
    t2 = mod.CoefficientTerm(psi=lambda mu: mu[1] * mu[1], scattering_weight=lambda x, y: 0.3 + 0.05 * x)
    return mod.ProblemDefinition(mod.SLAB1D, [t0, t1, t2], lambda x, y: 1.0 + x, inflow_left=2.0, inflow_right=0.5,
                                 n_params=2)


def affine_2d(mod):
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.4, scattering_weight=lambda x, y: 0.5)
    t1 = mod.CoefficientTerm(psi=lambda mu: mu[0], absorption_weight=lambda x, y: 0.7)
    t2 = mod.CoefficientTerm(psi=lambda mu: mu[1], scattering_weight=lambda x, y: 1.3)
    return mod.ProblemDefinition(mod.XY2D, [t0, t1, t2], lambda x, y: 1.0 + x, inflow_left=1.0, inflow_bottom=0.5,
                                 n_params=2)


def systems(geom):
    from paper_2402_10488_b200 import rte
    mus = [[0.3, 1.4], [1.7, 0.2]]
    if geom == 1:
        om = ro.Mesh.slab([0.0, 0.5, 1.0, 1.6, 2.0])
        pm = rte.Mesh.slab([0.0, 0.5, 1.0, 1.6, 2.0])
        osys = [ro.TransportSystem(affine_1d(ro), om, ro.build_dg_space(om), ro.gauss_legendre(8), m) for m in mus]
        b = rte.TransportBatch(affine_1d(rte), pm, rte.gauss_legendre(8), mus)
    else:
        om = ro.Mesh.rect_uniform(0, 1.2, 7, 0, 1, 5)
        pm = rte.Mesh.rect_uniform(0, 1.2, 7, 0, 1, 5)
        osys = [ro.TransportSystem(affine_2d(ro), om, ro.build_dg_space(om), ro.chebyshev_legendre(8, 4), m)
                for m in mus]
        b = rte.TransportBatch(affine_2d(rte), pm, rte.chebyshev_legendre(8, 4), mus)
    return osys, b


@pytest.mark.parametrize("geom", [1, 2])
def test_kinetic_sweep_and_density(geom):
    osys, b = systems(geom)
    rho = np.random.default_rng(4).uniform(0, 1, (2, b.n_dof()))
    f = b.kinetic_sweep(rho).cpu().numpy()
    d = b.density_of(f).cpu().numpy()
    for s, o in enumerate(osys):
        fo = o.kinetic_sweep(rho[s])
        assert rel_l2(f[s], fo) < 1e-10
        assert rel_l2(d[s], o.density_of(fo)) < 1e-10


@pytest.mark.parametrize("geom", [1, 2])
def test_apply_term_kinetic(geom):
    osys, b = systems(geom)
    u = np.random.default_rng(8).uniform(-1, 1, (3, b.kinetic_dim()))
    for k in range(3):
        out = b.apply_term_kinetic(k, u).cpu().numpy()
        for c in range(3):
            ref = osys[0].apply_term_kinetic(k, u[c])
            assert np.max(np.abs(out[c] - ref)) < 1e-12 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("geom", [1, 2])
def test_apply_kinetic_streaming_collision_and_rhs(geom):
    """apply_kinetic (transport_system.cpp:598-613) per sample, the
    streaming-collision operator and its sweep inverse (test_sweep.cpp:30-50:
    (D_j + Sigma_t) sweep_j(r) = r), and the kinetic right-hand side; the
    converged kinetic solution satisfies A_mu f = b (test_assembly.cpp:100-110)."""
    osys, b = systems(geom)
    rng = np.random.default_rng(12)
    u = rng.uniform(-1, 1, (2, b.kinetic_dim()))
    au = b.apply_kinetic(u).cpu().numpy()
    kb = b.kinetic_rhs().cpu().numpy()
    for s, o in enumerate(osys):
        ref = o.apply_kinetic(u[s])
        assert np.max(np.abs(au[s] - ref)) < 1e-12 * max(1.0, np.max(np.abs(ref)))
        assert np.max(np.abs(kb[s] - o.kinetic_rhs())) < 1e-13
    f = rng.uniform(-1, 1, (2, b.n_dof()))
    for j in (0, b.quad.n() // 2, b.quad.n() - 1):
        sc = b.apply_streaming_collision(j, f).cpu().numpy()
        back = b.apply_streaming_collision(j, b.sweep_direction(j, f)).cpu().numpy()
        for s, o in enumerate(osys):
            ref = o.apply_streaming_collision(j, f[s])
            assert np.max(np.abs(sc[s] - ref)) < 1e-12 * max(1.0, np.max(np.abs(ref)))
            assert rel_l2(back[s], f[s]) < 1e-12
    # the kinetic fixed point: A_mu f* = b
    from paper_2402_10488_b200 import rte
    rho, _ = rte.sisa_solve(b, "SI", rte.SolveConfig(eps_sisa=1e-13, max_iters=20000))
    fk = b.kinetic_sweep(rho)
    res = (b.apply_kinetic(fk) - b.kinetic_rhs()).cpu().numpy()
    assert np.max(np.abs(res)) < 1e-9 * max(1.0, np.max(np.abs(kb)))


def test_pin_cell_offline_and_romsad():
    """BASELINE configs[3] shape at reduced size: device training, POD,
    projections and ROMSAD(3,5) vs the oracle with the device-built model."""
    from paper_2402_10488_b200 import configs, rte
    nx = 16
    train, test = configs.c4_params(8, 4)
    make = pin_cell(ro)
    om = ro.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    pm = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    quad_o, quad_p = ro.chebyshev_legendre(8, 4), rte.chebyshev_legendre(8, 4)
    tb = rte.TransportBatch(pin_cell(rte)(nx), pm, quad_p, train)
    snaps = rte.collect_snapshots(tb, 3, 1e-8)
    osn = []
    for s, mu in enumerate(train):
        o = ro.TransportSystem(make(nx), om, ro.build_dg_space(om), quad_o, mu)
        sn = ro.collect_snapshots(o, ro.build_dsa(o), window=3, eps_train=1e-8)
        osn.append(sn)
        assert int(snaps.n_iter[s]) == sn.n_conv
    F = rte.snapshot_matrix(tb, snaps, "correction")
    r = 10
    U, sig = rte.pod(F, r)
    eps_pod = float(np.sum(sig[r:]) / np.sum(sig))
    dm = rte.build_reduced_model(tb, U, sig, eps_pod, 1e-8, "c")
    om_ = ro.ReducedModel(dm.geometry, dm.n_v, dm.n_dof, dm.rank, dm.k_affine, dm.kind, dm.eps_pod, dm.eps_train,
                          dm.u_rho, dm.u_iso, dm.a_r, dm.singular_values, dm.discarded_fraction, dm.b_r)
    b = rte.TransportBatch(pin_cell(rte)(nx), pm, quad_p, test)
    rte.load_rom(b, 1, dm)
    eps_r = ro.romsad_tolerance(1e-8, eps_pod)
    rho, reps = rte.sisa_solve(b, "ROMSAD", rte.SolveConfig(eps_sisa=1e-8, theta=5, eps_romsad=eps_r))
    rho = rho.cpu().numpy()
    for s, mu in enumerate(test):
        o = ro.TransportSystem(make(nx), om, ro.build_dg_space(om), quad_o, mu)
        o_rho, o_rep = ro.sisa_solve(o, ro.RomsadStrategy(om_, ro.build_dsa(o), 5, eps_r), ro.SolveConfig(eps_sisa=1e-8))
        assert reps[s].iterations == o_rep.iterations and reps[s].correction_log == o_rep.correction_log
        assert rel_l2(rho[s], o_rho) < 1e-8
