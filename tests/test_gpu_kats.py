"""The reference's own known-answer tests, restated directly on the device
path (no oracle in between):

* exact initial guess: 1 iteration, 2 sweeps (test_solvers.cpp:64-86);
* pure absorber with left inflow: analytic attenuation of the cell averages
  (test_sweep.cpp:74-99);
* 2D upwind causality: exactly zero upstream of a point source
  (test_sweep.cpp:101-125);
* symmetric slab: symmetric converged density (test_sweep.cpp:127-149);
* one DSA-accelerated iteration equals preconditioned Richardson
  (test_dsa.cpp:58-69), 1D (DemoSlab) and XY;
* pure absorber: SI converges in 2 iterations / 3 sweeps (test_dsa.cpp:147-163).
"""
import numpy as np
import pytest

from tests.problems import homog

pytestmark = pytest.mark.gpu


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def scatter_slab(mod):  # test_solvers.cpp:12-22
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.3, scattering_weight=lambda x, y: 0.8 + 0.1 * x)
    return mod.ProblemDefinition(mod.SLAB1D, [t0], lambda x, y: 1.0 + 0.2 * x, inflow_left=0.5)


def test_exact_initial_guess_one_iteration():
    R = rte()
    b = R.TransportBatch(scatter_slab(R), R.Mesh.slab_uniform(0.0, 3.0, 48), R.gauss_legendre(8), [[]])
    rho, rep0 = R.sisa_solve(b, "SI", R.SolveConfig(eps_sisa=1e-10))
    assert rep0[0].converged and rep0[0].initial_guess == "zero"
    rho1, rep1 = R.sisa_solve(b, "SI", R.SolveConfig(eps_sisa=1e-10, initial_guess=rho))
    assert rep1[0].converged and rep1[0].iterations == 1 and rep1[0].n_sweep == 2
    assert rep1[0].initial_guess == "supplied"
    r, r1 = rho.cpu().numpy(), rho1.cpu().numpy()
    assert np.max(np.abs(r1 - r)) < 1e-9 * np.max(np.abs(r))
    rg, repg = R.gmres_solve(b, None, R.SolveConfig(initial_guess=rho))
    assert repg[0].converged and repg[0].iterations <= 1 and repg[0].initial_guess == "supplied"


def test_pure_absorber_analytic_attenuation():
    R = rte()
    sig, g_in = 2.0, 1.5
    mesh = R.Mesh.slab_uniform(0.0, 1.0, 64)
    quad = R.gauss_legendre(4)
    b = R.TransportBatch(homog(R, R.SLAB1D, sig, 0.0, 0.0, inflow_left=g_in), mesh, quad, [[]])
    kr = b.kinetic_rhs().cpu().numpy()[0]  # block j = G + g_j^bc with G = 0
    nd = b.n_dof()
    h = 1.0 / 64
    for j in range(4):
        v = quad.directions[j][0]
        f = b.sweep_direction(j, kr[j * nd:(j + 1) * nd][None]).cpu().numpy()[0]
        avg = f[0::2] / np.sqrt(h)  # orthonormal mode 0 = 1/sqrt(h)
        if v < 0:
            assert np.max(np.abs(avg)) == 0.0
        else:
            for i in range(0, 64, 13):
                x0 = i * h
                exact = g_in * v / (sig * h) * (np.exp(-sig * x0 / v) - np.exp(-sig * (x0 + h) / v))
                assert abs(avg[i] - exact) < 1e-3 * g_in


def test_upwind_causality_2d():
    R = rte()
    mesh = R.Mesh.rect_uniform(0.0, 1.0, 8, 0.0, 1.0, 8)
    quad = R.chebyshev_legendre(4, 2)
    b = R.TransportBatch(homog(R, R.XY2D, 1.0, 0.0, 0.0), mesh, quad, [[]])
    sx, sy = 3, 4
    rhs = np.zeros((1, b.n_dof()))
    rhs[0, 4 * (sx + 8 * sy)] = 1.0
    for j in range(quad.n()):
        f = b.sweep_direction(j, rhs).cpu().numpy()[0].reshape(8, 8, 4)  # [iy][ix][local]
        dx = 1 if quad.directions[j][0] > 0 else -1
        dy = 1 if quad.directions[j][1] > 0 else -1
        for iy in range(8):
            for ix in range(8):
                down = (ix >= sx if dx > 0 else ix <= sx) and (iy >= sy if dy > 0 else iy <= sy)
                if not down:
                    assert np.all(f[iy, ix] == 0.0)


def test_symmetric_slab_symmetric_density():
    R = rte()
    n = 40
    t0 = R.CoefficientTerm(absorption_weight=lambda x, y: 0.3, scattering_weight=lambda x, y: 1.2)
    p = R.ProblemDefinition(R.SLAB1D, [t0], lambda x, y: np.exp(-30.0 * (x - 0.5) ** 2), inflow_left=0.8,
                            inflow_right=0.8)
    b = R.TransportBatch(p, R.Mesh.slab_uniform(0.0, 1.0, n), R.gauss_legendre(8), [[]])
    rho, rep = R.sisa_solve(b, "SI", R.SolveConfig(eps_sisa=1e-13, max_iters=4000))
    avg = rho.cpu().numpy()[0][0::2] * np.sqrt(n)
    for i in range(n // 2):
        assert abs(avg[i] - avg[n - 1 - i]) < 1e-11


@pytest.mark.parametrize("geom", ["1d", "2d"])
def test_dsa_step_equals_preconditioned_richardson(geom):
    R = rte()
    if geom == "1d":  # DemoSlab (test_dsa.cpp:24-30)
        b = R.TransportBatch(homog(R, R.SLAB1D, 0.0, 1.0, 0.01), R.Mesh.slab_uniform(0, 10, 400),
                             R.gauss_legendre(16), [[]])
        tol = 1e-12
    else:
        b = R.TransportBatch(homog(R, R.XY2D, 0.2, 1.8, 1.0, inflow_left=0.3), R.Mesh.rect_uniform(0, 1, 16, 0, 1, 16),
                             R.chebyshev_legendre(8, 4), [[]])
        tol = 1e-10
    d = R.DsaOperator(b)
    if geom == "2d":
        d.set_tolerance(1e-14, 4000)
    r0 = np.random.default_rng(21).uniform(-1, 1, (1, b.n_dof()))
    bbar = b.assemble_rhs()
    rho_star = b.apply_L(r0) + bbar
    step = rho_star + d.correct(rho_star - b._dev(r0))
    resid = bbar - (b._dev(r0) - b.apply_L(r0))
    rich = b._dev(r0) + resid + d.solve_density(b.apply_Ms(resid))
    diff = (step - rich).abs().max().item()
    assert diff < tol * max(1.0, step.abs().max().item())


def test_pure_absorber_si_counts():
    R = rte()
    b = R.TransportBatch(homog(R, R.SLAB1D, 1.0, 0.0, 1.0), R.Mesh.slab_uniform(0, 1, 8), R.gauss_legendre(4), [[]])
    rho, rep = R.sisa_solve(b, "SI", R.SolveConfig())
    assert rep[0].iterations == 2 and rep[0].n_sweep == 3
