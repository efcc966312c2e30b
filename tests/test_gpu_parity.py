"""GPU parity tests: the sm_100a path (through the C-ABI) against the CPU
oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star): scalar flux within 1e-10 relative L2
per sweep, 1e-8 at convergence; identical iteration counts and ROMSAD switch
iteration.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import homog, prob1d, parametric_slab, prob2d_const, rel_l2, two_region_slab

pytestmark = pytest.mark.gpu

SWEEP_TOL = 1e-10
CONV_TOL = 1e-8


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def pair_1d(problem_fn, bounds, nq, mus):
    R = rte()
    om = ro.Mesh.slab(bounds)
    pm = R.Mesh.slab(bounds)
    osys = [ro.TransportSystem(problem_fn(ro), om, ro.build_dg_space(om), ro.gauss_legendre(nq), m) for m in mus]
    batch = R.TransportBatch(problem_fn(R), pm, R.gauss_legendre(nq), mus)
    return osys, batch


def pair_2d(problem_fn, nx, ny, cl, mus, extent=(0.0, 1.0, 0.0, 1.0)):
    R = rte()
    x0, x1, y0, y1 = extent
    om = ro.Mesh.rect_uniform(x0, x1, nx, y0, y1, ny)
    pm = R.Mesh.rect_uniform(x0, x1, nx, y0, y1, ny)
    osys = [ro.TransportSystem(problem_fn(ro), om, ro.build_dg_space(om), ro.chebyshev_legendre(*cl), m) for m in mus]
    batch = R.TransportBatch(problem_fn(R), pm, R.chebyshev_legendre(*cl), mus)
    return osys, batch


CASES_1D = [
    ("demo_slab", lambda m: homog(m, m.SLAB1D, 0.0, 1.0, 0.01), np.linspace(0, 10, 401), 16, [[]]),
    ("nonuniform_inflow", prob1d, [0.0, 0.3, 0.7, 1.2, 2.0, 2.2, 2.9], 8, [[]]),
    ("c1_thick", lambda m: homog(m, m.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0),
     np.linspace(0, 1, 257), 16, [[]]),
    ("rom_tiny_batch", parametric_slab, np.linspace(0, 2, 9), 4, [[0.1], [0.4], [0.77]]),
    ("two_region_batch", two_region_slab, np.linspace(0, 1, 257), 16, [[1e-3, 0.95], [0.2, 0.9999], [1.0, 0.9]]),
]


@pytest.mark.parametrize("name,fn,bounds,nq,mus", CASES_1D, ids=[c[0] for c in CASES_1D])
def test_1d_operator_parity(name, fn, bounds, nq, mus):
    osys, batch = pair_1d(fn, bounds, nq, mus)
    rng = np.random.default_rng(11)
    rho = rng.uniform(-1, 1, (len(mus), osys[0].n_dof()))
    L = batch.apply_L(rho).cpu().numpy()
    B = batch.assemble_rhs().cpu().numpy()
    F = batch.fixed_point(rho).cpu().numpy()
    Ms = batch.apply_Ms(rho).cpu().numpy()
    for s, o in enumerate(osys):
        lo, bo = o.apply_L(rho[s]), o.assemble_rhs()
        assert rel_l2(L[s], lo) < SWEEP_TOL
        assert rel_l2(B[s], bo) < SWEEP_TOL
        assert rel_l2(F[s], lo + bo) < SWEEP_TOL
        assert rel_l2(Ms[s], o.apply_Ms(rho[s])) < 1e-14
    for j in (0, osys[0].quad.n() - 1):
        f = batch.sweep_direction(j, rho).cpu().numpy()
        for s, o in enumerate(osys):
            assert rel_l2(f[s], o.sweep_direction(j, rho[s])) < SWEEP_TOL


@pytest.mark.parametrize("name,fn,bounds,nq,mus", CASES_1D[:3], ids=[c[0] for c in CASES_1D[:3]])
def test_1d_kinetic_sweep_parity(name, fn, bounds, nq, mus):
    osys, batch = pair_1d(fn, bounds, nq, mus)
    rho = np.random.default_rng(5).uniform(0, 1, (1, osys[0].n_dof()))
    f = batch.kinetic_sweep(rho).cpu().numpy()
    fo = osys[0].kinetic_sweep(rho[0])
    assert rel_l2(f[0], fo) < SWEEP_TOL
    d = batch.density_of(f).cpu().numpy()
    assert rel_l2(d[0], osys[0].density_of(fo)) < SWEEP_TOL


@pytest.mark.parametrize("name,fn,bounds,nq,mus", CASES_1D, ids=[c[0] for c in CASES_1D])
def test_1d_dsa_parity(name, fn, bounds, nq, mus):
    osys, batch = pair_1d(fn, bounds, nq, mus)
    R = rte()
    dsa = R.DsaOperator(batch)
    assert dsa.coupled_dim() == 2 * osys[0].n_dof()
    rng = np.random.default_rng(3)
    rhs = rng.uniform(-1, 1, (len(mus), osys[0].n_dof()))
    x = dsa.solve_density(rhs).cpu().numpy()
    c = dsa.correct(rhs).cpu().numpy()
    for s, o in enumerate(osys):
        od = ro.build_dsa(o)
        assert rel_l2(x[s], od.solve_density(rhs[s])) < 1e-10
        assert rel_l2(c[s], od.correct(rhs[s])) < 1e-10


@pytest.mark.parametrize("method", ["SI", "DSA"])
@pytest.mark.parametrize("name,fn,bounds,nq,mus", CASES_1D, ids=[c[0] for c in CASES_1D])
def test_1d_solve_parity(method, name, fn, bounds, nq, mus):
    if method == "SI" and name in ("c1_thick", "demo_slab", "two_region_batch"):
        pytest.skip("plain SI needs thousands of sweeps here (covered by DSA)")
    osys, batch = pair_1d(fn, bounds, nq, mus)
    R = rte()
    eps = 1e-10
    rho, reps = R.sisa_solve(batch, method, R.SolveConfig(eps_sisa=eps, max_iters=3000))
    rho = rho.cpu().numpy()
    for s, o in enumerate(osys):
        strat = ro.DsaStrategy(ro.build_dsa(o)) if method == "DSA" else None
        ro_rho, ro_rep = ro.sisa_solve(o, strat, ro.SolveConfig(eps_sisa=eps, max_iters=3000))
        r = reps[s]
        assert r.converged == ro_rep.converged
        assert r.iterations == ro_rep.iterations, (r.iterations, ro_rep.iterations)
        assert r.n_sweep == ro_rep.n_sweep
        assert r.correction_log == ro_rep.correction_log
        assert rel_l2(rho[s], ro_rho) < CONV_TOL
        np.testing.assert_allclose(r.change_history, ro_rep.change_history, rtol=1e-6, atol=1e-14)
        assert r.final_residual < 100 * eps


def test_1d_rel_norm_and_fixed_iterations():
    osys, batch = pair_1d(CASES_1D[2][1], CASES_1D[2][2], 16, [[]])
    R = rte()
    rho, reps = R.sisa_solve(batch, "DSA", R.SolveConfig(eps_sisa=1e-8, norm="rel"))
    o_rho, o_rep = ro.sisa_solve(osys[0], ro.DsaStrategy(ro.build_dsa(osys[0])),
                                 ro.SolveConfig(eps_sisa=1e-8, norm="rel"))
    assert reps[0].iterations == o_rep.iterations
    assert rel_l2(rho.cpu().numpy()[0], o_rho) < CONV_TOL
    rho5, reps5 = R.sisa_solve(batch, "DSA", R.SolveConfig(fixed_iters=5, max_iters=5))
    assert reps5[0].iterations == 5 and not reps5[0].converged


# ---- 2D ----

CASES_2D = [
    ("box_inflow", lambda m: prob2d_const(m, 0.4, 0.8, lambda x, y: 1.0 + x + 0.5 * y, inflow_left=1.0,
                                          inflow_bottom=0.7, inflow_right=0.2, inflow_top=0.3),
     9, 7, (8, 4), [[]], (0.0, 1.2, -0.5, 1.0)),
    ("c3_like_small", lambda m: prob2d_const(m, 10 * 0.001, 10 * 0.999, lambda x, y: 1.0), 40, 33, (16, 8), [[]],
     (0.0, 1.0, 0.0, 1.0)),
    ("batch_thin", lambda m: m.ProblemDefinition(m.XY2D, [
        m.CoefficientTerm(absorption_weight=lambda x, y: 0.5, scattering_weight=lambda x, y: 0.2),
        m.CoefficientTerm(psi=lambda mu: mu[0], scattering_weight=lambda x, y: 1.0)],
        lambda x, y: np.exp(-10 * ((x - .5) ** 2 + (y - .5) ** 2))),
     70, 65, (8, 2), [[0.3], [1.5], [4.0]], (0.0, 1.0, 0.0, 1.0)),
    # nx a multiple of the chunk width: the TMA bulk-copy staging, with inflow on all sides and a ragged top band
    ("bulk_inflow_ragged", lambda m: prob2d_const(m, 0.6, 1.4, lambda x, y: 0.5 + x * y, inflow_left=0.9,
                                                  inflow_bottom=0.4, inflow_right=0.6, inflow_top=0.1),
     44, 37, (8, 4), [[]], (0.0, 1.0, 0.0, 0.8)),
]


@pytest.mark.parametrize("name,fn,nx,ny,cl,mus,ext", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_2d_operator_parity(name, fn, nx, ny, cl, mus, ext):
    osys, batch = pair_2d(fn, nx, ny, cl, mus, ext)
    rng = np.random.default_rng(21)
    rho = rng.uniform(-1, 1, (len(mus), osys[0].n_dof()))
    L = batch.apply_L(rho).cpu().numpy()
    B = batch.assemble_rhs().cpu().numpy()
    F = batch.fixed_point(rho).cpu().numpy()
    for s, o in enumerate(osys):
        lo, bo = o.apply_L(rho[s]), o.assemble_rhs()
        assert rel_l2(L[s], lo) < SWEEP_TOL
        assert rel_l2(B[s], bo) < SWEEP_TOL
        assert rel_l2(F[s], lo + bo) < SWEEP_TOL
    for j in (0, 3, osys[0].quad.n() - 1):
        f = batch.sweep_direction(j, rho).cpu().numpy()
        for s, o in enumerate(osys):
            assert rel_l2(f[s], o.sweep_direction(j, rho[s])) < SWEEP_TOL


def test_2d_si_solve_parity():
    name, fn, nx, ny, cl, mus, ext = CASES_2D[0]
    osys, batch = pair_2d(fn, nx, ny, cl, mus, ext)
    R = rte()
    rho, reps = R.sisa_solve(batch, "SI", R.SolveConfig(eps_sisa=1e-10))
    o_rho, o_rep = ro.sisa_solve(osys[0], None, ro.SolveConfig(eps_sisa=1e-10))
    assert reps[0].iterations == o_rep.iterations
    assert rel_l2(rho.cpu().numpy()[0], o_rho) < CONV_TOL


def test_2d_sweep_is_deterministic():
    name, fn, nx, ny, cl, mus, ext = CASES_2D[2]
    _, batch = pair_2d(fn, nx, ny, cl, mus, ext)
    rho = np.random.default_rng(1).uniform(0, 1, (len(mus), batch.n_dof()))
    a = batch.fixed_point(rho).cpu().numpy()
    b = batch.fixed_point(rho).cpu().numpy()
    assert np.array_equal(a, b)


DSA_CASES_2D = CASES_2D + [
    ("c3_32", lambda m: prob2d_const(m, 10 * 0.001, 10 * 0.999, lambda x, y: 1.0), 32, 32, (16, 8), [[]],
     (0.0, 1.0, 0.0, 1.0)),
    ("thin_random_32", None, 32, 32, (8, 4), [[]], (0.0, 1.0, 0.0, 1.0)),
    # 48 x 40 -> 24 x 20 -> 12 x 10 -> 6 x 5: the coarsest level (30 cells) cannot
    # coarsen further and is smoothed instead of solved densely
    ("partial_coarsening_48x40", lambda m: prob2d_const(m, 0.05, 2.0, lambda x, y: 1.0 + y, inflow_bottom=0.3),
     48, 40, (8, 4), [[]], (0.0, 1.2, 0.0, 1.0)),
]


def _thin_random(mod, nx=32):
    rng = np.random.default_rng(5)
    st = np.exp(np.log(0.1) + (np.log(100.0) - np.log(0.1)) * rng.uniform(size=(nx, nx))) * nx / 1024
    c = 0.5 + 0.49 * rng.uniform(size=(nx, nx))

    def idx(x, y):
        ix = np.clip(np.floor(np.asarray(x) * nx).astype(int), 0, nx - 1)
        iy = np.clip(np.floor(np.asarray(y) * nx).astype(int), 0, nx - 1)
        return iy, ix
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: ((1 - c) * st)[idx(x, y)],
                             scattering_weight=lambda x, y: (c * st)[idx(x, y)])
    return mod.ProblemDefinition(mod.XY2D, [t0], lambda x, y: 1.0)


def _dsa_case(case):
    name, fn, nx, ny, cl, mus, ext = case
    if fn is None:
        fn = _thin_random
    return pair_2d(fn, nx, ny, cl, mus, ext)


@pytest.mark.parametrize("case", DSA_CASES_2D, ids=[c[0] for c in DSA_CASES_2D])
def test_2d_dsa_parity(case):
    osys, batch = _dsa_case(case)
    R = rte()
    dsa = R.DsaOperator(batch)
    assert dsa.coupled_dim() == 3 * osys[0].n_dof()
    rhs = np.random.default_rng(9).uniform(-1, 1, (len(osys), osys[0].n_dof()))
    x = dsa.solve_density(rhs).cpu().numpy()
    assert dsa.last_iterations() > 0  # first solve starts from zero
    # the correction's right-hand side Ms rhs is a multiple of rhs for a constant
    # sigma_s, so the warm start (previous solution scaled) may already converge
    c = dsa.correct(rhs).cpu().numpy()
    for s, o in enumerate(osys):
        od = ro.build_dsa(o)
        assert rel_l2(x[s], od.solve_density(rhs[s])) < 1e-9
        assert rel_l2(c[s], od.correct(rhs[s])) < 1e-9


@pytest.mark.parametrize("case", [DSA_CASES_2D[0], DSA_CASES_2D[3]], ids=["box_inflow", "c3_32"])
def test_2d_dsa_solve_parity(case):
    osys, batch = _dsa_case(case)
    R = rte()
    eps = 1e-10
    rho, reps = R.sisa_solve(batch, "DSA", R.SolveConfig(eps_sisa=eps, max_iters=500))
    o_rho, o_rep = ro.sisa_solve(osys[0], ro.DsaStrategy(ro.build_dsa(osys[0])), ro.SolveConfig(eps_sisa=eps,
                                                                                              max_iters=500))
    assert reps[0].converged and o_rep.converged
    assert reps[0].iterations == o_rep.iterations, (reps[0].iterations, o_rep.iterations)
    assert rel_l2(rho.cpu().numpy()[0], o_rho) < CONV_TOL
    np.testing.assert_allclose(reps[0].change_history, o_rep.change_history, rtol=1e-5, atol=1e-13)


def _pin_cell_case(nx=32, n=6):
    from paper_2402_10488_b200 import configs
    _, mus = configs.c4_params(0, n)
    make = configs.pin_cell
    return pair_2d(lambda m: make(m)(nx), nx, nx, (16, 8), mus)


@pytest.mark.parametrize("case", ["c3_32", "thin_random_32", "pin_cell_32x6"])
@pytest.mark.parametrize("inner", [1e-2, 1e-3])
def test_2d_dsa_inner_tolerance(case, inner):
    """rte_si_config.dsa_inner (SPEC.md:174 inner tolerance 1e-2 eps_SISA):
    each correction solved to relative residual inner * eps / change.  Outer
    iteration counts equal the oracle's exact (SuperLU) DSA and the converged
    flux is within the 1e-8 bar."""
    if case == "pin_cell_32x6":
        osys, batch = _pin_cell_case()
    else:
        osys, batch = _dsa_case([c for c in DSA_CASES_2D if c[0] == case][0])
    R = rte()
    eps = 1e-8
    cfg = R.SolveConfig(eps_sisa=eps, max_iters=500, dsa_inner=inner)
    rho, reps = R.sisa_solve(batch, "DSA", cfg)
    rho = rho.cpu().numpy()
    for s, o in enumerate(osys):
        o_rho, o_rep = ro.sisa_solve(o, ro.DsaStrategy(ro.build_dsa(o)), ro.SolveConfig(eps_sisa=eps, max_iters=500))
        assert reps[s].converged and o_rep.converged
        assert reps[s].iterations == o_rep.iterations, (s, reps[s].iterations, o_rep.iterations)
        assert rel_l2(rho[s], o_rho) < CONV_TOL
        np.testing.assert_allclose(reps[s].change_history, o_rep.change_history, rtol=1e-2, atol=1e-13)


@pytest.mark.parametrize("case", ["c3_32", "partial_coarsening_48x40"])
def test_2d_dsa_coarse_cycle_kernel_is_bitwise_identical(case, monkeypatch):
    """k_coarse_cycle (the levels <= RTE_DSA_CTA_CELLS cells in one CTA per
    sample) performs the per-level kernels' arithmetic in the same order."""
    R = rte()
    c = [c for c in DSA_CASES_2D if c[0] == case][0]
    rhs = np.random.default_rng(4).uniform(-1, 1, (len(c[5]), _dsa_case(c)[0][0].n_dof()))
    out = []
    for cells in ("0", "1024"):
        monkeypatch.setenv("RTE_DSA_CTA_CELLS", cells)
        _, batch = _dsa_case(c)
        d = R.DsaOperator(batch)
        out.append((d.solve_density(rhs).cpu().numpy(), d.last_iterations()))
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])


def test_2d_dsa_history_warm_start():
    """The warm start is the minimal-residual combination of the sample's
    previous solutions: a repeated right-hand side and a linear combination of
    earlier ones start (nearly) converged, and every solve still matches the
    oracle's SuperLU solution."""
    R = rte()
    osys, batch = _dsa_case(DSA_CASES_2D[3])  # c3_32, one sample
    d = R.DsaOperator(batch)
    od = ro.build_dsa(osys[0])
    rng = np.random.default_rng(11)
    b1, b2 = (rng.uniform(-1, 1, (1, osys[0].n_dof())) for _ in range(2))
    x1 = d.solve_density(b1).cpu().numpy()
    n1 = d.last_iterations()
    x2 = d.solve_density(b2).cpu().numpy()
    assert n1 > 0 and d.last_iterations() > 0
    x1b = d.solve_density(b1).cpu().numpy()
    assert d.last_iterations() <= 1
    b3 = 0.3 * b1 - 2.0 * b2
    x3 = d.solve_density(b3).cpu().numpy()
    assert d.last_iterations() <= 1
    for b, x in ((b1, x1), (b2, x2), (b1, x1b), (b3, x3)):
        assert rel_l2(x[0], od.solve_density(b[0])) < 1e-9


def test_2d_sweep_rejects_misaligned_vectors():
    """The sweep stages its operands with 16-byte copies (TMA bulk / cp.async):
    a device vector that is not 16-byte aligned is an invalid argument, not a
    device fault."""
    import torch
    from paper_2402_10488_b200 import capi
    name, fn, nx, ny, cl, mus, ext = CASES_2D[3]
    _, batch = pair_2d(fn, nx, ny, cl, mus, ext)
    buf = torch.zeros(batch.S * batch.nd + 1, dtype=torch.float64, device="cuda")
    out = torch.zeros(batch.S * batch.nd, dtype=torch.float64, device="cuda")
    with pytest.raises(capi.RteError, match="aligned"):
        batch._call(capi.load().rte_apply_L, buf.data_ptr() + 8, out.data_ptr(), batch._stream())
    batch._call(capi.load().rte_apply_L, buf.data_ptr(), out.data_ptr(), batch._stream())  # aligned: fine
    torch.cuda.synchronize()
