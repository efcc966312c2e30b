"""Parity of the production 2D sweep plans against the oracle (SURVEY
s8(a) A2/A4/A5; reference transport_system.cpp:312-363 sweep, :393-404
apply_L, :406-418 assemble_rhs).

The XY sweep kernel is instantiated per "directions per lane" D (sweep2d.cu):
the C5 stress config (1024^2, CL(32,16), 16 samples) runs D = 8, the C3/C4
configs (CL(16,8)) D = 2, small single-sample problems D = 1.  Each plan is
forced here on C5-distributed coefficients (per-cell sigma_t ~ logU[0.1,100],
c ~ U[0.5,0.99]) and compared with the oracle at the north_star per-sweep
tolerance, and one full 1024^2 C5 sample is compared through the production
plan itself.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from paper_2402_10488_b200 import configs
from tests.problems import rel_l2

pytestmark = pytest.mark.gpu

SWEEP_TOL = 1e-10


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def oracle_cells(nx, cl, st, ss, inflow=(0.0, 0.0, 0.0, 0.0)):
    """Oracle TransportSystem with per-cell constant coefficients."""
    return ro.cell_constant_system(nx, nx, st, ss, ro.chebyshev_legendre(*cl), inflow=inflow)


def device_cells(nx, cl, st, ss, inflow=(0, 0, 0, 0)):
    R = rte()
    mesh = R.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    px, _ = mesh.cell_points()
    g = mesh.project(np.ones(px.size))
    return R.TransportBatch.from_cells(mesh, R.chebyshev_legendre(*cl), st, ss, g, inflow=inflow)


PLANS = [(8, (32, 16)), (4, (32, 16)), (2, (32, 16)), (2, (16, 8)), (1, (16, 8))]


@pytest.mark.parametrize("dpl,cl", PLANS, ids=["D%d_CL%d_%d" % (d, *c) for d, c in PLANS])
def test_forced_sweep_plan_parity(monkeypatch, dpl, cl):
    """apply_L, assemble_rhs (with inflow on all four sides) and the fused
    fixed point of every forced plan, 64^2, 4 samples, vs the oracle."""
    monkeypatch.setenv("RTE_SWEEP_DPL", str(dpl))
    nx, S = 64, 4
    st, ss = configs.c5_coefficients(nx, S, seed=configs.SEEDS["c5"] + 7)
    inflow = (0.7, 0.2, 0.4, 1.1)
    batch = device_cells(nx, cl, st, ss, inflow)
    assert batch.sweep_plan()[0] == dpl
    rho = np.random.default_rng(dpl).uniform(-1, 1, (S, batch.n_dof()))
    L = batch.apply_L(rho).cpu().numpy()
    B = batch.assemble_rhs().cpu().numpy()
    F = batch.fixed_point(rho).cpu().numpy()
    for s in range(S):
        o = oracle_cells(nx, cl, st[s], ss[s], inflow)
        lo, bo = o.apply_L(rho[s]), o.assemble_rhs()
        assert rel_l2(L[s], lo) < SWEEP_TOL, (s, rel_l2(L[s], lo))
        assert rel_l2(B[s], bo) < SWEEP_TOL, (s, rel_l2(B[s], bo))
        assert rel_l2(F[s], lo + bo) < SWEEP_TOL


@pytest.mark.parametrize("dpl,cl", [(8, (32, 16)), (2, (16, 8))], ids=["D8", "D2"])
def test_forced_plan_kinetic_sweep_parity(monkeypatch, dpl, cl):
    """The kinetic store (f of both +/-vz directions of each slot) of the
    production plans vs the oracle's kinetic_sweep (transport_system.cpp:420-431)."""
    monkeypatch.setenv("RTE_SWEEP_DPL", str(dpl))
    nx, S = 48, 2
    st, ss = configs.c5_coefficients(nx, S, seed=configs.SEEDS["c5"] + 11)
    batch = device_cells(nx, cl, st, ss)
    rho = np.random.default_rng(5).uniform(0, 1, (S, batch.n_dof()))
    f = batch.kinetic_sweep(rho).cpu().numpy()
    for s in range(S):
        fo = oracle_cells(nx, cl, st[s], ss[s]).kinetic_sweep(rho[s])
        assert rel_l2(f[s], fo) < SWEEP_TOL


def test_production_plan_selection():
    """The plans the configs actually run: C5 (1024^2, CL(32,16), 16
    samples) D = 8 in one group per quadrant; C4 (128^2, CL(16,8), 64
    samples) D = 2; C3 (256^2, CL(16,8), 1 sample) D = 1."""
    for nx, cl, S, want in ((1024, (32, 16), 16, 8), (128, (16, 8), 64, 2), (256, (16, 8), 1, 1)):
        st = np.full((S, nx * nx), 10.0)
        b = device_cells(nx, cl, st, 0.999 * st)
        assert b.sweep_plan()[0] == want, (nx, cl, S, b.sweep_plan())
        del b


@pytest.mark.slow
def test_c5_full_sample_operator_parity():
    """One full C5 sample (1024^2 cells, 256 unique directions of CL(32,16))
    through the production D = 8 plan of the 16-sample batch: apply_L and
    assemble_rhs of samples 0 and 15 vs the oracle (uncached slot-major
    sweep: the reference's per-slot inverse cache would be 34 GB)."""
    nx, S = 1024, 16
    st, ss = configs.c5_coefficients(nx, S)
    batch = device_cells(nx, (32, 16), st, ss)
    assert batch.sweep_plan() == (8, 1)
    rng = np.random.default_rng(42)
    rho = rng.uniform(0.0, 1.0, (S, batch.n_dof()))
    L = batch.apply_L(rho).cpu().numpy()
    B = batch.assemble_rhs().cpu().numpy()
    del batch
    for s in (0, S - 1):
        o = oracle_cells(nx, (32, 16), st[s], ss[s])
        assert not o.is_cached()
        assert rel_l2(L[s], o.apply_L(rho[s])) < SWEEP_TOL
        assert rel_l2(B[s], o.assemble_rhs()) < SWEEP_TOL
