"""Failure detection of the iterative XY DSA (the reference's direct SparseLU
throws when it fails, dsa.cpp:253-256, 269-271) and independence of a solve
from earlier calls (the warm-start history is cleared when a solve starts)."""
import numpy as np
import pytest

from tests.problems import prob2d_const

pytestmark = pytest.mark.gpu


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def batch(nx=24, mus=([],)):
    R = rte()
    m = R.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    return R.TransportBatch(prob2d_const(R, 0.01, 0.99, lambda x, y: 1.0), m, R.chebyshev_legendre(8, 4),
                            [list(x) for x in mus])


def test_direct_solve_reports_iteration_cap():
    from paper_2402_10488_b200 import capi
    b = batch()
    d = rte().DsaOperator(b)
    d.set_tolerance(1e-15, 2)
    rhs = np.random.default_rng(1).uniform(-1, 1, (1, b.n_dof()))
    with pytest.raises(capi.RteError, match="iteration cap"):
        d.solve_density(rhs)
    d.set_tolerance(1e-12, 1000)
    d.solve_density(rhs)  # a converging solve succeeds again


def test_si_solve_fails_loudly_with_per_sample_status():
    from paper_2402_10488_b200 import capi
    R = rte()
    b = batch()
    R.DsaOperator(b).set_tolerance(1e-15, 1)
    with pytest.raises(capi.RteError, match="DSA correction") as ei:
        R.sisa_solve(b, "DSA", R.SolveConfig(eps_sisa=1e-8, max_iters=50))
    assert ei.value.dsa_status == [capi.RTE_DSA_MAXIT]
    R.DsaOperator(b).set_tolerance(1e-12, 1000)
    _, reps = R.sisa_solve(b, "DSA", R.SolveConfig(eps_sisa=1e-8, max_iters=50))
    assert reps[0].converged and reps[0].dsa_status == capi.RTE_DSA_OK


def test_repeated_solves_are_bitwise_identical():
    """The DSA warm start draws on earlier solutions; rte_si_solve clears that
    history first, so repeating a solve repeats it exactly (the reference's
    DsaOperator is stateless)."""
    R = rte()
    b = batch(mus=([], []))
    cfg = R.SolveConfig(eps_sisa=1e-9, max_iters=100)
    r1, p1 = R.sisa_solve(b, "DSA", cfg)
    r2, p2 = R.sisa_solve(b, "DSA", cfg)
    assert np.array_equal(r1.cpu().numpy(), r2.cpu().numpy())
    assert [r.change_history for r in p1] == [r.change_history for r in p2]


def test_fixed_iters_above_max_iters_rejected():
    R = rte()
    with pytest.raises(ValueError):
        R.si_config(R.SolveConfig(fixed_iters=5, max_iters=4), 1)


def test_iteration_log_has_one_entry_per_correction():
    """rte_dsa_iteration_log: the Krylov iteration count of every XY DSA solve
    of the last rte_si_solve, one per SI iteration that applied a correction
    (the converging iteration returns rho* without one, sisa.cpp:36-44).  The
    device loop runs on to the next host poll of the active count
    (check_every); those masked trips log 0."""
    R = rte()
    b = batch(mus=([], []))
    d = R.DsaOperator(b)
    d.set_tolerance(1e-10, 1000)
    _, reps = R.sisa_solve(b, "DSA", R.SolveConfig(eps_sisa=1e-8, max_iters=100))
    log = d.iteration_log()
    its = max(r.iterations for r in reps)
    assert len(log) >= its - 1
    assert all(1 <= v <= 1000 for v in log[:its - 1]) and all(v == 0 for v in log[its - 1:])
    # a second solve starts a new log
    R.sisa_solve(b, "DSA", R.SolveConfig(fixed_iters=3, max_iters=3, compute_residual=False))
    log3 = d.iteration_log()
    assert len(log3) == 3 and all(v >= 1 for v in log3)
