"""The round-off floor rule of the XY DSA solves (rte_si_config.dsa_floor,
used by the C5 bench): SI iteration l accepts a DSA correction with relative
residual min(0.1, c 2^-53 ||rho*||_inf / ||rho* - rho||_inf) when that is
looser than the DSA tolerance.  Below that accuracy the correction cannot move
the iterate by more than ~c ulps of rho* times its gain, so the iterates are
those of exact DSA corrections to round-off.

Checked on C5-distributed coefficients (configs[4]: per-cell sigma_t ~
logU[0.1,100], c ~ U[0.5,0.99]) with the C5 quadrature CL(32,16), a fixed 20
SI-DSA iterations from zero: the floor rule's fluxes equal the strict rule's
to 1e-13 and the oracle's (exact SuperLU DSA, sisa.cpp:14-54 stopped by
max_iters = 20) to the north_star per-sweep tolerance, the change histories
agree while they are above round-off, and the last solves (noise right-hand
sides) take at most 2 BiCGStab iterations instead of the strict rule's
(DSA tolerance 1e-12 here) many.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from paper_2402_10488_b200 import configs
from tests.problems import rel_l2

pytestmark = pytest.mark.gpu


def test_floor_rule_matches_strict_and_oracle():
    from paper_2402_10488_b200 import rte
    nx, S, K = 64, 2, 20
    st, ss = configs.c5_coefficients(nx, S, seed=configs.SEEDS["c5"] + 11)
    mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    px, _ = mesh.cell_points()
    b = rte.TransportBatch.from_cells(mesh, rte.chebyshev_legendre(32, 16), st, ss, mesh.project(np.ones(px.size)))
    d = rte.DsaOperator(b)
    d.set_tolerance(1e-12, 2000)  # strict enough that noise right-hand sides take many iterations
    out = {}
    for floor in (0.0, 1.0):
        cfg = rte.SolveConfig(fixed_iters=K, max_iters=K, compute_residual=False, dsa_floor=floor)
        rho, reps = rte.sisa_solve(b, "DSA", cfg)
        out[floor] = (rho.cpu().numpy(), reps, d.last_iterations())
    (r0, rep0, it0), (r1, rep1, it1) = out[0.0], out[1.0]
    assert it1 <= 2 < it0, (it1, it0)
    for s in range(S):
        assert rel_l2(r1[s], r0[s]) < 1e-13
        assert rep1[s].dsa_status == 0 and rep1[s].iterations == K
        osys = ro.cell_constant_system(nx, nx, st[s], ss[s], ro.chebyshev_legendre(32, 16))
        rho_o, rep_o = ro.sisa_solve(osys, ro.DsaStrategy(ro.build_dsa(osys)), ro.SolveConfig(eps_sisa=0.0,
                                                                                           max_iters=K))
        assert rep_o.iterations == K and not rep_o.converged
        assert rel_l2(r1[s], rho_o) < 1e-10
        h_o = np.asarray(rep_o.change_history)
        above = h_o > 1e-10 * np.abs(rho_o).max()  # well above the round-off of rho* - rho
        np.testing.assert_allclose(np.asarray(rep1[s].change_history)[above], h_o[above], rtol=1e-5)
