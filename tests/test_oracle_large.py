"""The oracle's large-problem paths (test infrastructure checks, CPU only):
the uncached slot-major sweep used above the inverse-cache budget (C5 needs
34 GB of per-slot inverses per sample, transport_system.cpp:189-261) and the
nested-dissection ordering of the 2D DSA direct solve agree with the
reference-ordered paths."""
import numpy as np

from oracle import rte_oracle as ro
from tests.problems import prob2d_const, rel_l2


def _system(nx, ny, cl=(8, 4), inflow=True):
    kw = dict(inflow_left=1.0, inflow_bottom=0.5, inflow_top=0.2) if inflow else {}
    fn = prob2d_const(ro, 0.3, 0.9, lambda x, y: 1.0 + x * y, **kw)
    m = ro.Mesh.rect_uniform(0.0, 1.0, nx, 0.0, 1.3, ny)
    return ro.TransportSystem(fn, m, ro.build_dg_space(m), ro.chebyshev_legendre(*cl), [])


def test_uncached_sweep_matches_cached():
    cached = _system(13, 11)
    try:
        ro.set_cache_budget(0)
        lazy = _system(13, 11)
    finally:
        ro.set_cache_budget(4e9)
    assert cached.is_cached() and not lazy.is_cached()
    rho = np.random.default_rng(2).uniform(-1, 1, cached.n_dof())
    # per-direction sweeps: identical arithmetic (same operands, same inverse)
    for j in (0, 5, 31):
        assert np.array_equal(cached.sweep_direction(j, rho), lazy.sweep_direction(j, rho))
    # L and bbar: slot-major accumulation, differs only in the order of additions
    assert rel_l2(lazy.apply_L(rho), cached.apply_L(rho)) < 1e-14
    assert rel_l2(lazy.assemble_rhs(), cached.assemble_rhs()) < 1e-14


def test_apply_L_dirs_sums_to_apply_L():
    s = _system(9, 7, inflow=False)
    rho = np.random.default_rng(3).uniform(0, 1, s.n_dof())
    n = s.quad.n()
    parts = s.apply_L_dirs(rho, 0, n // 2) + s.apply_L_dirs(rho, n // 2, n)
    assert rel_l2(parts, s.apply_L(rho)) < 1e-14


def test_nested_dissection_order_is_a_permutation():
    cells = ro.nested_dissection_cells(37, 23)
    assert np.array_equal(np.sort(cells), np.arange(37 * 23))


def test_dsa_nested_dissection_solve_matches_colamd():
    s = _system(24, 20)
    d = ro.build_dsa(s)
    rhs = np.random.default_rng(4).uniform(-1, 1, s.n_dof())
    x = d.solve_density(rhs)
    full = np.zeros(d.coupled_dim())
    full[: s.n_dof()] = rhs
    ref = ro._splu(d.coupled).solve(full)[: s.n_dof()]
    assert rel_l2(x, ref) < 1e-12
