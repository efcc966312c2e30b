"""The CorrectionStrategy plugin point (solvers.hpp:38-51) on the device loop
(RTE_CUSTOM): caller strategies see rho* - rho and return corrections and
kind letters per sample, as the reference's test stubs do.

* ZeroCorrection (test_solvers.cpp:30-62): reproduces plain SI bitwise, log
  'Z' x (iterations - 1), label "ZERO".
* A strategy that applies the device DSA operator reproduces the built-in
  DSA method bitwise (same kernels, same order).
* Exact correction (acceptance.cpp:230-285): the oracle's exact kinetic
  correction, computed on the host per sample, converges in <= 2 iterations.
* A failing callback aborts the solve with the callback's exception.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import rel_l2, two_region_slab
from tests.test_gpu_parity import pair_1d, pair_2d

pytestmark = pytest.mark.gpu


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


class Zero:
    def setup(self, batch):
        pass

    def correct(self, l, delta, active, out):
        out.zero_()
        return ["Z" if a else "" for a in active]

    def label(self):
        return "ZERO"


class DeviceDsa:
    def setup(self, batch):
        self.dsa = rte().DsaOperator(batch)

    def correct(self, l, delta, active, out):
        out.copy_(self.dsa.correct(delta))
        return ["D" if a else "" for a in active]

    def label(self):
        return "DSA"


MUS = [[1e-3, 0.95], [0.2, 0.9999], [1.0, 0.9]]


def test_zero_correction_reproduces_si_bitwise():
    R = rte()
    osys, batch = pair_1d(two_region_slab, np.linspace(0, 1, 65), 8, MUS)
    cfg = R.SolveConfig(eps_sisa=1e-10, max_iters=20000)
    rho_si, rep_si = R.sisa_solve(batch, "SI", cfg)
    strat = Zero()
    rho_z, rep_z = R.sisa_solve(batch, strat, cfg)
    assert rep_z[0].strategy == "ZERO"
    for a, b in zip(rep_si, rep_z):
        assert a.iterations == b.iterations and a.n_sweep == b.n_sweep and a.converged == b.converged
        assert a.change_history == b.change_history
        assert b.correction_log == "Z" * (b.iterations - 1) and a.correction_log == ""
    assert np.array_equal(rho_si.cpu().numpy(), rho_z.cpu().numpy())


@pytest.mark.parametrize("geom", ["1d", "2d"])
def test_plugin_dsa_matches_builtin_dsa(geom):
    R = rte()
    if geom == "1d":
        osys, batch = pair_1d(two_region_slab, np.linspace(0, 1, 129), 16, MUS)
    else:
        from tests.problems import prob2d_const
        osys, batch = pair_2d(lambda m: prob2d_const(m, 0.2, 3.0, lambda x, y: 1.0), 16, 16, (8, 4), [[]])
    cfg = R.SolveConfig(eps_sisa=1e-9)
    rho_b, rep_b = R.sisa_solve(batch, "DSA", cfg)
    rho_p, rep_p = R.sisa_solve(batch, DeviceDsa(), cfg)
    for a, b in zip(rep_b, rep_p):
        assert a.iterations == b.iterations and a.correction_log == b.correction_log
        assert a.change_history == b.change_history
        assert a.switch_iter == b.switch_iter
    assert np.array_equal(rho_b.cpu().numpy(), rho_p.cpu().numpy())


class HostExact:
    """acceptance.cpp:230-255: exact correction of the kinetic error, on the host."""

    def __init__(self, osys):
        self.osys = osys
        self.A = [o.materialize_kinetic() for o in osys]

    def setup(self, batch):
        pass

    def correct(self, l, delta, active, out):
        import torch
        d = delta.cpu().numpy()
        res = np.zeros_like(d)
        for s, o in enumerate(self.osys):
            if active[s]:
                rhs = np.tile(o.apply_Ms(d[s]), o.quad.n())
                res[s] = o.density_of(np.linalg.solve(self.A[s], rhs))
        out.copy_(torch.from_numpy(res))
        return ["X" if a else "" for a in active]

    def label(self):
        return "EXACT"


def test_exact_correction_converges_in_two_steps():
    R = rte()
    osys, batch = pair_1d(two_region_slab, np.linspace(0, 1, 17), 4, MUS)
    cfg = R.SolveConfig(eps_sisa=1e-11, max_iters=20000)
    rho_si, rep_si = R.sisa_solve(batch, "SI", cfg)
    rho_x, rep_x = R.sisa_solve(batch, HostExact(osys), cfg)
    for s in range(len(MUS)):
        assert rep_x[s].converged and rep_x[s].iterations <= 2 < rep_si[s].iterations
        o_rho, _ = ro.sisa_solve(osys[s], None, ro.SolveConfig(eps_sisa=1e-13, max_iters=100000))
        assert rel_l2(rho_x.cpu().numpy()[s], o_rho) < 1e-8


class Failing:
    def setup(self, batch):
        pass

    def correct(self, l, delta, active, out):
        raise ValueError("strategy failed at iteration %d" % l)

    def label(self):
        return "FAIL"


def test_failing_callback_propagates():
    R = rte()
    osys, batch = pair_1d(two_region_slab, np.linspace(0, 1, 17), 4, MUS[:1])
    with pytest.raises(ValueError, match="strategy failed at iteration 1"):
        R.sisa_solve(batch, Failing(), R.SolveConfig(eps_sisa=1e-10))
