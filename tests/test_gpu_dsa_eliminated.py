"""DsaOperator::apply_eliminated (dsa.cpp:279-293) on the device:
S x = A_rr x - A_rJ T^-1 A_Jr x, with the current block T factored lazily
(slab: block cyclic reduction; XY: CG on the SPD current block).

* the reference's KAT (test_dsa.cpp:49-56, DemoSlab): S inverts
  solve_density to 1e-9;
* agreement with the oracle's SuperLU-based apply_eliminated (1e-12 slab,
  1e-10 XY, sigma-I and full 4x4 blocks), batched over samples;
* linearity, and aliasing rejected like the other operator entry points.
"""
import numpy as np
import pytest

from tests.problems import homog, prob2d_const, rel_l2, two_region_slab
from tests.test_gpu_full_blocks import varying
from tests.test_gpu_parity import pair_1d, pair_2d

pytestmark = pytest.mark.gpu


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def test_eliminated_inverts_solve_density_demo_slab():
    R = rte()
    b = R.TransportBatch(homog(R, R.SLAB1D, 0.0, 1.0, 0.01), R.Mesh.slab_uniform(0, 10, 400),
                         R.gauss_legendre(16), [[]])
    d = R.DsaOperator(b)
    rhs = np.random.default_rng(3).uniform(-1, 1, (1, b.n_dof()))
    drho = d.solve_density(rhs)
    back = d.apply_eliminated(drho).cpu().numpy()
    assert np.max(np.abs(back - rhs)) < 1e-9 * np.max(np.abs(rhs))


def test_eliminated_slab_batch_matches_oracle():
    R = rte()
    mus = [[1e-3, 0.95], [0.2, 0.9999], [1.0, 0.9]]
    osys, batch = pair_1d(two_region_slab, np.linspace(0, 1, 97), 16, mus)
    d = R.DsaOperator(batch)
    x = np.random.default_rng(8).uniform(-1, 1, (len(mus), batch.n_dof()))
    y = d.apply_eliminated(x).cpu().numpy()
    for s, o in enumerate(osys):
        ref = ro_dsa(o).apply_eliminated(x[s])
        assert rel_l2(y[s], ref) < 1e-12
    # linearity
    z = np.random.default_rng(9).uniform(-1, 1, x.shape)
    lhs = d.apply_eliminated(0.3 * x - 2.0 * z).cpu().numpy()
    rhs = 0.3 * y - 2.0 * d.apply_eliminated(z).cpu().numpy()
    assert np.max(np.abs(lhs - rhs)) < 1e-12 * np.max(np.abs(rhs))


def ro_dsa(o):
    from oracle import rte_oracle as ro
    return ro.build_dsa(o)


@pytest.mark.parametrize("case", ["sigma", "full"])
def test_eliminated_xy_matches_oracle(case):
    R = rte()
    if case == "sigma":
        osys, batch = pair_2d(lambda m: prob2d_const(m, 0.2, 1.8, lambda x, y: 1.0), 12, 10, (8, 4), [[]])
    else:
        osys, batch = pair_2d(varying, 9, 11, (8, 4), [[]])
        assert batch._keep[0].shape[-1] == 16
    d = R.DsaOperator(batch)
    x = np.random.default_rng(11).uniform(-1, 1, (1, batch.n_dof()))
    y = d.apply_eliminated(x).cpu().numpy()[0]
    ref = ro_dsa(osys[0]).apply_eliminated(x[0])
    assert rel_l2(y, ref) < 1e-10
    # S inverts the (tight) iterative solve_density
    d.set_tolerance(1e-13, 4000)
    rhs = np.random.default_rng(12).uniform(-1, 1, (1, batch.n_dof()))
    back = d.apply_eliminated(d.solve_density(rhs)).cpu().numpy()
    assert np.max(np.abs(back - rhs)) < 1e-9 * np.max(np.abs(rhs))


def test_eliminated_rejects_aliasing():
    R = rte()
    from paper_2402_10488_b200 import capi
    b = R.TransportBatch(homog(R, R.SLAB1D, 0.5, 0.5, 1.0), R.Mesh.slab_uniform(0, 1, 16), R.gauss_legendre(4), [[]])
    R.DsaOperator(b)
    x = b._dev(np.ones((1, b.n_dof())), (1, b.n_dof()))
    with pytest.raises(capi.RteError):
        b._call(capi.load().rte_dsa_apply_eliminated, x.data_ptr(), x.data_ptr(), b._stream())
