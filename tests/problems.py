"""Shared test problems, built identically for the oracle (oracle.rte_oracle)
and the B200 host API (paper_2402_10488_b200.rte): both expose the
reference's ProblemDefinition / CoefficientTerm / Mesh / quadrature names."""
import numpy as np

from paper_2402_10488_b200.configs import pin_cell, two_region_slab  # noqa: F401 (BASELINE configs[1], [3])


def homog(mod, geom, sig_a, sig_s, src, **inflow):
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: sig_a, scattering_weight=lambda x, y: sig_s)
    return mod.ProblemDefinition(geom, [t0], lambda x, y: src, **inflow)


def prob1d(mod):  # test_assembly.cpp:11-22 (intra-cell varying sigma_s, inflow both sides)
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.3, scattering_weight=lambda x, y: 0.6 + 0.1 * x)
    return mod.ProblemDefinition(mod.SLAB1D, [t0], lambda x, y: 1.0 + x, inflow_left=2.0, inflow_right=0.5)


def parametric_slab(mod):  # test_rom.cpp:12-31
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: 0.2, scattering_weight=lambda x, y: 0.5)
    t1 = mod.CoefficientTerm(psi=lambda mu: mu[0], scattering_weight=lambda x, y: 0.3)
    return mod.ProblemDefinition(mod.SLAB1D, [t0, t1], lambda x, y: 1.0, inflow_left=0.3, n_params=1,
                                 param_ranges=[(0.0, 1.0)])


def prob2d_const(mod, sig_a, sig_s, src, **inflow):
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: sig_a, scattering_weight=lambda x, y: sig_s)
    return mod.ProblemDefinition(mod.XY2D, [t0], src, **inflow)


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
