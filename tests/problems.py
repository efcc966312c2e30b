"""Shared test problems, built identically for the oracle (oracle.rte_oracle)
and the B200 host API (paper_2402_10488_b200.rte): both expose the
reference's ProblemDefinition / CoefficientTerm / Mesh / quadrature names."""
import numpy as np


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


def two_region_slab(mod):
    """BASELINE configs[1]: x<0.5: sigma_t = 1/eps, x>=0.5: sigma_t = 1; c = mu[1];
    q = 1 on the left half (SURVEY s8(d) C2 affine terms)."""
    chiL = lambda x, y: np.where(np.asarray(x) < 0.5, 1.0, 0.0)
    chiR = lambda x, y: np.where(np.asarray(x) < 0.5, 0.0, 1.0)
    terms = [
        mod.CoefficientTerm(absorption_weight=chiR, name="right total"),
        mod.CoefficientTerm(psi=lambda mu: mu[1], absorption_weight=lambda x, y: -chiR(x, y),
                            scattering_weight=chiR, name="right scattering"),
        mod.CoefficientTerm(psi=lambda mu: 1.0 / mu[0], absorption_weight=chiL, name="left total"),
        mod.CoefficientTerm(psi=lambda mu: mu[1] / mu[0], absorption_weight=lambda x, y: -chiL(x, y),
                            scattering_weight=chiL, name="left scattering"),
    ]
    return mod.ProblemDefinition(mod.SLAB1D, terms, chiL, n_params=2, param_ranges=[(1e-3, 1.0), (0.9, 0.9999)])


def prob2d_const(mod, sig_a, sig_s, src, **inflow):
    t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: sig_a, scattering_weight=lambda x, y: sig_s)
    return mod.ProblemDefinition(mod.XY2D, [t0], src, **inflow)


def pin_cell(mod):
    """BASELINE configs[3] affine structure: pin = centroid
    within r <= 0.3 of (0.5, 0.5).  The closures classify a point by its
    cell's centroid, so coefficients are constant per cell (nx given)."""
    def make(nx):
        h = 1.0 / nx

        def chiP(x, y):
            cx = (np.floor(np.asarray(x) / h) + 0.5) * h
            cy = (np.floor(np.asarray(y) / h) + 0.5) * h
            return np.where((cx - 0.5) ** 2 + (cy - 0.5) ** 2 <= 0.09, 1.0, 0.0)

        chiM = lambda x, y: 1.0 - chiP(x, y)
        terms = [
            mod.CoefficientTerm(name="floor"),
            mod.CoefficientTerm(psi=lambda mu: mu[0], absorption_weight=chiP, name="pin total"),
            mod.CoefficientTerm(psi=lambda mu: mu[2] * mu[0], absorption_weight=lambda x, y: -chiP(x, y),
                                scattering_weight=chiP, name="pin scattering"),
            mod.CoefficientTerm(psi=lambda mu: 1.0 / mu[1], absorption_weight=chiM, name="moderator total"),
            mod.CoefficientTerm(psi=lambda mu: mu[2] / mu[1], absorption_weight=lambda x, y: -chiM(x, y),
                                scattering_weight=chiM, name="moderator scattering"),
        ]
        return mod.ProblemDefinition(mod.XY2D, terms, chiP, n_params=3,
                                     param_ranges=[(1.0, 10.0), (1e-3, 1e-1), (0.9, 0.9999)])
    return make


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
