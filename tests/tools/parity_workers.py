"""Oracle worker processes for the full-size parity tests
(tests/test_gpu_fullsize_parity.py) and the CPU time-to-tolerance baseline
(bench.py).  Test infrastructure: each call builds the oracle system of ONE
parameter sample and runs the reference's solves on it (sisa.cpp:14-54 with
DsaStrategy / romig + DSA / RomsadStrategy), timing each stage."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _model(ro, d):
    if d is None:
        return None
    return ro.ReducedModel(d["geometry"], d["n_v"], d["n_dof"], d["rank"], d["k_affine"], d["kind"], d["eps_pod"],
                           d["eps_train"], d["u_rho"], d["u_iso"], d["a_r"], d["singular_values"],
                           d["discarded_fraction"], d["b_r"])


def model_dict(m):
    """rte.ReducedModel (device-built) -> picklable dict for the oracle."""
    return {k: getattr(m, k) for k in ("geometry", "n_v", "n_dof", "rank", "k_affine", "kind", "eps_pod", "eps_train",
                                       "u_rho", "u_iso", "a_r", "singular_values", "discarded_fraction", "b_r")}


def system(ro, config, mu):
    from paper_2402_10488_b200 import configs
    if config == "c2":
        m = ro.Mesh.slab_uniform(0.0, 1.0, 256)
        return ro.TransportSystem(configs.two_region_slab(ro), m, ro.build_dg_space(m), ro.gauss_legendre(16), mu)
    if config == "c4":
        m = ro.Mesh.rect_uniform(0, 1, 128, 0, 1, 128)
        return ro.TransportSystem(configs.pin_cell(ro)(128), m, ro.build_dg_space(m), ro.chebyshev_legendre(16, 8),
                                  mu)
    raise ValueError(config)


def solve_sample(job):
    """job = (config, mu, methods, eps, norm, theta, eps_romsad, primary, correction, keep_rho).
    Returns {method: {...report..., 'rho', 'seconds'}, 'setup_seconds': ...}."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np  # noqa: F401
    from oracle import rte_oracle as ro
    config, mu, methods, eps, norm, theta, eps_r, primary, correction, keep_rho = job
    t0 = time.perf_counter()
    s = system(ro, config, mu)
    t_sys = time.perf_counter() - t0
    t0 = time.perf_counter()
    d = ro.build_dsa(s)
    t_dsa = time.perf_counter() - t0
    pm, cm = _model(ro, primary), _model(ro, correction)
    out = {"setup_seconds": t_sys + t_dsa, "system_seconds": t_sys, "dsa_setup_seconds": t_dsa}
    for meth in methods:
        t0 = time.perf_counter()
        cfg = ro.SolveConfig(eps_sisa=eps, norm=norm, max_iters=500)
        if meth == "DSA":
            strat = ro.DsaStrategy(d)
        elif meth == "ROMIG":
            strat = ro.DsaStrategy(d)
            cfg.initial_guess = ro.romig(pm, s)
        elif meth == "ROMSAD":
            strat = ro.RomsadStrategy(cm, d, theta, eps_r)
        else:
            raise ValueError(meth)
        rho, rep = ro.sisa_solve(s, strat, cfg)
        dt = time.perf_counter() - t0
        out[meth] = {"iterations": rep.iterations, "n_sweep": rep.n_sweep, "converged": rep.converged,
                     "log": rep.correction_log, "history": list(rep.change_history), "seconds": dt,
                     "rho": rho if keep_rho else None}
    return out
