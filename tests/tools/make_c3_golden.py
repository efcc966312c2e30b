"""Full-size C3 golden fixture from the CPU oracle (BASELINE configs[2]:
[0,1]^2 at 256x256 cells, CL(16,8), sigma_t = 10, c = 0.999, q = 1, vacuum,
SI-DSA).  The oracle's exact DSA is a SuperLU factorization of the 786 432-
unknown coupled system (nested-dissection order, ~2-3 min and ~8 GB here), too
slow to repeat inside the GPU test, so the converged flux and the reference
convergence record are stored: tests/golden/c3_full_si_dsa.npz, compared by
tests/test_gpu_fullsize_parity.py.

  python tests/tools/make_c3_golden.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np

from oracle import rte_oracle as ro
from tests.problems import homog


def main():
    nx = 256
    mesh = ro.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    t0 = time.time()
    s = ro.TransportSystem(homog(ro, ro.XY2D, 10 * 0.001, 10 * 0.999, 1.0), mesh, ro.build_dg_space(mesh),
                           ro.chebyshev_legendre(16, 8), [])
    t_sys = time.time() - t0
    t0 = time.time()
    d = ro.build_dsa(s)
    t_dsa = time.time() - t0
    out = {}
    for norm in ("rel", "abs"):
        t0 = time.time()
        rho, rep = ro.sisa_solve(s, ro.DsaStrategy(d), ro.SolveConfig(eps_sisa=1e-8, norm=norm))
        t_solve = time.time() - t0
        out[norm] = (rho, rep, t_solve)
        print(norm, rep.iterations, rep.converged, "%.1f s" % t_solve, flush=True)
    rr, ra = out["rel"], out["abs"]
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3_full_si_dsa.npz"),
                        rho_rel=rr[0], history_rel=np.array(rr[1].change_history), iterations_rel=rr[1].iterations,
                        n_sweep_rel=rr[1].n_sweep, final_residual_rel=rr[1].final_residual,
                        rho_abs=ra[0], history_abs=np.array(ra[1].change_history), iterations_abs=ra[1].iterations,
                        n_sweep_abs=ra[1].n_sweep,
                        oracle_seconds=np.array([t_sys, t_dsa, rr[2], ra[2]]))
    print("system %.1f s, DSA factorization %.1f s" % (t_sys, t_dsa))


if __name__ == "__main__":
    main()
