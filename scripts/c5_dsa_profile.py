"""C5 (BASELINE configs[4]) SI-DSA step profile: the bench's workload
(3 warm-up iterations, then a fixed number of timed SI-DSA iterations from
that state) with a chosen DSA tolerance rule; prints the per-iteration change
history and device time, saves the final flux for cross-rule comparison.
With RTE_DSA_REPORT=1 the library prints per-solve BiCGStab counts.

  python scripts/c5_dsa_profile.py [--floor C] [--inner-tol T] [--iters K] [--save f.npy]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2402_10488_b200 import configs, rte


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=1024)
    ap.add_argument("--samples", type=int, default=16)
    ap.add_argument("--phi", type=int, default=32)
    ap.add_argument("--vz", type=int, default=16)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--floor", type=float, default=0.0)
    ap.add_argument("--inner-tol", type=float, default=1e-8)
    ap.add_argument("--save", default="")
    a = ap.parse_args()
    mesh = rte.Mesh.rect_uniform(0, 1, a.nx, 0, 1, a.nx)
    quad = rte.chebyshev_legendre(a.phi, a.vz)
    st, ss = configs.c5_coefficients(a.nx, a.samples)
    px, _ = mesh.cell_points()
    b = rte.TransportBatch.from_cells(mesh, quad, st, ss, mesh.project(np.ones(px.size)))
    d = rte.DsaOperator(b)
    d.set_tolerance(a.inner_tol, 2000)

    def solve(k, guess):
        cfg = rte.SolveConfig(fixed_iters=k, max_iters=k, compute_residual=False, initial_guess=guess,
                              check_every=max(k, 1), dsa_floor=a.floor, norm="rel")
        return rte.sisa_solve(b, "DSA", cfg)

    rho, _ = solve(a.warmup, None)
    torch.cuda.synchronize()
    sys.stderr.write("[profile] timed region\n")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rho, reps = solve(a.iters, rho)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    hist = np.array([r.change_history for r in reps])
    out = {"floor": a.floor, "inner_tol": a.inner_tol, "iters": a.iters, "ms_total": ms, "ms_per_iter": ms / a.iters,
           "rel_change_max_per_iter": hist.max(axis=0).tolist(), "rel_change_min_per_iter": hist.min(axis=0).tolist(),
           "dsa_status": [r.dsa_status for r in reps]}
    print(json.dumps(out))
    if a.save:
        np.save(a.save, rho.cpu().numpy())


if __name__ == "__main__":
    main()
