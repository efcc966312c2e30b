"""Warm time-to-tolerance probe of one small config (C1 slab SI-DSA or C3 XY
SI-DSA) for launch-list profiling: builds the problem once, runs the solve
`--reps` times and prints the CUDA-event time of each.

  python scripts/ttt_probe.py c1|c3 [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2402_10488_b200 import rte
from tests.problems import homog


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c1", "c3"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--inner", type=float, default=1e-3)
    a = ap.parse_args()
    if a.config == "c1":
        b = rte.TransportBatch(homog(rte, rte.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0),
                               rte.Mesh.slab_uniform(0.0, 1.0, 256), rte.gauss_legendre(16), [[]])
        cfg = rte.SolveConfig(eps_sisa=1e-8, norm="rel")
    else:
        b = rte.TransportBatch(homog(rte, rte.XY2D, 10.0 * (1 - 0.999), 10.0 * 0.999, 1.0),
                               rte.Mesh.rect_uniform(0, 1, 256, 0, 1, 256), rte.chebyshev_legendre(16, 8), [[]])
        cfg = rte.SolveConfig(eps_sisa=1e-8, norm="rel", dsa_inner=a.inner)
    rte.DsaOperator(b)
    for k in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        _, reps = rte.sisa_solve(b, "DSA", cfg)
        e1.record()
        torch.cuda.synchronize()
        print("%s rep %d: %.3f ms, %d iterations" % (a.config, k, e0.elapsed_time(e1), reps[0].iterations),
              flush=True)


if __name__ == "__main__":
    main()
