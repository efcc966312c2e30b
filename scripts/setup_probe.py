"""Online setup breakdown (setup counts in time to tolerance)
for BASELINE configs[1..3]: host system assembly (closures, weighted_mass,
projection, psi combination), rte_create (upload), DSA setup, ROM upload.

  python scripts/setup_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2402_10488_b200 import capi, configs, rte
from tests.problems import homog


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def probe(name, prob, mesh, quad, mus):
    b, tb = t(lambda: rte.TransportBatch(prob, mesh, quad, mus))
    _, td = t(lambda: rte.DsaOperator(b))
    print("%-6s S=%4d  TransportBatch %.1f ms, DsaOperator %.1f ms" % (name, len(mus), tb * 1e3, td * 1e3), flush=True)
    return b


torch.zeros(1, device="cuda")
for rep in range(2):
    train, test = configs.c2_params(32, 512)
    probe("C2", configs.two_region_slab(rte), rte.Mesh.slab_uniform(0.0, 1.0, 256), rte.gauss_legendre(16), test)
    probe("C3", homog(rte, rte.XY2D, 10.0 * (1 - 0.999), 10.0 * 0.999, 1.0), rte.Mesh.rect_uniform(0, 1, 256, 0, 1, 256),
          rte.chebyshev_legendre(16, 8), [[]])
    train, test = configs.c4_params(40, 64)
    probe("C4", configs.pin_cell(rte)(128), rte.Mesh.rect_uniform(0, 1, 128, 0, 1, 128), rte.chebyshev_legendre(16, 8),
          test)
