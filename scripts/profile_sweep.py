"""Small C5-shaped sweep run for ncu captures: python scripts/profile_sweep.py NX S ITERS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2402_10488_b200 import configs, rte

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
it = int(sys.argv[3]) if len(sys.argv) > 3 else 3
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
quad = rte.chebyshev_legendre(32, 16)
st, ss = configs.c5_coefficients(nx, S)
px, py = mesh.cell_points()
g = mesh.project(np.ones(px.size))
b = rte.TransportBatch.from_cells(mesh, quad, st, ss, g)
rho = torch.zeros(S, b.n_dof(), dtype=torch.float64, device="cuda")
for _ in range(it):
    rho = b.fixed_point(rho)
torch.cuda.synchronize()
print("ok", float(rho.sum()))
