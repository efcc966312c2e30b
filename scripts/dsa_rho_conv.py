"""How fast does the density block of the C5 DSA correction converge compared
with the full (rho, Jx, Jy) residual?  Real SI right-hand side (delta of SI
iteration 2 of the C5 batch), cold start, solves capped at k BiCGStab
iterations vs a 1e-12 reference.  python scripts/dsa_rho_conv.py [NX] [S]"""
import os, sys
os.environ["RTE_DSA_WARM"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_10488_b200 import rte, configs
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
quad = rte.chebyshev_legendre(32, 16)
st, ss = configs.c5_coefficients(nx, S)
g = mesh.project(np.ones(mesh.cell_points()[0].size))
b = rte.TransportBatch.from_cells(mesh, quad, st, ss, g)
d = rte.DsaOperator(b)
rho, _ = rte.sisa_solve(b, "DSA", rte.SolveConfig(fixed_iters=1, max_iters=1, compute_residual=False))
delta = b.fixed_point(rho) - rho
d.set_tolerance(1e-13, 2000)
ref = d.correct(delta).clone()
kref = d.last_iterations()
print("reference: %d iterations" % kref, flush=True)
for k in range(2, kref + 1, 2):
    d.set_tolerance(1e-30, k)
    x = d.correct(delta)
    err = (x - ref).norm(dim=1) / ref.norm(dim=1)
    einf = (x - ref).abs().amax(dim=1) / ref.abs().amax(dim=1)
    print("k=%2d  rho rel L2 err max %.2e  rel inf err max %.2e" % (k, err.max().item(), einf.max().item()), flush=True)
for tol in (1e-4, 1e-6, 1e-8, 1e-10):
    d.set_tolerance(tol, 2000)
    x = d.correct(delta)
    err = (x - ref).norm(dim=1) / ref.norm(dim=1)
    print("tol %.0e: %d its, rho rel L2 err max %.2e" % (tol, d.last_iterations(), err.max().item()), flush=True)
