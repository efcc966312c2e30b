"""BASELINE configs[2] (C3): 256x256, CL(16,8) folded to 64 slots, sigma_t=10,
c=0.999, q=1, vacuum, single sample, SI-DSA to 1e-8 relative change."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
from paper_2402_10488_b200 import rte, capi

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
norm = sys.argv[2] if len(sys.argv) > 2 else "rel"
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
quad = rte.chebyshev_legendre(16, 8)
n = nx * nx
px, py = mesh.cell_points()
g = mesh.project(np.ones(px.size))
b = rte.TransportBatch.from_cells(mesh, quad, np.full((1, n), 10.0), np.full((1, n), 9.99), g)
L = capi.load()
t0 = time.time()
dsa = rte.DsaOperator(b)
torch.cuda.synchronize()
print("dsa setup %.3f s" % (time.time() - t0))
L.rte_profile_enable(b._h, 1)
t0 = time.time()
rho, reps = rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm=norm, max_iters=200))
torch.cuda.synchronize()
t = time.time() - t0
NK = len(capi.PROF_KINDS)  # rte_profile_read writes RTE_PROF_KINDS entries
ms = (ctypes.c_double * NK)(); nk = (ctypes.c_long * NK)()
L.rte_profile_read(b._h, ms, nk)
r = reps[0]
print("C3 %s: converged=%s iterations=%d n_sweep=%d residual=%.2e time-to-tol=%.3f s" % (norm, r.converged, r.iterations,
      r.n_sweep, r.final_residual, t))
print("kernel ms:", {k: round(ms[i], 2) for i, k in enumerate(capi.PROF_KINDS)}, "launches", list(nk))
print("last DSA krylov iterations:", dsa.last_iterations())
print("history:", ["%.2e" % h for h in r.change_history])
np.save("/tmp/c3_rho.npy", rho.cpu().numpy())
