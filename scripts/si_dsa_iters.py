"""C5 SI-DSA: BiCGStab iterations and time per SI iteration (RTE_DSA_REPORT)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RTE_DSA_REPORT", "1")
import numpy as np, torch
from paper_2402_10488_b200 import configs, rte
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
its = int(sys.argv[3]) if len(sys.argv) > 3 else 8
st, ss = configs.c5_coefficients(nx, S)
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
px, py = mesh.cell_points()
b = rte.TransportBatch.from_cells(mesh, rte.chebyshev_legendre(32, 16), st, ss, mesh.project(np.ones(px.size)))
d = rte.DsaOperator(b)
d.set_tolerance(1e-8, 2000)
cfg = rte.SolveConfig(fixed_iters=its, max_iters=its, compute_residual=False, check_every=its)
torch.cuda.synchronize(); t0 = time.time()
rho, reps = rte.sisa_solve(b, "DSA", cfg)
torch.cuda.synchronize()
print("%d SI-DSA iterations: %.3f s (%.1f ms/iteration); last change %.3e" %
      (its, time.time() - t0, 1e3 * (time.time() - t0) / its, reps[0].change_history[-1]), flush=True)
