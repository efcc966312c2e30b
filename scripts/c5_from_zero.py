"""C5 bench job (20 SI-DSA iterations from the zero guess, floor rule) timed
once warm: ms per step and the BiCGStab iterations per step, for sweeps over
the DSA development knobs (RTE_DSA_NU, RTE_DSA_NU_COARSE, RTE_DSA_WARM, ...)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_10488_b200 import configs, rte
nx, S, K = 1024, 16, 20
tol = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-8
st, ss = configs.c5_coefficients(nx, S)
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
px, py = mesh.cell_points()
b = rte.TransportBatch.from_cells(mesh, rte.chebyshev_legendre(32, 16), st, ss, mesh.project(np.ones(px.size)))
d = rte.DsaOperator(b)
d.set_tolerance(tol, 2000)
cfg = rte.SolveConfig(fixed_iters=K, max_iters=K, compute_residual=False, check_every=K, dsa_floor=1.0)
rte.sisa_solve(b, "DSA", rte.SolveConfig(fixed_iters=2, max_iters=2, compute_residual=False, check_every=2, dsa_floor=1.0))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
rho, reps = rte.sisa_solve(b, "DSA", cfg)
e1.record(); torch.cuda.synchronize()
log = d.iteration_log()
print("knobs %s: %.1f ms/step, BiCGStab its %s (sum %d), checksum %.12e" % (
    {k: v for k, v in os.environ.items() if k.startswith("RTE_DSA")}, e0.elapsed_time(e1) / K, log, sum(log),
    float(rho.sum())), flush=True)
