"""Where the end-to-end C5 job spends its time: rte_create (H2D), DSA setup, the 20 SI-DSA iterations from zero, D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_10488_b200 import configs, rte

nx, S, K = 1024, 16, 20
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
quad = rte.chebyshev_legendre(32, 16)
st, ss = configs.c5_coefficients(nx, S, seed=configs.SEEDS["c5"])
px, py = mesh.cell_points()
g = mesh.project(np.ones(px.size))
st_p = torch.from_numpy(st).pin_memory(); ss_p = torch.from_numpy(ss).pin_memory()
for rep in range(3):
    out_h = torch.empty((S, 4 * nx * nx), dtype=torch.float64).pin_memory()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b = rte.TransportBatch.from_cells(mesh, quad, st_p.numpy(), ss_p.numpy(), g)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    d = rte.DsaOperator(b); d.set_tolerance(1e-8, 2000)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    cfg = rte.SolveConfig(fixed_iters=K, max_iters=K, compute_residual=False, check_every=K, dsa_floor=1.0)
    r, _ = rte.sisa_solve(b, "DSA", cfg)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    out_h.copy_(r); torch.cuda.synchronize(); t4 = time.perf_counter()
    print("rep %d: create %.3f  dsa_setup %.3f  solve %.3f  d2h %.3f  total %.3f s" % (rep, t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0), flush=True)
    del b, d, r
