"""C4 offline POD on the device (for ncu captures of the Gram / right-multiply
kernels): 40 training samples, correction snapshots (window 3), rank 20."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_10488_b200 import configs, rte
from tests.problems import pin_cell
nx = 128
train, _ = configs.c4_params(40, 1)
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
tb = rte.TransportBatch(pin_cell(rte)(nx), mesh, rte.chebyshev_legendre(16, 8), train)
snaps = rte.collect_snapshots(tb, 3, 1e-8)
F = rte.snapshot_matrix(tb, snaps, "correction")
torch.cuda.synchronize(); t0 = time.time()
U, s = rte.pod(F, 20)
torch.cuda.synchronize()
print("POD of %d x %d: %.3f s, sigma_1 %.3e" % (F.shape[1], F.shape[0], time.time() - t0, s[0]))
