"""Quick C5 sweep timing (BASELINE configs[4]): fixed-point sweep rho* = L rho + bbar."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_10488_b200 import rte, capi

def c5_inputs(nx, S, seed=20260822):
    n = nx * nx
    u = np.zeros(2 * n * S)
    capi.check(capi.load().rte_unit_draws(seed, u.size, capi.dptr(u)))
    st = np.empty((S, n)); ss = np.empty((S, n))
    for s in range(S):
        a = u[2 * n * s: 2 * n * s + n]; b = u[2 * n * s + n: 2 * n * (s + 1)]
        st[s] = np.exp(np.log(0.1) + (np.log(100.0) - np.log(0.1)) * a)
        ss[s] = (0.5 + (0.99 - 0.5) * b) * st[s]
    return st, ss

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
nphi, nvz = (32, 16) if len(sys.argv) <= 3 else map(int, sys.argv[3].split(","))
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
quad = rte.chebyshev_legendre(nphi, nvz)
st, ss = c5_inputs(nx, S)
px, py = mesh.cell_points()
g = mesh.project(np.ones(px.size))
t0 = time.time()
b = rte.TransportBatch.from_cells(mesh, quad, st, ss, g)
print("setup %.2fs slots %d ndof %d" % (time.time() - t0, b.n_slots(), b.n_dof()), flush=True)
rho = torch.zeros(S, b.n_dof(), dtype=torch.float64, device="cuda")
for _ in range(2):
    out = b.fixed_point(rho)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 3
ev0.record()
for _ in range(K):
    out = b.fixed_point(out)
ev1.record(); torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / K
upd = nx * nx * b.n_slots() * S
print("sweep+reduce %.3f ms  %.3e updates/s  operand-stream %.1f GB/s  (%.2f GFLOP/s at 66 flop)" %
      (ms, upd / ms * 1e3, upd * 40 / ms / 1e6, upd * 66 / ms / 1e6))
print("checksum", float(out.sum()))
