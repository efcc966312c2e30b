"""One 2D DSA solve (for launch lists): python scripts/dsa_once.py NX S TOL [c3|c5|h<st>:<c>|r<a>:<b>]"""
import os, sys, time
os.environ.setdefault("RTE_DSA_WARM", "0")  # repeated solves of one rhs: time cold solves
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_10488_b200 import rte, configs
nx = int(sys.argv[1]); S = int(sys.argv[2]); tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-12
kind = sys.argv[4] if len(sys.argv) > 4 else "c3"
mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
quad = rte.chebyshev_legendre(16, 8)
n = nx * nx
if kind == "c3":
    st, ss = np.full((S, n), 10.0), np.full((S, n), 9.99)
elif kind.startswith("h"):  # homogeneous h<sigma_t>:<c>
    sg, cc = (float(v) for v in kind[1:].split(":"))
    st, ss = np.full((S, n), sg), np.full((S, n), sg * cc)
elif kind.startswith("r"):  # random sigma_t ~ logU[a,b] per cell, c ~ U[0.5,0.99]: r<a>:<b>
    a_, b_ = (float(v) for v in kind[1:].split(":"))
    rg = np.random.default_rng(5)
    st = np.exp(np.log(a_) + (np.log(b_) - np.log(a_)) * rg.uniform(size=(S, n)))
    ss = rg.uniform(0.5, 0.99, size=(S, n)) * st
else:
    st, ss = configs.c5_coefficients(nx, S)
px, py = mesh.cell_points()
g = mesh.project(np.ones(px.size))
b = rte.TransportBatch.from_cells(mesh, quad, st, ss, g)
d = rte.DsaOperator(b)
d.set_tolerance(tol, 2000)
rhs = torch.rand(S, b.n_dof(), dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
ts = []
for k in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize(); t0 = time.time()
    x = d.solve_density(rhs)
    torch.cuda.synchronize()
    ts.append(time.time() - t0)
print("solve %.3f s (min of %s), krylov iterations %d, %.2f ms/iteration"
      % (min(ts), " ".join("%.3f" % t for t in ts), d.last_iterations(), 1e3 * min(ts) / max(1, d.last_iterations())),
      flush=True)
