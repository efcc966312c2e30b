"""DSA 2D convergence per grid size (diagnostic): python scripts/dsa_levels.py [sizes]
Prints the relative residual history of sample 0 (needs RTE_DSA_TRACE=1 for
the per-iteration history; iteration counts are otherwise rounded up to the
host polling interval)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_10488_b200 import rte
sizes = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8,16,32,64,128").split(",")]
for nx in sizes:
    mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    quad = rte.chebyshev_legendre(16, 8)
    n = nx * nx
    st, ss = np.full((1, n), 10.0), np.full((1, n), 9.99)
    px, py = mesh.cell_points()
    b = rte.TransportBatch.from_cells(mesh, quad, st, ss, mesh.project(np.ones(px.size)))
    d = rte.DsaOperator(b)
    d.set_tolerance(1e-8, int(os.environ.get("MAXIT", "60")))
    rhs = torch.rand(1, b.n_dof(), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize(); t0 = time.time()
    d.solve_density(rhs)
    torch.cuda.synchronize()
    print("nx %d: %.3f s, %d iterations" % (nx, time.time() - t0, d.last_iterations()), flush=True)
