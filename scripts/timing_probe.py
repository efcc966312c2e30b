"""Repeat small C1/C2 solves to separate first-call costs from steady state."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_10488_b200 import configs, rte
from tests.problems import homog, two_region_slab


def timed(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    return out, time.perf_counter() - t0


mesh = rte.Mesh.slab_uniform(0.0, 1.0, 256)
prob = homog(rte, rte.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0)
for norm in ("rel", "abs", "rel", "abs"):
    b, tb = timed(lambda: rte.TransportBatch(prob, mesh, rte.gauss_legendre(16), [[]]))
    (rho, reps), t = timed(lambda: rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm=norm)))
    print("C1 %s: create %.4f s, solve %.4f s, its %d" % (norm, tb, t, reps[0].iterations), flush=True)
train, test = configs.c2_params(32, 512)
quad = rte.gauss_legendre(16)
tb = rte.TransportBatch(two_region_slab(rte), mesh, quad, train)
snaps = rte.collect_snapshots(tb, 3, 1e-8)
Fp = rte.snapshot_matrix(tb, snaps, "primary")
Up, sp = rte.pod(Fp, 16)
pm = rte.build_reduced_model(tb, Up, sp, float(np.sum(sp[16:]) / np.sum(sp)), 1e-8, "p")
b = rte.TransportBatch(two_region_slab(rte), mesh, quad, test)
rte.load_rom(b, 0, pm)
for k in range(3):
    (g, st), t = timed(lambda: rte.romig(b))
    print("C2 romig guess: %.4f s" % t, flush=True)
for k in range(3):
    (rho, reps), t = timed(lambda: rte.sisa_solve(b, "ROMIG", rte.SolveConfig(eps_sisa=1e-8, norm="abs", max_iters=500)))
    print("C2 ROMIG solve: %.4f s mean n_sweep %.2f" % (t, np.mean([r.n_sweep for r in reps])), flush=True)
for k in range(2):
    (rho, reps), t = timed(lambda: rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm="abs", max_iters=500)))
    print("C2 DSA solve: %.4f s mean n_sweep %.2f" % (t, np.mean([r.n_sweep for r in reps])), flush=True)
