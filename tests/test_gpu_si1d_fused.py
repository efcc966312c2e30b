"""The fused slab SI loop (si1d.cu: the whole sisa_solve loop of a sample in
one CTA) against the per-kernel loop it replaces (RTE_SI1D_FUSED=0, run in a
subprocess because the switch is read once per process) on C2-shaped
batches: SI-DSA, plain SI and ROMIG are bitwise identical (same sweep, same
cyclic reduction, same arithmetic); ROMSA/ROMSAD reproduce the logs, switch
iterations and iteration counts with fluxes to 1e-13 (the reduced projection
sums in a different fixed order).  Oracle parity of the fused path is covered
by the existing slab suites (test_gpu_parity, test_gpu_rom,
test_gpu_fullsize_parity), which now run through it."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.problems import rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
from paper_2402_10488_b200 import configs, rte
from tests.problems import homog, two_region_slab
out = {}
train, test = configs.c2_params(8, 24)
mesh, quad = rte.Mesh.slab_uniform(0.0, 1.0, 256), rte.gauss_legendre(16)
tb = rte.TransportBatch(two_region_slab(rte), mesh, quad, train)
sn = rte.collect_snapshots(tb, 3, 1e-8)
Uc, sc = rte.pod(rte.snapshot_matrix(tb, sn, "correction"), 8)
Up, sp = rte.pod(rte.snapshot_matrix(tb, sn, "primary"), 6)
cm = rte.build_reduced_model(tb, Uc, sc, float(np.sum(sc[8:]) / np.sum(sc)), 1e-8, "c")
pm = rte.build_reduced_model(tb, Up, sp, float(np.sum(sp[6:]) / np.sum(sp)), 1e-8, "p")
b = rte.TransportBatch(two_region_slab(rte), mesh, quad, test)
rte.load_rom(b, 0, pm)
rte.load_rom(b, 1, cm)
er = rte.romsad_tolerance(1e-8, cm.discarded_fraction)
for m in ("SI", "DSA", "ROMIG", "ROMSA", "ROMSAD"):
    cfg = rte.SolveConfig(eps_sisa=1e-8, norm="rel", theta=3, eps_romsad=er, max_iters=400)
    rho, reps = rte.sisa_solve(b, m, cfg)
    np.save(%(dir)r + "/" + m + ".npy", rho.cpu().numpy())
    out[m] = [[r.iterations, r.correction_log, r.switch_iter, r.converged, list(r.change_history)] for r in reps]
c1 = rte.TransportBatch(homog(rte, rte.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0), mesh, quad, [[]])
rho, reps = rte.sisa_solve(c1, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm="rel"))
np.save(%(dir)r + "/C1.npy", rho.cpu().numpy())
out["C1"] = [[r.iterations, r.correction_log, r.switch_iter, r.converged, list(r.change_history)] for r in reps]
print(json.dumps(out))
'''


def run(tmp, fused):
    d = os.path.join(tmp, "fused" if fused else "unfused")
    os.makedirs(d, exist_ok=True)
    env = dict(os.environ, RTE_SI1D_FUSED="1" if fused else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "dir": d}], cwd=ROOT, env=env,
                       capture_output=True, text=True, check=True)
    return d, json.loads(r.stdout.strip().splitlines()[-1])


def test_fused_slab_loop_matches_per_kernel_loop(tmp_path):
    df, rf = run(str(tmp_path), True)
    du, ru = run(str(tmp_path), False)
    for m in ("SI", "DSA", "ROMIG", "ROMSA", "ROMSAD", "C1"):
        a, b = np.load(os.path.join(df, m + ".npy")), np.load(os.path.join(du, m + ".npy"))
        for s, (x, y) in enumerate(zip(rf[m], ru[m])):
            assert x[:4] == y[:4], (m, s, x[:4], y[:4])
        if m in ("ROMSA", "ROMSAD"):
            assert max(rel_l2(a[s], b[s]) for s in range(a.shape[0])) < 1e-13, m
            for x, y in zip(rf[m], ru[m]):
                np.testing.assert_allclose(x[4], y[4], rtol=1e-9, atol=1e-15)
        else:
            assert np.array_equal(a, b), m
            assert all(x[4] == y[4] for x, y in zip(rf[m], ru[m])), m
