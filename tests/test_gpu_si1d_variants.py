"""The fused slab SI kernel's other instantiations against the oracle
(sisa.cpp:14-54 with DsaStrategy; transport_system.cpp:279-310 sweeps;
dsa.cpp:154-277 direct DSA): slabs whose cyclic-reduction factors do not fit
in shared memory (N = 1000 and 2000 cells: 32 and 64 cells per lane, factors
read from HBM), an odd-sized slab, and every case with the sweep cache
disabled (RTE_SLAB_CACHE=0: cell inverses on the fly; a subprocess, the
switch is read once).  The bar: identical iteration counts, 1e-8 flux."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import homog, rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(1000, 10.0, 0.99), (2000, 40.0, 0.999), (77, 5.0, 0.9)]

SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
from paper_2402_10488_b200 import rte
from tests.problems import homog
out = []
for n, st, c in %(cases)r:
    b = rte.TransportBatch(homog(rte, rte.SLAB1D, st * (1 - c), st * c, 1.0), rte.Mesh.slab_uniform(0.0, 1.0, n),
                           rte.gauss_legendre(16), [[]])
    rho, reps = rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-10))
    out.append([reps[0].iterations, rho.cpu().numpy()[0].tolist()])
print(json.dumps(out))
'''


def oracle(n, st, c):
    m = ro.Mesh.slab_uniform(0.0, 1.0, n)
    s = ro.TransportSystem(homog(ro, ro.SLAB1D, st * (1 - c), st * c, 1.0), m, ro.build_dg_space(m),
                           ro.gauss_legendre(16), [])
    return ro.sisa_solve(s, ro.DsaStrategy(ro.build_dsa(s)), ro.SolveConfig(eps_sisa=1e-10))


@pytest.mark.parametrize("cache", ["1", "0"])
def test_fused_slab_variants_match_oracle(cache):
    env = dict(os.environ, RTE_SLAB_CACHE=cache)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "cases": CASES}], cwd=ROOT, env=env,
                       capture_output=True, text=True, check=True)
    dev = json.loads(r.stdout.strip().splitlines()[-1])
    for (n, st, c), (its, rho) in zip(CASES, dev):
        rho_o, rep_o = oracle(n, st, c)
        assert its == rep_o.iterations, (n, its, rep_o.iterations)
        assert rel_l2(np.array(rho), rho_o) < 1e-8, n
