"""The tensor-core (DMMA) Gram / right-multiply kernels of the POD against
their CUDA-core versions (RTE_POD_DMMA=0, read once per process: a
subprocess) and against numpy, on shapes with ragged rows and columns."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2402_10488_b200 import rte
rng = np.random.default_rng(7)
out = {}
for (m, n) in [(70001, 37), (4096, 128), (12345, 120), (333, 5)]:
    F = rng.standard_normal((n, m)) * np.logspace(0, -6, n)[:, None]   # columns of decaying size
    U, s = rte.pod(torch.from_numpy(F).cuda(), min(n, 20))
    out["s_%%d_%%d" %% (m, n)] = np.asarray(s)
    out["U_%%d_%%d" %% (m, n)] = U.cpu().numpy()
    out["F_%%d_%%d" %% (m, n)] = F
np.savez(sys.argv[1], **out)
""" % ROOT


def _run(tmp, dmma):
    env = dict(os.environ, RTE_POD_DMMA=dmma)
    path = os.path.join(tmp, "pod_%s.npz" % dmma)
    subprocess.run([sys.executable, "-c", SCRIPT, path], check=True, env=env, timeout=600)
    return np.load(path)


def test_dmma_pod_matches_cuda_core_pod_and_numpy(tmp_path):
    a, b = _run(str(tmp_path), "1"), _run(str(tmp_path), "0")
    for key in a.files:
        if not key.startswith("s_"):
            continue
        tag = key[2:]
        s1, s0 = a[key], b[key]
        F = a["F_" + tag]
        sv = np.linalg.svd(F, compute_uv=False)
        np.testing.assert_allclose(s1, s0, rtol=1e-12, atol=1e-14 * sv[0])
        np.testing.assert_allclose(s1[:len(sv)], sv[:len(s1)], rtol=1e-10, atol=1e-13 * sv[0])
        U = a["U_" + tag]   # (rank, m): orthonormal rows spanning the leading left singular vectors
        assert np.abs(U @ U.T - np.eye(U.shape[0])).max() < 1e-12
        r = U.shape[0]
        proj = np.linalg.norm(F - (F @ U.T) @ U, 2)
        assert proj <= sv[r] * (1 + 1e-6) + 1e-12 * sv[0] if r < len(sv) else proj < 1e-10 * sv[0]
