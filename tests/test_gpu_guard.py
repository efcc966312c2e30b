"""Bounds checking of every device kernel family without compute-sanitizer
(closed on the GPU pool): the parity suites re-run in a subprocess with
RTE_GUARD=1, where every library allocation carries 4 KB guard zones of 0xFF
bytes and starts filled with that pattern (NaN as fp64/fp32).  An
out-of-bounds write shows up as an overwritten guard zone
(rte_guard_check), an out-of-bounds or uninitialised read as NaN in a result
the parity tests compare with the oracle."""
import ctypes
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SUITES = ["tests/test_gpu_parity.py", "tests/test_gpu_production_plans.py", "tests/test_gpu_rom.py",
          "tests/test_gpu_offline.py", "tests/test_gpu_gmres.py", "tests/test_gpu_kinetic.py",
          "tests/test_gpu_full_blocks.py", "tests/test_gpu_dsa_status.py", "tests/test_gpu_dsa_eliminated.py",
          "tests/test_gpu_pod_kat.py", "tests/test_gpu_strategy_plugin.py", "tests/test_gpu_kats.py"]


def _run(code):
    env = dict(os.environ, RTE_GUARD="1")
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)


def test_guard_detects_a_one_element_overflow():
    r = _run("import ctypes\n"
             "from paper_2402_10488_b200 import capi\n"
             "L = capi.load()\n"
             "assert L.rte_guard_selftest(0) == 0\n"
             "v, c = ctypes.c_long(), ctypes.c_long()\n"
             "assert L.rte_guard_check(ctypes.byref(v), ctypes.byref(c)) == 0\n"
             "print(v.value, c.value)\n")
    assert r.returncode == 0, r.stderr
    v, c = map(int, r.stdout.split())
    assert v >= 1 and c >= 1


def test_guard_off_reports_unsupported():
    from paper_2402_10488_b200 import capi
    if os.environ.get("RTE_GUARD"):
        pytest.skip("RTE_GUARD set in this process")
    v, c = ctypes.c_long(), ctypes.c_long()
    assert capi.load().rte_guard_check(ctypes.byref(v), ctypes.byref(c)) == capi.RTE_ERR_UNSUPPORTED


def test_parity_suites_clean_under_guard(tmp_path):
    report = tmp_path / "guard.json"
    env = dict(os.environ, RTE_GUARD="1", RTE_GUARD_REPORT=str(report))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu"] + SUITES,
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=3000)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    g = json.loads(report.read_text())
    assert g["rc"] == 0 and g["violations"] == 0, g
    assert g["checked"] > 100, g
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "guard_report.json"), "w") as f:
            json.dump(dict(g, suites=SUITES, summary=r.stdout.strip().splitlines()[-1]), f, indent=1)
