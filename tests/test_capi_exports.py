"""CPU checks of the drop-in boundary: librte_b200.so builds, loads and
exports every symbol include/rte_b200.h declares (no compute calls)."""
import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rte_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rte_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2402_10488_b200 import build, capi
    build.build()
    lib = ctypes.CDLL(capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in capi.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound


def test_host_helpers_match_oracle():
    """Host-side setup helpers (no GPU): GL nodes, cell points, weighted mass,
    projection and the mt19937_64 unit draws agree with the oracle."""
    from oracle import rte_oracle as ro
    from paper_2402_10488_b200 import rte
    x, w = rte.gauss_legendre_nodes(16)
    xo, wo = ro.gauss_legendre_nodes(16)
    assert np.array_equal(x, xo) and np.array_equal(w, wo)
    mesh_p = rte.Mesh.slab([0.0, 0.3, 0.7, 1.2, 2.0])
    mesh_o = ro.Mesh.slab([0.0, 0.3, 0.7, 1.2, 2.0])
    px, py = mesh_p.cell_points()
    qx, qy = ro.cell_points(mesh_o)
    assert np.array_equal(px, qx)
    f = lambda x, y: 1.0 + x
    assert np.max(np.abs(mesh_p.project(f(px, py)) - ro.project(mesh_o, ro.build_dg_space(mesh_o), f))) < 1e-15
    from paper_2402_10488_b200 import capi
    out = np.zeros(5)
    capi.check(capi.load().rte_unit_draws(20260822, 5, capi.dptr(out)))
    assert np.array_equal(out, ro.unit_draws(20260822, 5))


def test_invalid_arguments_are_reported_not_raised_across_the_abi():
    from paper_2402_10488_b200 import capi
    L = capi.load()
    p = capi.Problem()
    p.geometry = 7
    h = ctypes.c_void_p()
    assert L.rte_create(ctypes.byref(p), 0, ctypes.byref(h)) == capi.RTE_ERR_INVALID
    assert b"geometry" in L.rte_last_error(None)
