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


def test_struct_layouts_match_the_header(tmp_path):
    """Every struct the ctypes binding mirrors has the C header's size and field
    offsets (a C program compiled against include/rte_b200.h prints them)."""
    import subprocess
    from paper_2402_10488_b200 import capi
    structs = {"rte_problem": capi.Problem, "rte_affine": capi.Affine, "rte_rom": capi.Rom,
               "rte_si_config": capi.SiConfig, "rte_si_report": capi.SiReport,
               "rte_gmres_config": capi.GmresConfig, "rte_gmres_report": capi.GmresReport}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rte_b200.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append('printf("%s size %%zu\\n", sizeof(%s));' % (cname, cname))
        for fname, _ in py._fields_:
            lines.append('printf("%s.%s %%zu\\n", offsetof(%s, %s));' % (cname, fname, cname, fname))
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    str(src), "-o", str(exe)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got["%s size" % cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got["%s.%s" % (cname, fname)]) == getattr(py, fname).offset, (cname, fname)


def test_solve_config_maps_onto_the_c_struct():
    """rte.SolveConfig -> rte_si_config field by field (no device needed)."""
    from paper_2402_10488_b200 import capi, rte
    c = rte.SolveConfig(eps_sisa=1e-8, norm="rel", max_iters=77, fixed_iters=0, theta=5, eps_romsad=3e-9,
                        compute_residual=False, check_every=2, dsa_inner=1e-2)
    s = rte.si_config(c, capi.RTE_ROMSAD)
    assert (s.method, s.eps, s.norm, s.max_iters, s.fixed_iters, s.theta) == (capi.RTE_ROMSAD, 1e-8, capi.RTE_NORM_REL,
                                                                             77, 0, 5)
    assert (s.eps_romsad, s.use_guess, s.compute_residual, s.check_every, s.dsa_inner) == (3e-9, 0, 0, 2, 1e-2)
    import pytest
    for bad in (dict(norm="l2"), dict(max_iters=0), dict(dsa_inner=1.5)):
        with pytest.raises(ValueError):
            rte.si_config(rte.SolveConfig(**bad), capi.RTE_DSA)


def test_batch_assembly_helpers_match_numpy():
    """rte_combine_terms / rte_scalar_blocks (setup.cpp) against the numpy
    formulas they replace in rte.TransportBatch: bitwise."""
    import numpy as np
    from paper_2402_10488_b200 import capi
    L = capi.load()
    rng = np.random.default_rng(5)
    S, K, n = 7, 4, 1000
    psi = rng.uniform(-2, 3, (S, K))
    terms = rng.uniform(-1, 1, (K, n))
    out = np.empty((S, n))
    assert L.rte_combine_terms(S, K, n, capi.dptr(psi), capi.dptr(terms), capi.dptr(out)) == 0
    ref = np.zeros((S, n))
    for k in range(K):
        ref = ref + psi[:, k][:, None] * terms[k][None]
    assert np.array_equal(out, ref)
    d0 = rng.uniform(0.5, 2, 50)
    blocks = d0[:, None, None] * np.eye(4)[None]
    sc = np.empty(50)
    assert L.rte_scalar_blocks(50, 4, capi.dptr(np.ascontiguousarray(blocks)), capi.dptr(sc)) == 0
    assert np.array_equal(sc, d0)
    blocks[3, 0, 1] = 1e-6
    assert L.rte_scalar_blocks(50, 4, capi.dptr(np.ascontiguousarray(blocks)), capi.dptr(sc)) == capi.RTE_ERR_UNSUPPORTED


def test_constant_weight_helpers_match_array_versions():
    """rte_weighted_mass_const / rte_project_const == the per-point versions
    on a constant array, bitwise (slab and XY)."""
    import numpy as np
    from paper_2402_10488_b200 import rte
    for mesh in (rte.Mesh.slab([0.0, 0.1, 0.35, 0.6, 1.0]), rte.Mesh.rect_uniform(0, 1, 5, 0, 2, 3)):
        px, _ = mesh.cell_points()
        for c in (0.0, 1.0, 0.3 * 0.999, 12.5):
            assert np.array_equal(mesh.weighted_mass(c), mesh.weighted_mass(np.full(px.size, c)))
            assert np.array_equal(mesh.project(c), mesh.project(np.full(px.size, c)))
