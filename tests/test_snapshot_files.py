"""RTESNP1 snapshot files (snapshots.cpp:15-78, 128-176, 224-314): the host
mirror writes the reference's byte layout -- header of 58 + 8 n_params
bytes with w_mu / n_conv / converged at the patch offset 49 + 8 n_params,
then w_mu records (f^(l) in the store precision, delta_rho^(l) in fp64) and
the converged kinetic vector -- and reads it back."""
import struct

import numpy as np
import pytest

from paper_2402_10488_b200 import rte


def _data(rng, nv=4, nd=6, w=3):
    return (rng.standard_normal((w, nv * nd)), rng.standard_normal((w, nd)), rng.standard_normal(nv * nd))


def test_layout_matches_reference_writer(tmp_path):
    rng = np.random.default_rng(1)
    fi, dr, fc = _data(rng)
    p = str(tmp_path / "snap_000.snap")
    rte.write_snapshot_file(p, 0, 4, 6, [0.25, 0.9], 3, 1e-8, fi, dr, fc, n_conv=7, converged=True)
    b = open(p, "rb").read()
    hb = rte.snapshot_header_bytes(2)
    assert hb == 74 and rte.snapshot_patch_offset(2) == 65
    # header fields in the writer's order (snapshots.cpp:135-146)
    assert b[:8] == b"RTESNP1\0"
    assert struct.unpack_from("<IIQQI", b, 8) == (1, 0, 4, 6, 2)
    assert struct.unpack_from("<2d", b, 36) == (0.25, 0.9)
    assert struct.unpack_from("<IdB", b, 52) == (3, 1e-8, 8)
    assert struct.unpack_from("<IIB", b, rte.snapshot_patch_offset(2)) == (3, 7, 1)
    # records then the converged vector
    rec = 4 * 6 * 8 + 6 * 8
    assert len(b) == hb + 3 * rec + 4 * 6 * 8
    assert np.array_equal(np.frombuffer(b, np.float64, 24, hb), fi[0])
    assert np.array_equal(np.frombuffer(b, np.float64, 6, hb + 24 * 8), dr[0])
    assert np.array_equal(np.frombuffer(b, np.float64, 24, hb + 3 * rec), fc)
    r = rte.read_snapshot_file(p)
    assert (r["w_mu"], r["n_conv"], r["converged"], r["mu"], r["window"]) == (3, 7, True, [0.25, 0.9], 3)
    assert np.array_equal(r["f_iter"], fi) and np.array_equal(r["drho"], dr) and np.array_equal(r["f_conv"], fc)


def test_short_solve_and_float32_store(tmp_path):
    rng = np.random.default_rng(2)
    fi, dr, fc = _data(rng)
    p = str(tmp_path / "s.snap")
    # converged after 2 iterations with window 3 -> w_mu = 2 records
    rte.write_snapshot_file(p, 1, 4, 6, [], 3, 1e-6, fi[:2], dr[:2], fc, n_conv=2, converged=False, float32=True)
    b = open(p, "rb").read()
    assert len(b) == rte.snapshot_header_bytes(0) + 2 * (24 * 4 + 6 * 8) + 24 * 4
    r = rte.read_snapshot_file(p)
    assert r["dsize"] == 4 and r["w_mu"] == 2 and not r["converged"]
    assert np.array_equal(r["f_iter"], fi[:2].astype(np.float32).astype(np.float64))
    assert np.array_equal(r["drho"], dr[:2])


def test_errors(tmp_path):
    rng = np.random.default_rng(3)
    fi, dr, fc = _data(rng)
    p = tmp_path / "a.snap"
    rte.write_snapshot_file(str(p), 0, 4, 6, [0.5], 3, 1e-8, fi, dr, fc, n_conv=5, converged=True)
    data = p.read_bytes()
    (tmp_path / "t.snap").write_bytes(data[:-3])
    with pytest.raises(RuntimeError, match="truncated"):
        rte.read_snapshot_file(str(tmp_path / "t.snap"))
    (tmp_path / "m.snap").write_bytes(b"RTEROM1\0" + data[8:])
    with pytest.raises(RuntimeError, match="not a snapshot file"):
        rte.read_snapshot_file(str(tmp_path / "m.snap"))
    (tmp_path / "empty").mkdir()
    with pytest.raises(RuntimeError, match="no .snap files"):
        rte.load_snapshots(str(tmp_path / "empty"))
