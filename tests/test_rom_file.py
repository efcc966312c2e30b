"""RTEROM1 artifact round trip (reduced_model.cpp:41-104): the host mirror
writes byte-identical files to the oracle restatement and reads files the
oracle wrote; truncated / wrong-magic files raise as the reference does."""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from paper_2402_10488_b200.rte import ReducedModel


def _model(cls, rng, nd=24, r=3, k=2):
    m = cls(1, 8, nd, r, k, "c", 1e-3, 1e-8)
    m.u_rho = rng.standard_normal((nd, r))
    m.u_iso = rng.standard_normal((nd, r))
    m.a_r = [rng.standard_normal((r, r)) for _ in range(k)]
    m.singular_values = np.sort(rng.random(r))[::-1].copy()
    m.b_r = rng.standard_normal(r)
    m.discarded_fraction = 0.125
    return m


def test_rom_file_bytes_match_oracle(tmp_path):
    rng = np.random.default_rng(7)
    a = _model(ReducedModel, rng)
    o = ro.ReducedModel(a.geometry, a.n_v, a.n_dof, a.rank, a.k_affine, a.kind, a.eps_pod, a.eps_train,
                        a.u_rho, a.u_iso, a.a_r, a.singular_values, a.discarded_fraction, a.b_r)
    a.save(str(tmp_path / "p.rom"))
    o.save(str(tmp_path / "o.rom"))
    assert (tmp_path / "p.rom").read_bytes() == (tmp_path / "o.rom").read_bytes()
    b = ReducedModel.load(str(tmp_path / "o.rom"))
    assert (b.geometry, b.n_v, b.n_dof, b.rank, b.k_affine, b.kind) == (1, 8, 24, 3, 2, "c")
    assert b.eps_pod == a.eps_pod and b.discarded_fraction == a.discarded_fraction
    for x, y in [(b.u_rho, a.u_rho), (b.u_iso, a.u_iso), (b.singular_values, a.singular_values), (b.b_r, a.b_r)]:
        assert np.array_equal(x, y)
    for x, y in zip(b.a_r, a.a_r):
        assert np.array_equal(x, y)


def test_rom_file_errors(tmp_path):
    rng = np.random.default_rng(8)
    a = _model(ReducedModel, rng)
    p = tmp_path / "m.rom"
    a.save(str(p))
    data = p.read_bytes()
    (tmp_path / "t.rom").write_bytes(data[:-5])
    with pytest.raises(RuntimeError, match="truncated"):
        ReducedModel.load(str(tmp_path / "t.rom"))
    (tmp_path / "w.rom").write_bytes(b"RTESNP1\0" + data[8:])
    with pytest.raises(RuntimeError, match="wrong magic"):
        ReducedModel.load(str(tmp_path / "w.rom"))
    bad = bytearray(data)
    bad[8] = 2
    (tmp_path / "v.rom").write_bytes(bytes(bad))
    with pytest.raises(RuntimeError, match="unsupported version"):
        ReducedModel.load(str(tmp_path / "v.rom"))
    with pytest.raises(RuntimeError, match="cannot open"):
        ReducedModel.load(str(tmp_path / "missing.rom"))
