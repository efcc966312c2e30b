"""The device POD (rte_pod: repeated shifted CholeskyQR + Jacobi SVD of the
small factor, csrc/pod.cu) against the reference's POD known-answer tests,
proj/tests/unit/test_pod.cpp (restated in numpy: the spectrum is exact by
construction whatever Gaussian generator builds the orthonormal factors)."""
import numpy as np
import pytest

from oracle import rte_oracle as ro

pytestmark = pytest.mark.gpu


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def device_pod(a, rank):
    """a: numpy m x n -> (U numpy m x rank, all singular values)."""
    import torch
    F = torch.as_tensor(np.ascontiguousarray(a.T), device="cuda:0")  # [n_cols][m] = column-major m x n
    U, sv = rte().pod(F, rank)
    return U.cpu().numpy().T, sv


def ortho_defect(q):
    return float(np.abs(q.T @ q - np.eye(q.shape[1])).max())


def synthetic_spectrum(m=3000, n=40, seed=42):  # test_pod.cpp:15-36
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = 10.0 ** (-0.5 * np.arange(n))
    return (u * s) @ v.T, s


def test_known_spectrum():  # test_pod.cpp:72-81 (kappa = 10^19.5, past 1/u)
    a, s = synthetic_spectrum()
    U, sv = device_pod(a, 40)
    r = rte().truncation_rank(sv, 1e-9)
    assert r == 18
    assert sv.size == 40
    for k in range(30):  # trailing values drown in roundoff
        assert abs(sv[k] - s[k]) < 1e-12 * s[k] + 1e-15, (k, sv[k], s[k])
    assert ortho_defect(U[:, :r]) < 1e-13
    # the retained subspace equals the dense reference's (test_pod.cpp:129-132)
    ud = np.linalg.svd(a, full_matrices=False)[0][:, :r]
    assert np.linalg.svd(U[:, :r].T @ ud, compute_uv=False).min() > 1.0 - 1e-12
    # projection error meets the tail bound (test_pod.cpp:135-138)
    proj = np.linalg.norm(a - U[:, :r] @ (U[:, :r].T @ a))
    assert proj <= np.sqrt(np.sum(s[r:] ** 2)) * (1.0 + 1e-6)
    # the oracle (dgesdd) agrees on the rank
    assert ro.pod_truncate(a, 1e-9).rank == r


def test_gram_eigenvalues_cross_check():  # test_pod.cpp:146-158
    small = np.random.default_rng(7).standard_normal((50, 10))
    lam = np.linalg.eigvalsh(small.T @ small)[::-1]
    _, sv = device_pod(small, 10)
    assert np.all(np.abs(np.sqrt(np.maximum(lam, 0.0)) - sv) < 1e-12)


def test_rank_deficient():  # test_pod.cpp:160-175
    base = np.random.default_rng(11).standard_normal((200, 3))
    dup = np.hstack([base, base])  # numerical rank 3
    U, sv = device_pod(dup, 6)
    r = rte().truncation_rank(sv, 1e-15)
    assert r == 3
    assert np.all(sv[3:] < 1e-13 * sv[0])
    ur = U[:, :r]
    assert ortho_defect(ur) < 1e-13
    assert np.linalg.norm(dup - ur @ (ur.T @ dup)) < 1e-12 * np.linalg.norm(dup)


def test_degenerate_inputs_rejected():  # test_pod.cpp:177-181
    from paper_2402_10488_b200 import capi
    with pytest.raises(capi.RteError, match="zero"):
        device_pod(np.zeros((5, 3)), 1)


def test_wide_matrix():  # test_pod.cpp:183-193
    wide = np.random.default_rng(3).standard_normal((8, 20))
    U, sv = device_pod(wide, 8)
    assert rte().truncation_rank(sv, 1e-14) == 8
    assert ortho_defect(U) < 1e-13
    assert np.linalg.norm(wide - U @ (U.T @ wide)) < 1e-12 * np.linalg.norm(wide)
    np.testing.assert_allclose(sv[:8], np.linalg.svd(wide, compute_uv=False), rtol=1e-12)
