"""GPU parity of the offline stage: batched snapshot collection
(snapshots.cpp:118-194), POD (pod.cpp, dgesdd in the oracle) and the Galerkin
projections (reduced_model.cpp:106-199) on the device, against the oracle,
plus the end-to-end check that a device-built ROM drives ROMSAD to the same
iteration counts as the oracle-built one."""
import numpy as np
import pytest

from oracle import rte_oracle as ro
from tests.problems import rel_l2, two_region_slab

pytestmark = pytest.mark.gpu

EPS_TRAIN = 1e-8
WINDOW = 3
NCELL = 128


@pytest.fixture(scope="module")
def setup():
    from paper_2402_10488_b200 import configs, rte
    train, test = configs.c2_params(16, 8)
    om = ro.Mesh.slab_uniform(0.0, 1.0, NCELL)
    sp = ro.build_dg_space(om)
    quad = ro.gauss_legendre(16)
    prob = two_region_slab(ro)
    osnaps = []
    for mu in train:
        s = ro.TransportSystem(prob, om, sp, quad, mu)
        osnaps.append(ro.collect_snapshots(s, ro.build_dsa(s), window=WINDOW, eps_train=EPS_TRAIN))
    pm = rte.Mesh.slab(om.boundaries)
    tb = rte.TransportBatch(two_region_slab(rte), pm, rte.gauss_legendre(16), train)
    dsnaps = rte.collect_snapshots(tb, WINDOW, EPS_TRAIN)
    return dict(train=train, test=test, om=om, prob=prob, quad=quad, osnaps=osnaps, tb=tb, dsnaps=dsnaps, pm=pm)


def test_snapshot_collection_parity(setup):
    o, d = setup["osnaps"], setup["dsnaps"]
    fi = d.f_iter.cpu().numpy()
    fc = d.f_conv.cpu().numpy()
    dr = d.drho.cpu().numpy()
    for s, sn in enumerate(o):
        assert bool(d.converged[s]) == sn.converged
        assert int(d.n_iter[s]) == sn.n_conv
        assert int(d.w_mu[s]) == sn.w_mu
        for l in range(sn.w_mu):
            assert rel_l2(fi[s, l], sn.iterates[l]) < 1e-10
            assert rel_l2(dr[s, l], sn.delta_rho[l]) < 1e-9
        assert rel_l2(fc[s], sn.converged_f) < 1e-8


def test_pod_parity(setup):
    from paper_2402_10488_b200 import rte
    o, tb = setup["osnaps"], setup["tb"]
    for kind in ("primary", "correction"):
        Fd = rte.snapshot_matrix(tb, setup["dsnaps"], kind)
        Fo = ro.primary_matrix(o) if kind == "primary" else ro.correction_matrix(o, WINDOW)
        assert Fd.shape[0] == Fo.shape[1]
        assert rel_l2(Fd.cpu().numpy().T, Fo) < 1e-8
        r = min(12, Fo.shape[1])
        U, sig = rte.pod(Fd, r)
        ref = ro.pod_truncate(Fo, 1e-16)
        s0 = ref.singular_values[0]
        big = ref.singular_values > 1e-7 * s0
        np.testing.assert_allclose(sig[big], ref.singular_values[big], rtol=1e-6)
        assert rte.truncation_rank(sig, 1e-6) == ro.truncation_rank(ref.singular_values, 1e-6)
        Ud = U.cpu().numpy().T
        assert np.max(np.abs(Ud.T @ Ud - np.eye(r))) < 1e-12
        # leading subspace agrees (modes well separated from the tail)
        k = int(min(r, np.sum(ref.singular_values > 1e-6 * s0)))
        cos = np.linalg.svd(Ud[:, :k].T @ ref.u[:, :k], compute_uv=False)
        assert cos.min() > 1 - 1e-8


def test_build_reduced_model_parity(setup):
    from paper_2402_10488_b200 import rte
    tb = setup["tb"]
    Fd = rte.snapshot_matrix(tb, setup["dsnaps"], "correction")
    U, sig = rte.pod(Fd, 10)
    dm = rte.build_reduced_model(tb, U, sig, 1e-9, EPS_TRAIN, "c")
    repr_sys = ro.TransportSystem(setup["prob"], setup["om"], ro.build_dg_space(setup["om"]), setup["quad"],
                                  setup["train"][0])
    om_ = ro.build_reduced_model(repr_sys, U.cpu().numpy().T, sig, 1e-9, EPS_TRAIN, "c")
    assert dm.rank == om_.rank and dm.k_affine == om_.k_affine
    for k in range(dm.k_affine):
        assert np.max(np.abs(dm.a_r[k] - om_.a_r[k])) < 1e-10 * max(1.0, np.max(np.abs(om_.a_r[k])))
    assert np.max(np.abs(dm.b_r - om_.b_r)) < 1e-12 * max(1.0, np.max(np.abs(om_.b_r)))
    assert np.max(np.abs(dm.u_rho - om_.u_rho)) < 1e-14 and np.max(np.abs(dm.u_iso - om_.u_iso)) < 1e-13
    assert abs(dm.discarded_fraction - om_.discarded_fraction) < 1e-15


def test_device_offline_drives_romsad_like_oracle(setup):
    """Device ROM (snapshots + POD + projections all on the B200) vs the
    oracle's: same ROMSAD(3,3) iteration counts / logs on test samples."""
    from paper_2402_10488_b200 import rte
    tb, o = setup["tb"], setup["osnaps"]
    Fd = rte.snapshot_matrix(tb, setup["dsnaps"], "correction")
    r = 12
    U, sig = rte.pod(Fd, r)
    eps_pod = float(np.sum(sig[r:]) / np.sum(sig))
    dm = rte.build_reduced_model(tb, U, sig, eps_pod, EPS_TRAIN, "c")
    ref = ro.pod_truncate(ro.correction_matrix(o, WINDOW), 1e-16)
    repr_sys = ro.TransportSystem(setup["prob"], setup["om"], ro.build_dg_space(setup["om"]), setup["quad"],
                                  setup["train"][0])
    om_ = ro.build_reduced_model(repr_sys, ref.u[:, :r], ref.singular_values, eps_pod, EPS_TRAIN, "c")
    test = setup["test"]
    b = rte.TransportBatch(two_region_slab(rte), setup["pm"], rte.gauss_legendre(16), test)
    rte.load_rom(b, 1, dm)
    eps_r = ro.romsad_tolerance(EPS_TRAIN, eps_pod)
    rho, reps = rte.sisa_solve(b, "ROMSAD", rte.SolveConfig(eps_sisa=1e-8, theta=3, eps_romsad=eps_r))
    rho = rho.cpu().numpy()
    for s, mu in enumerate(test):
        sys_ = ro.TransportSystem(setup["prob"], setup["om"], ro.build_dg_space(setup["om"]), setup["quad"], mu)
        o_rho, o_rep = ro.sisa_solve(sys_, ro.RomsadStrategy(om_, ro.build_dsa(sys_), 3, eps_r),
                                     ro.SolveConfig(eps_sisa=1e-8))
        assert reps[s].iterations == o_rep.iterations and reps[s].correction_log == o_rep.correction_log
        assert rel_l2(rho[s], o_rho) < 1e-8


def test_snapshot_store_round_trip(setup, tmp_path):
    """Device snapshots -> RTESNP1 files (snap_%03d.snap) -> SnapshotStore
    reader -> identical training matrices and POD on the device."""
    from paper_2402_10488_b200 import rte
    tb, d = setup["tb"], setup["dsnaps"]
    paths = rte.save_snapshots(tb, d, str(tmp_path / "snaps"), EPS_TRAIN)
    assert len(paths) == tb.S and paths[0].endswith("snap_000.snap")
    hdr = rte.read_snapshot_file(paths[1])
    assert hdr["mu"] == list(setup["train"][1]) and hdr["n_v"] == 16 and hdr["n_dof"] == tb.n_dof()
    back = rte.load_snapshots(str(tmp_path / "snaps"))
    for kind in ("primary", "correction"):
        a = rte.snapshot_matrix(tb, d, kind).cpu().numpy()
        b = rte.snapshot_matrix(tb, back, kind).cpu().numpy()
        assert np.array_equal(a, b)
    Fa = rte.snapshot_matrix(tb, d, "correction")
    Fb = rte.snapshot_matrix(tb, back, "correction")
    (_, sa), (_, sb) = rte.pod(Fa, 8), rte.pod(Fb, 8)
    assert np.array_equal(sa, sb)
