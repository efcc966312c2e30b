"""Oracle parity at the BASELINE.json configs' stated sizes:

* C2 (configs[1]): all 512 test samples, SI-DSA / ROMIG / ROMSAD(3,3), device
  offline stage (32 training samples, POD rank 16) shared with the oracle;
* C3 (configs[2]): the full 256^2 CL(16,8) SI-DSA solve against the oracle's
  golden record (tests/tools/make_c3_golden.py: exact SuperLU DSA);
* C4 (configs[3]): all 64 test samples, SI-DSA and ROMSAD(3,5), with the DSA
  solved to 1e-12 and with the inner tolerance tied to the stop test
  (dsa_inner = 1e-3; at 1e-2 iteration counts and logs still match on every
  sample but the converged flux of a few samples drifts to 4e-8, above the
  1e-8 bar: the correction of a diffusive sample is ~100x its delta).

The bar (north_star): identical iteration counts, correction logs and ROMSAD
switch iterations, flux within 1e-8 relative L2 at convergence.  A sample
whose stop (or switch) decision lies within 1e-6 relative of its threshold in
the oracle's own history is flagged *borderline*: there a last-ulp difference
may legitimately flip the decision, so it is reported, not failed.  With
RTE_PARITY_OUT=path the per-config summary is written there as JSON.
"""
import json
import multiprocessing as mp
import os

import numpy as np
import pytest

from paper_2402_10488_b200 import configs
from tests.problems import rel_l2
from tests.tools import parity_workers as pw

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONV_TOL = 1e-8
BORDER = 1e-6


def rte():
    from paper_2402_10488_b200 import rte as m
    return m


def oracle_pool(jobs):
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1, 16)) as pool:
        return pool.map(pw.solve_sample, jobs, chunksize=1)


def margins(hist, eps, theta=None, eps_r=None):
    """Relative distance of the oracle's stop/switch decisions from their thresholds."""
    h = np.asarray(hist)
    m = [abs(h[-1] - eps) / eps]
    if h.size > 1:
        m.append(abs(h[-2] - eps) / eps)
    if theta is not None:
        m += [abs(v - eps_r) / eps_r for v in h[:theta]]
    return float(min(m))


def compare(label, reps, rho, oracle, eps, theta=None, eps_r=None, hist_rtol=1e-6):
    rows, bad = [], []
    for s, (r, o) in enumerate(zip(reps, oracle)):
        sw_o = o["log"].find("D") + 1 if theta is not None else None
        row = {"sample": s, "iters": r.iterations, "iters_oracle": o["iterations"],
               "log_match": r.correction_log == o["log"], "rel_l2": rel_l2(rho[s], o["rho"]),
               "margin": margins(o["history"], eps, theta, eps_r)}
        if theta is not None:
            row["switch"], row["switch_oracle"] = r.switch_iter, (sw_o if sw_o > 0 else -1)
        ok = (row["iters"] == row["iters_oracle"] and row["log_match"] and row["rel_l2"] < CONV_TOL and
              (theta is None or row["switch"] == row["switch_oracle"]))
        if ok and r.iterations == o["iterations"]:
            n = r.iterations
            ok = np.allclose(r.change_history[:n], o["history"][:n], rtol=hist_rtol, atol=1e-14)
        row["ok"] = bool(ok)
        if not ok and row["margin"] >= BORDER:
            bad.append(row)
        rows.append(row)
    summary = {"method": label, "samples": len(rows), "matched": sum(r["ok"] for r in rows),
               "borderline": [r["sample"] for r in rows if r["margin"] < BORDER],
               "max_rel_l2": max(r["rel_l2"] for r in rows),
               "min_margin": min(r["margin"] for r in rows),
               "mean_iterations": float(np.mean([r["iters"] for r in rows]))}
    return summary, bad


def record(name, summaries):
    path = os.environ.get("RTE_PARITY_OUT")
    if not path:
        return
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[name] = summaries
    json.dump(data, open(path, "w"), indent=1)


def test_c2_all_samples_all_methods():
    R = rte()
    train, test = configs.c2_params(32, 512)
    mesh, quad = R.Mesh.slab_uniform(0.0, 1.0, 256), R.gauss_legendre(16)
    eps, eps_train, theta = 1e-8, 1e-8, 3
    tb = R.TransportBatch(configs.two_region_slab(R), mesh, quad, train)
    snaps = R.collect_snapshots(tb, 3, eps_train)
    models = []
    for kind in ("primary", "correction"):
        U, sv = R.pod(R.snapshot_matrix(tb, snaps, kind), 16)
        models.append(R.build_reduced_model(tb, U, sv, float(np.sum(sv[16:]) / np.sum(sv)), eps_train, kind[0]))
    del tb, snaps
    b = R.TransportBatch(configs.two_region_slab(R), mesh, quad, test)
    R.load_rom(b, 0, models[0])
    R.load_rom(b, 1, models[1])
    eps_r = R.romsad_tolerance(eps_train, models[1].discarded_fraction)
    cfg = R.SolveConfig(eps_sisa=eps, norm="abs", theta=theta, eps_romsad=eps_r, max_iters=500)
    dev = {m: R.sisa_solve(b, m, cfg) for m in ("DSA", "ROMIG", "ROMSAD")}
    pm, cm = pw.model_dict(models[0]), pw.model_dict(models[1])
    jobs = [("c2", mu, ["DSA", "ROMIG", "ROMSAD"], eps, "abs", theta, eps_r, pm, cm, True) for mu in test]
    orc = oracle_pool(jobs)
    summaries, bad = [], []
    for m in ("DSA", "ROMIG", "ROMSAD"):
        rho, reps = dev[m]
        sm, bd = compare(m, reps, rho.cpu().numpy(), [o[m] for o in orc], eps,
                         theta if m == "ROMSAD" else None, eps_r)
        summaries.append(sm)
        bad += [dict(r, method=m) for r in bd]
    record("c2_slab_parametric", summaries)
    assert not bad, bad[:5]


def test_c3_full_size_si_dsa_golden():
    g = np.load(os.path.join(ROOT, "tests", "golden", "c3_full_si_dsa.npz"))
    R = rte()
    mesh = R.Mesh.rect_uniform(0, 1, 256, 0, 1, 256)
    from tests.problems import homog
    b = R.TransportBatch(homog(R, R.XY2D, 10 * 0.001, 10 * 0.999, 1.0), mesh, R.chebyshev_legendre(16, 8), [[]])
    summaries = []
    for norm in ("rel", "abs"):
        for inner in (0.0, 1e-3):
            rho, reps = R.sisa_solve(b, "DSA", R.SolveConfig(eps_sisa=1e-8, norm=norm, dsa_inner=inner))
            r = reps[0]
            err = rel_l2(rho.cpu().numpy()[0], g["rho_" + norm])
            summaries.append({"norm": norm, "dsa_inner": inner, "iters": r.iterations,
                              "iters_oracle": int(g["iterations_" + norm]), "rel_l2": err})
            assert r.converged and r.iterations == int(g["iterations_" + norm])
            assert r.n_sweep == int(g["n_sweep_" + norm])
            assert err < CONV_TOL, err
            np.testing.assert_allclose(r.change_history, g["history_" + norm], rtol=1e-6 if inner == 0 else 1e-2,
                                       atol=1e-14)
    record("c3_xy", summaries)


def test_c4_all_samples_si_dsa_and_romsad():
    import torch
    R = rte()
    nx, eps, eps_train, theta = 128, 1e-8, 1e-8, 5
    train, test = configs.c4_params(40, 64)
    mesh, quad, make = R.Mesh.rect_uniform(0, 1, nx, 0, 1, nx), R.chebyshev_legendre(16, 8), configs.pin_cell(R)
    tb = R.TransportBatch(make(nx), mesh, quad, train)
    snaps = R.collect_snapshots(tb, 3, eps_train)
    U, sv = R.pod(R.snapshot_matrix(tb, snaps, "correction"), 20)
    cm = R.build_reduced_model(tb, U, sv, float(np.sum(sv[20:]) / np.sum(sv)), eps_train, "c")
    del tb, snaps, U
    torch.cuda.empty_cache()
    b = R.TransportBatch(make(nx), mesh, quad, test)
    R.load_rom(b, 1, cm)
    eps_r = R.romsad_tolerance(eps_train, cm.discarded_fraction)
    dev = {}
    for inner in (0.0, 1e-3):
        cfg = R.SolveConfig(eps_sisa=eps, norm="abs", theta=theta, eps_romsad=eps_r, max_iters=500, dsa_inner=inner)
        for m in ("DSA", "ROMSAD"):
            rho, reps = R.sisa_solve(b, m, cfg)
            dev[(m, inner)] = (rho.cpu().numpy(), reps)
    jobs = [("c4", mu, ["DSA", "ROMSAD"], eps, "abs", theta, eps_r, None, pw.model_dict(cm), True) for mu in test]
    orc = oracle_pool(jobs)
    summaries, bad = [], []
    for (m, inner), (rho, reps) in dev.items():
        label = m + ("" if inner == 0 else " dsa_inner=%g" % inner)
        sm, bd = compare(label, reps, rho, [o[m] for o in orc], eps, theta if m == "ROMSAD" else None, eps_r,
                         hist_rtol=1e-6 if inner == 0 else 5e-2)
        summaries.append(sm)
        bad += [dict(r, method=label) for r in bd]
    record("c4_xy_pin_cell", summaries)
    assert not bad, bad[:5]
