"""Full BASELINE.json configs C1-C4 on the B200: time-to-tolerance per sample
(SI-DSA, ROMIG, ROMSAD) with the offline stage on the device, and oracle
parity (iteration counts, switch iterations, scalar flux) on a subset of
samples.  Writes one JSON document (stdout).

  python tests/tools/run_configs.py [--parity N] [--configs c1,c2,c3,c4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from oracle import rte_oracle as ro
from paper_2402_10488_b200 import configs, reports, rte
from tests.problems import homog, pin_cell, rel_l2, two_region_slab


# XY DSA inner tolerance of the "dsa_inner" legs (rte_si_config.dsa_inner): 1e-3 keeps every
# C3 / C4 flux within 1e-8 of the oracle's exact-DSA solve (the bench's choice); 1e-2 matches the iteration
# counts too but leaves 3 of 16 checked C4 fluxes at 2-3e-8
INNER = 1e-3


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def timed_warm(fn, reps=2):
    """(result, cold seconds, warm seconds): the first call pays lazy module
    loading and allocations; the warm figure is the best of the repeats."""
    out, cold = timed(fn)
    warm = cold
    for _ in range(reps):
        out, t = timed(fn)
        warm = min(warm, t)
    return out, cold, warm


def check_gmres(osys_fn, mus, reps, rho, idx, pre, romig_model=None, tol=1e-11):
    res = []
    for s in idx:
        o = osys_fn(mus[s])
        g0 = ro.romig(romig_model, o) if romig_model is not None else None
        o_rho, o_rep = ro.gmres_solve(o, ro.build_dsa(o) if pre else None,
                                      ro.SolveConfig(gmres_rel_tol=tol, initial_guess=g0))
        res.append({"sample": int(s), "iters_dev": reps[s].iterations, "iters_oracle": o_rep.iterations,
                    "n_sweep_dev": reps[s].n_sweep, "n_sweep_oracle": o_rep.n_sweep,
                    "rel_l2": rel_l2(rho[s], o_rho)})
    ok = all(r["iters_dev"] == r["iters_oracle"] and r["n_sweep_dev"] == r["n_sweep_oracle"] and r["rel_l2"] < 1e-8
             for r in res)
    return {"ok": ok, "samples": res}


def check(osys_fn, mus, reps, rho, strategy_fn, idx, cfg_o):
    res = []
    for s in idx:
        o = osys_fn(mus[s])
        o_rho, o_rep = ro.sisa_solve(o, strategy_fn(o), cfg_o(o))
        res.append({"sample": int(s), "iters_dev": reps[s].iterations, "iters_oracle": o_rep.iterations,
                    "log_match": reps[s].correction_log == o_rep.correction_log,
                    "rel_l2": rel_l2(rho[s], o_rho)})
    ok = all(r["iters_dev"] == r["iters_oracle"] and r["log_match"] and r["rel_l2"] < 1e-8 for r in res)
    return {"ok": ok, "samples": res}


def c1(args):
    mesh = rte.Mesh.slab_uniform(0.0, 1.0, 256)
    prob = lambda m: homog(m, m.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0)
    out = {}
    for norm in ("rel", "abs"):
        (b, tset) = timed(lambda: rte.TransportBatch(prob(rte), mesh, rte.gauss_legendre(16), [[]]))
        (res, t, tw) = timed_warm(lambda: rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm=norm)))
        rho, reps = res
        om = ro.Mesh.slab_uniform(0.0, 1.0, 256)
        par = check(lambda mu: ro.TransportSystem(prob(ro), om, ro.build_dg_space(om), ro.gauss_legendre(16), mu),
                    [[]], reps, rho.cpu().numpy(), lambda o: ro.DsaStrategy(ro.build_dsa(o)), [0],
                    lambda o: ro.SolveConfig(eps_sisa=1e-8, norm=norm))
        out[norm] = {"iterations": reps[0].iterations, "n_sweep": reps[0].n_sweep, "time_to_tol_s": tw,
                     "time_to_tol_cold_s": t, "setup_s": tset, "parity": par}
    return out


def c2(args):
    train, test = configs.c2_params(32, 512)
    mesh = rte.Mesh.slab_uniform(0.0, 1.0, 256)
    quad = rte.gauss_legendre(16)
    eps_train, window, theta = 1e-8, 3, 3
    # offline on the device
    (tb, t0) = timed(lambda: rte.TransportBatch(two_region_slab(rte), mesh, quad, train))
    (snaps, t_snap) = timed(lambda: rte.collect_snapshots(tb, window, eps_train))
    Fp = rte.snapshot_matrix(tb, snaps, "primary")
    Fc = rte.snapshot_matrix(tb, snaps, "correction")
    ((Up, sp), t_pp) = timed(lambda: rte.pod(Fp, 16))
    ((Uc, sc), t_pc) = timed(lambda: rte.pod(Fc, 16))
    eps_p = float(np.sum(sp[16:]) / np.sum(sp))
    eps_c = float(np.sum(sc[16:]) / np.sum(sc))
    (pm, t_bp) = timed(lambda: rte.build_reduced_model(tb, Up, sp, eps_p, eps_train, "p"))
    (cm, t_bc) = timed(lambda: rte.build_reduced_model(tb, Uc, sc, eps_c, eps_train, "c"))
    offline = {"snapshot_s": t_snap, "pod_s": t_pp + t_pc, "projection_s": t_bp + t_bc,
               "rank_primary": 16, "rank_correction": 16, "eps_pod_primary": eps_p, "eps_pod_correction": eps_c,
               "training_converged": int(snaps.converged.sum())}
    (b, tset) = timed(lambda: rte.TransportBatch(two_region_slab(rte), mesh, quad, test))
    rte.load_rom(b, 0, pm)
    rte.load_rom(b, 1, cm)
    eps_r = rte.romsad_tolerance(eps_train, eps_c)
    S = len(test)
    out = {"offline": offline, "samples": S, "setup_s": tset}
    om = ro.Mesh.slab_uniform(0.0, 1.0, 256)
    osys = lambda mu: ro.TransportSystem(two_region_slab(ro), om, ro.build_dg_space(om), ro.gauss_legendre(16), mu)
    opm = ro.ReducedModel(0, 16, b.n_dof(), 16, 4, "p", eps_p, eps_train, pm.u_rho, pm.u_iso, pm.a_r, pm.singular_values,
                          pm.discarded_fraction, pm.b_r)
    ocm = ro.ReducedModel(0, 16, b.n_dof(), 16, 4, "c", eps_c, eps_train, cm.u_rho, cm.u_iso, cm.a_r, cm.singular_values,
                          cm.discarded_fraction, cm.b_r)
    idx = list(range(0, S, max(1, S // args.parity)))[:args.parity] if args.parity > 0 else []
    table = reports.MetricsTable("c2_slab_parametric", [], [("snapshot_seconds", offline["snapshot_s"]),
                                                             ("pod_seconds", offline["pod_s"]),
                                                             ("projection_seconds", offline["projection_s"])])
    for method in ("DSA", "ROMIG", "ROMSAD"):
        cfg = rte.SolveConfig(eps_sisa=1e-8, norm="abs", theta=theta, eps_romsad=eps_r, max_iters=500)
        ((rho, reps), tc, t) = timed_warm(lambda: rte.sisa_solve(b, method, cfg))
        if method == "DSA":
            t_dsa = t
        label, rp, rc = {"DSA": ("DSA", 0, 0), "ROMIG": ("ROMIG", 16, 0), "ROMSAD": ("ROMSAD-3,3", 0, 16)}[method]
        table.rows.append(reports.metrics_row(label, reps, t / t_dsa, rp, rc))
        rho = rho.cpu().numpy()
        if method == "DSA":
            strat = lambda o: ro.DsaStrategy(ro.build_dsa(o))
            cfgo = lambda o: ro.SolveConfig(eps_sisa=1e-8)
        elif method == "ROMIG":
            strat = lambda o: ro.DsaStrategy(ro.build_dsa(o))
            cfgo = lambda o: ro.SolveConfig(eps_sisa=1e-8, initial_guess=ro.romig(opm, o))
        else:
            strat = lambda o: ro.RomsadStrategy(ocm, ro.build_dsa(o), theta, eps_r)
            cfgo = lambda o: ro.SolveConfig(eps_sisa=1e-8)
        out[method] = {"time_to_tol_per_sample_s": t / S, "batch_s": t, "batch_cold_s": tc,
                       "mean_n_sweep": float(np.mean([r.n_sweep for r in reps])),
                       "converged": int(sum(r.converged for r in reps)),
                       "parity": check(osys, test, reps, rho, strat, idx, cfgo)}
    dsa_op = rte.DsaOperator(b)
    for label, rg in (("PGMRES", False), ("PGMRES-ROMIG", True)):
        gcfg = rte.SolveConfig(gmres_rel_tol=1e-11, max_iters=500)
        ((rho, reps), tc, t) = timed_warm(lambda: rte.gmres_solve(b, dsa_op, gcfg, romig_guess=rg))
        rho = rho.cpu().numpy()
        out[label] = {"time_to_tol_per_sample_s": t / S, "batch_s": t, "batch_cold_s": tc,
                      "mean_n_sweep": float(np.mean([r.n_sweep for r in reps])),
                      "converged": int(sum(r.converged for r in reps)),
                      "parity": check_gmres(osys, test, reps, rho, idx[:4], True, opm if rg else None)}
    out["summary_v1"] = reports.serialize_summary(table)  # the reference runner's summary format
    return out


def c3(args):
    nx = 256
    mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    quad = rte.chebyshev_legendre(16, 8)
    prob = lambda m: homog(m, m.XY2D, 10 * 0.001, 10 * 0.999, 1.0)
    (b, tset) = timed(lambda: rte.TransportBatch(prob(rte), mesh, quad, [[]]))
    (d, tdsa) = timed(lambda: rte.DsaOperator(b))
    ((rho, reps), tc, t) = timed_warm(lambda: rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm="rel")),
                                      reps=1)
    r = reps[0]
    out = {"iterations": r.iterations, "n_sweep": r.n_sweep, "final_residual": r.final_residual,
           "time_to_tol_s": t, "time_to_tol_cold_s": tc, "setup_s": tset + tdsa, "history": r.change_history}
    ((_, ireps), _, ti) = timed_warm(lambda: rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm="rel",
                                                                                      dsa_inner=INNER)), reps=1)
    out["dsa_inner=%g" % INNER] = {"iterations": ireps[0].iterations, "time_to_tol_s": ti,
                             "history_max_rel_diff": float(np.max(np.abs(np.array(ireps[0].change_history) -
                                                                         np.array(r.change_history)) /
                                                                  np.array(r.change_history)))}
    ((grho, greps), gtc, gt) = timed_warm(lambda: rte.gmres_solve(b, d, rte.SolveConfig(gmres_rel_tol=1e-11)),
                                          reps=1)
    out["PGMRES"] = {"iterations": greps[0].iterations, "n_sweep": greps[0].n_sweep, "time_to_tol_s": gt,
                     "converged": greps[0].converged}
    if args.c3_oracle:
        om = ro.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
        (o, _) = timed(lambda: ro.TransportSystem(prob(ro), om, ro.build_dg_space(om), ro.chebyshev_legendre(16, 8), []))
        t0 = time.perf_counter()
        o_rho, o_rep = ro.sisa_solve(o, ro.DsaStrategy(ro.build_dsa(o)), ro.SolveConfig(eps_sisa=1e-8, norm="rel"))
        out["parity"] = {"iters_oracle": o_rep.iterations, "rel_l2": rel_l2(rho.cpu().numpy()[0], o_rho),
                         "oracle_s": time.perf_counter() - t0}
    return out


def c4(args):
    nx = 128
    train, test = configs.c4_params(40, 64)
    mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    quad = rte.chebyshev_legendre(16, 8)
    make = pin_cell(rte)
    eps_train, window, theta = 1e-8, 3, 5
    (tb, _) = timed(lambda: rte.TransportBatch(make(nx), mesh, quad, train))
    (snaps, t_snap) = timed(lambda: rte.collect_snapshots(tb, window, eps_train))
    Fc = rte.snapshot_matrix(tb, snaps, "correction")
    ((Uc, sc), t_pod) = timed(lambda: rte.pod(Fc, 20))
    eps_c = float(np.sum(sc[20:]) / np.sum(sc))
    (cm, t_b) = timed(lambda: rte.build_reduced_model(tb, Uc, sc, eps_c, eps_train, "c"))
    del tb, snaps, Fc
    torch.cuda.empty_cache()
    (b, tset) = timed(lambda: rte.TransportBatch(make(nx), mesh, quad, test))
    (dd, tdsa) = timed(lambda: rte.DsaOperator(b))
    rte.load_rom(b, 1, cm)
    eps_r = rte.romsad_tolerance(eps_train, eps_c)
    S = len(test)
    out = {"offline": {"snapshot_s": t_snap, "pod_s": t_pod, "projection_s": t_b, "rank_correction": 20,
                       "eps_pod_correction": eps_c}, "samples": S, "setup_s": tset + tdsa}
    mk = pin_cell(ro)
    om = ro.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    ocm = ro.ReducedModel(1, 128, b.n_dof(), 20, 5, "c", eps_c, eps_train, cm.u_rho, cm.u_iso, cm.a_r,
                          cm.singular_values, cm.discarded_fraction, cm.b_r)
    osys = lambda mu: ro.TransportSystem(mk(nx), om, ro.build_dg_space(om), ro.chebyshev_legendre(16, 8), mu)
    idx = list(range(0, S, max(1, S // args.parity4)))[:args.parity4] if args.parity4 > 0 else []
    table = reports.MetricsTable("c4_xy_pin_cell", [], [("snapshot_seconds", t_snap), ("pod_seconds", t_pod),
                                                         ("projection_seconds", t_b)])
    for method, inner in (("DSA", 0.0), ("ROMSAD", 0.0), ("DSA", INNER), ("ROMSAD", INNER)):
        cfg = rte.SolveConfig(eps_sisa=1e-8, theta=theta, eps_romsad=eps_r, max_iters=500, dsa_inner=inner)
        ((rho, reps), tc, t) = timed_warm(lambda: rte.sisa_solve(b, method, cfg), reps=1)
        if method == "DSA" and inner == 0:
            t_dsa = t
        label = ("DSA" if method == "DSA" else "ROMSAD-3,5") + ("" if inner == 0 else " dsa_inner=%g" % inner)
        table.rows.append(reports.metrics_row(label, reps, t / t_dsa, 0, 0 if method == "DSA" else 20))
        rho = rho.cpu().numpy()
        strat = (lambda o: ro.DsaStrategy(ro.build_dsa(o))) if method == "DSA" else \
            (lambda o: ro.RomsadStrategy(ocm, ro.build_dsa(o), theta, eps_r))
        # the oracle always solves the DSA exactly (SuperLU): the inner-tolerance
        # runs must reproduce its iteration counts and correction logs
        out[method + ("" if inner == 0 else " dsa_inner=%g" % inner)] = {"time_to_tol_per_sample_s": t / S, "batch_s": t, "batch_cold_s": tc,
                       "mean_n_sweep": float(np.mean([r.n_sweep for r in reps])),
                       "converged": int(sum(r.converged for r in reps)),
                       "switch_iters": [r.switch_iter for r in reps[:8]],
                       "parity": check(osys, test, reps, rho, strat, idx, lambda o: ro.SolveConfig(eps_sisa=1e-8))
                       if idx else None}
    ((grho, greps), gtc, gt) = timed_warm(lambda: rte.gmres_solve(b, dd, rte.SolveConfig(gmres_rel_tol=1e-11,
                                                                                         max_iters=500)), reps=1)
    out["PGMRES"] = {"time_to_tol_per_sample_s": gt / S, "batch_s": gt, "batch_cold_s": gtc,
                     "mean_n_sweep": float(np.mean([r.n_sweep for r in greps])),
                     "converged": int(sum(r.converged for r in greps)),
                     "parity": check_gmres(osys, test, greps, grho.cpu().numpy(), idx[:1], True) if idx else None}
    out["summary_v1"] = reports.serialize_summary(table)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--parity", type=int, default=16)
    ap.add_argument("--parity4", type=int, default=2)
    ap.add_argument("--c3-oracle", action="store_true")
    args = ap.parse_args()
    res = {}
    for name in args.configs.split(","):
        t0 = time.perf_counter()
        res[name] = globals()[name](args)
        res[name]["wall_s"] = time.perf_counter() - t0
        print("[%s done in %.1f s]" % (name, res[name]["wall_s"]), file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
