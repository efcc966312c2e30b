#!/usr/bin/env python
"""Benchmark of the batched parametric source-iteration hot path on B200.

Workload (BASELINE.json configs[4], the 2D sweep-throughput stress config):
[0,1]^2 at 1024x1024 cells, 256 unique directions (CL(32,16): 8 polar x 32
azimuthal per hemisphere, +/-vz folded), 16 samples with per-cell
sigma_t ~ logU[0.1,100] and c ~ U[0.5,0.99] drawn from seed, q = 1, vacuum.
One step = one SI-DSA iteration over the whole batch: the upwind sweep of
every (cell, direction, sample) with the fused source update and scalar-flux
reduction, the per-sample change norm, and the DSA correction (device
BiCGStab + multigrid to a relative residual of --dsa-tol).  The default run
is the config's "fixed 20 source iterations with DSA" (3 warm-up + 20 timed).
Metric: cell*direction*sample sweep updates per second of the whole step
(updates counted over unique directions); the sweep kernel alone is reported
as sweep_only_updates_per_s and sweep_roofline.

The line also carries `time_to_tol`: time to tolerance per parameter sample
for BASELINE.json configs[0..3] (SI-DSA, ROMIG, ROMSAD; offline stage on the
device), the metric's second half (rank 0 at N=1; --no-ttt skips it).

Contract: `python bench.py --gpus N --steps K --warmup W [--impl reference]`
prints one JSON line (rank 0).  Multi-GPU: samples shard across ranks (weak
scaling, no collective on the data path); timing is on the device, max over
ranks.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOP_PER_UPDATE = 66      # FP64 instructions of the on-the-fly cell solve (sweep2d.cu)
BYTES_PER_UPDATE = 40     # sigma_t + 4 source moments (operand-stream accounting)
PHI, VZ = 32, 16          # CL(32,16) -> 256 unique (vx, vy) slots


METRIC = "sweep cell*direction*sample updates/s (1 SI-DSA iteration per step)"


def bench_config(args, slots):
    """The workload both arms report (BASELINE.json configs[4])."""
    nx, S = args.nx, args.samples
    return {"workload": "c5_2d_sweep_stress", "cells": "%dx%d" % (nx, nx), "directions_unique": slots,
            "quadrature": "CL(%d,%d) folded" % (PHI, VZ), "samples_per_gpu": S,
            "dsa": "device BiCGStab+multigrid to rel. residual %g (reference: SuperLU)" % args.dsa_tol,
            "l2": "inputs (%.1f GB per step) exceed the 126 MB L2" % (S * nx * nx * 4 * 8 * 3 / 1e9)}


def gs_traffic():
    """DRAM bytes per fine-level k_gs launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "dsa_gs_traffic.json")
    try:
        return json.load(open(p)).get("dram_bytes_per_launch")
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi clock / throttle sampling during the timed region."""

    def __init__(self, device):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), "--query-gpu=" + q,
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init(init_group=True):
    """One process per GPU (torchrun env).  The process group is only needed by
    our arm (barrier + max-over-ranks timing); the reference arm runs on rank 0
    alone and the other ranks exit without work."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and init_group:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world, device=None):
    """Max of a per-rank scalar (device-timed milliseconds) over all ranks."""
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda:%d" % device if device is not None else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_seed(base_seed, rank):
    """Weak scaling: every rank owns an independent seeded 16-sample batch
    (samples are independent solves; no data-path collective)."""
    return base_seed + rank


def aggregate_value(updates_per_rank_step, steps, world, ms_max):
    """Whole-job throughput: units of all ranks / max-over-ranks time."""
    return updates_per_rank_step * steps * world / (ms_max * 1e-3)


# ---------------------------------------------------------------------------
# B200 arm

def run_b200(args, rank, world, device):
    import torch
    from paper_2402_10488_b200 import capi, configs, rte
    torch.cuda.set_device(device)
    L = capi.load()
    nx, S = args.nx, args.samples
    mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    quad = rte.chebyshev_legendre(PHI, VZ)
    st, ss = configs.c5_coefficients(nx, S, seed=shard_seed(configs.SEEDS["c5"], rank))
    px, py = mesh.cell_points()
    g = mesh.project(np.ones(px.size))
    batch = rte.TransportBatch.from_cells(mesh, quad, st, ss, g, device=device)
    slots = batch.n_slots()
    upd_step = nx * nx * slots * S
    # DSA availability for XY geometry in this build
    dsa_ok, dsa = True, None
    try:
        dsa = rte.DsaOperator(batch)
        dsa.set_tolerance(args.dsa_tol, 2000)
    except capi.RteError:
        dsa_ok = False
    method = "DSA" if dsa_ok else "SI"

    def solve(iters, guess):
        cfg = rte.SolveConfig(fixed_iters=iters, max_iters=iters, compute_residual=False,
                              initial_guess=guess, check_every=max(iters, 1))
        return rte.sisa_solve(batch, method, cfg)

    rho, _ = solve(args.warmup, None)
    torch.cuda.synchronize()
    L.rte_profile_enable(batch._h, 1)
    L.rte_profile_read(batch._h, None, None)
    clocks = Clocks(device)
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rho, reps = solve(args.steps, rho)
    e1.record()
    torch.cuda.synchronize()
    barrier(world)
    ck = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    NK = len(capi.PROF_KINDS)
    ms_k = (ctypes.c_double * NK)()
    n_k = (ctypes.c_long * NK)()
    capi.check(L.rte_profile_read(batch._h, ms_k, n_k), batch._h)
    L.rte_profile_enable(batch._h, 0)
    ms_max = max_over_ranks(ms_total, world, device)
    value = aggregate_value(upd_step, args.steps, world, ms_max)
    n_dof = batch.n_dof()
    batch = rho = reps = dsa = None  # release the timed context (~55 GB at C5) before the e2e one
    torch.cuda.empty_cache()

    # end-to-end through the C-ABI with host buffers: create (H2D of the
    # problem), K iterations, D2H of the result.
    e2e = None
    if not args.no_e2e:
        st_p = torch.from_numpy(st).pin_memory()
        ss_p = torch.from_numpy(ss).pin_memory()
        out_h = torch.empty((S, n_dof), dtype=torch.float64).pin_memory()
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b2 = rte.TransportBatch.from_cells(mesh, quad, st_p.numpy(), ss_p.numpy(), g, device=device)
        if dsa_ok:
            rte.DsaOperator(b2).set_tolerance(args.dsa_tol, 2000)
        cfg = rte.SolveConfig(fixed_iters=args.steps, max_iters=args.steps, compute_residual=False,
                              check_every=args.steps)
        r2, _ = rte.sisa_solve(b2, method, cfg)
        out_h.copy_(r2)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0, world, device)
        del b2, r2
        h2d = st.nbytes + ss.nbytes + g.nbytes
        e2e = {"value": upd_step * args.steps * world / t_e2e, "unit": "updates/s",
               "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(out_h.numel() * 8 / args.steps),
               "job": "rte_create(host arrays) + rte_dsa_setup + rte_si_solve(%d its) + D2H rho" % args.steps}

    sweep_ms = ms_k[0] / max(n_k[0], 1)
    hbm_peak, peak_kind = peaks()
    achieved = upd_step * BYTES_PER_UPDATE / (sweep_ms * 1e-3) / 1e9
    tf = ctypes.c_double()
    capi.check(L.rte_probe_dfma(device, ctypes.byref(tf)))
    fp64_ach = upd_step * FLOP_PER_UPDATE / (sweep_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "sweep2d_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    gpu_launches = int(sum(n_k[k] for k in range(5)))  # kind 5 is a subset of kind 2
    # dominant kernel of the step: the finest-level DSA smoother half-sweep
    # (k_gs_rb<true,*>).  Algorithmic bytes per own-colour cell (fp32 V-cycle
    # vectors, red-black layout): b read + x write (2 x 48 B), other-colour x
    # read (48 B), (sigma_t, sigma_a) (8 B) = 152 B; per V-cycle of 4 nu
    # half-sweeps one starts from x = 0 (104 B), one also reads x_old and
    # writes delta (248 B), one also reads the coarse correction (176 B).
    cells = S * nx * nx  # the library's smoothing schedule by batch size (dsa2d.cu, dsa2d_setup)
    nu = int(os.environ.get("RTE_DSA_NU", 10 if cells < (1 << 19) else 6 if cells < (4 << 20) else 4))
    gs_cell = (104 + 248 + 176 + (4 * nu - 3) * 152) / (4 * nu)
    gs_ms = ms_k[5] / max(n_k[5], 1)
    gs_bytes = gs_cell * S * nx * nx / 2
    gs_ach = gs_bytes / (gs_ms * 1e-3) / 1e9 if n_k[5] else None
    line = {
        "metric": METRIC,
        "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded mt19937_64, BASELINE configs[4])",
        "config": bench_config(args, slots),
        "e2e": e2e,
        "roofline": ({"bound": "hbm", "achieved": gs_ach, "peak": hbm_peak, "unit": "GB/s",
                      "frac": gs_ach / hbm_peak, "traffic": gs_traffic(),
                      "kernel": "k_gs_rb<true,*> (finest-level DSA red-black block Gauss-Seidel colour half-sweep, fp32, blocked red-black layout)",
                      "per_launch_ms": gs_ms, "bytes_per_launch": gs_bytes,
                      "share_of_step": ms_k[5] / ms_total, "peak_kind": peak_kind} if gs_ach else None),
        "sweep_roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": "sweep2d_kernel", "per_launch_ms": sweep_ms, "bytes_per_update": BYTES_PER_UPDATE,
                     "share_of_step": ms_k[0] / ms_total, "peak_kind": peak_kind,
                     "fp64": {"achieved_tflops": fp64_ach, "peak_tflops": tf.value, "frac": fp64_ach / tf.value,
                              "flop_per_update": FLOP_PER_UPDATE, "peak_kind": "measured DFMA probe"}},
        "kernel_ms": {k: ms_k[i] for i, k in enumerate(capi.PROF_KINDS)},
        "sweep_only_updates_per_s": upd_step / (sweep_ms * 1e-3),
        "kernel_launches": {k: int(n_k[i]) for i, k in enumerate(capi.PROF_KINDS)},
        "gpu_launches": gpu_launches,
        "clocks": ck,
    }
    if rank == 0 and world == 1 and not args.no_ttt:
        line["time_to_tol"] = time_to_tol(device)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_reference(args, budget_s=args.cpu_seconds)
    return line


# ---------------------------------------------------------------------------
# Time to tolerance per parameter sample (the metric's second half) on
# BASELINE.json configs[0..3], product path only (no oracle: parity for these
# runs is tests/tools/run_configs.py and tests/test_gpu_*.py).  Offline stage
# (snapshots, POD, projections) on the device; each online solve timed warm
# (best of `reps` after a cold call) with CUDA events around the batched call.

INNER = {1e-2: "", 0.0: "/dsa_tol_1e-12"}  # xy DSA inner tolerance: rte_si_config.dsa_inner -> label suffix


def time_to_tol(device, reps=2):
    import torch
    from paper_2402_10488_b200 import configs, rte
    torch.cuda.set_device(device)

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        return out, e0.elapsed_time(e1) * 1e-3

    def warm(fn):
        out, best = timed(fn)
        for _ in range(reps):
            out, t = timed(fn)
            best = min(best, t)
        return out, best

    def host_timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        return out, time.perf_counter() - t0

    def summary(reps_, t, S, setup=0.0):
        return {"per_sample_s": t / S, "batch_s": t, "online_setup_s": setup,
                "per_sample_with_setup_s": (t + setup) / S,
                "mean_iterations": float(np.mean([r.iterations for r in reps_])),
                "mean_n_sweep": float(np.mean([r.n_sweep for r in reps_])),
                "converged": int(sum(r.converged for r in reps_)), "samples": S}

    def homog(mod, geom, sig_t, c):
        t0 = mod.CoefficientTerm(absorption_weight=lambda x, y: sig_t * (1 - c),
                                 scattering_weight=lambda x, y: sig_t * c)
        return mod.ProblemDefinition(geom, [t0], lambda x, y: 1.0)

    out = {"timing": "CUDA events around the batched solve call, warm (best of %d after a cold call); "
                     "per_sample_s = batch_s / samples; per_sample_with_setup_s adds the online setup "
                     "(per-parameter system assembly on the host + upload, DSA setup, ROM upload; offline stage "
                     "excluded), SURVEY s8(d)" % reps,
           "xy_dsa": "unsuffixed: each DSA solve to relative residual 1e-2 * eps / change (SPEC.md:174 inner "
                     "tolerance 1e-2 eps_SISA; iteration counts equal the exact-DSA oracle, "
                     "tests/test_gpu_parity.py::test_2d_dsa_inner_tolerance); '/dsa_tol_1e-12': every DSA solve to "
                     "relative residual 1e-12"}
    # C1: 256-cell slab, S16, sigma_t = 100, c = 0.9999, SI-DSA to 1e-8 relative change
    def c1_setup():
        b = rte.TransportBatch(homog(rte, rte.SLAB1D, 100.0, 0.9999), rte.Mesh.slab_uniform(0.0, 1.0, 256),
                               rte.gauss_legendre(16), [[]], device=device)
        rte.DsaOperator(b)
        return b
    b, t_set = host_timed(c1_setup)
    (_, r), t = warm(lambda: rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm="rel")))
    out["c1_slab"] = {"SI-DSA": summary(r, t, 1, t_set)}
    del b
    # C2: two-region slab, 32 training + 512 test samples, POD rank 16
    train, test = configs.c2_params(32, 512)
    mesh, quad = rte.Mesh.slab_uniform(0.0, 1.0, 256), rte.gauss_legendre(16)
    eps_train, window, theta = 1e-8, 3, 3
    t_off = time.perf_counter()
    tb = rte.TransportBatch(configs.two_region_slab(rte), mesh, quad, train, device=device)
    snaps = rte.collect_snapshots(tb, window, eps_train)
    models = []
    for kind in ("primary", "correction"):
        U, sv = rte.pod(rte.snapshot_matrix(tb, snaps, kind), 16, device=device)
        eps_pod = float(np.sum(sv[16:]) / np.sum(sv))
        models.append(rte.build_reduced_model(tb, U, sv, eps_pod, eps_train, kind[0]))
    torch.cuda.synchronize()
    t_off = time.perf_counter() - t_off
    del tb, snaps
    def c2_setup():
        b = rte.TransportBatch(configs.two_region_slab(rte), mesh, quad, test, device=device)
        rte.DsaOperator(b)
        rte.load_rom(b, 0, models[0])
        rte.load_rom(b, 1, models[1])
        return b
    b, t_set = host_timed(c2_setup)
    cfg = rte.SolveConfig(eps_sisa=1e-8, norm="abs", theta=theta, max_iters=500,
                          eps_romsad=rte.romsad_tolerance(eps_train, models[1].discarded_fraction))
    c2 = {"offline_wall_s": t_off, "pod_rank": 16}
    for label, method in (("SI-DSA", "DSA"), ("ROMIG", "ROMIG"), ("ROMSAD", "ROMSAD")):
        (_, r), t = warm(lambda: rte.sisa_solve(b, method, cfg))
        c2[label] = summary(r, t, len(test), t_set)
    out["c2_slab_parametric"] = c2
    del b
    # C3: 256^2 XY, CL(16,8), sigma_t = 10, c = 0.999, SI-DSA to 1e-8 relative change
    def c3_setup():
        b = rte.TransportBatch(homog(rte, rte.XY2D, 10.0, 0.999), rte.Mesh.rect_uniform(0, 1, 256, 0, 1, 256),
                               rte.chebyshev_legendre(16, 8), [[]], device=device)
        rte.DsaOperator(b)
        return b
    b, t_set = host_timed(c3_setup)
    c3 = {}
    for inner in INNER:
        (_, r), t = warm(lambda: rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, norm="rel", dsa_inner=inner)))
        c3["SI-DSA" + INNER[inner]] = summary(r, t, 1, t_set)
    out["c3_xy"] = c3
    del b
    # C4: 128^2 pin cell, 40 training + 64 test samples, POD rank 20 (correction model)
    train, test = configs.c4_params(40, 64)
    mesh, quad, make = rte.Mesh.rect_uniform(0, 1, 128, 0, 1, 128), rte.chebyshev_legendre(16, 8), configs.pin_cell(rte)
    theta = 5
    t_off = time.perf_counter()
    tb = rte.TransportBatch(make(128), mesh, quad, train, device=device)
    snaps = rte.collect_snapshots(tb, window, eps_train)
    U, sv = rte.pod(rte.snapshot_matrix(tb, snaps, "correction"), 20, device=device)
    eps_pod = float(np.sum(sv[20:]) / np.sum(sv))
    cm = rte.build_reduced_model(tb, U, sv, eps_pod, eps_train, "c")
    torch.cuda.synchronize()
    t_off = time.perf_counter() - t_off
    del tb, snaps, U
    torch.cuda.empty_cache()
    def c4_setup():
        b = rte.TransportBatch(make(128), mesh, quad, test, device=device)
        rte.DsaOperator(b)
        rte.load_rom(b, 1, cm)
        return b
    b, t_set = host_timed(c4_setup)
    c4 = {"offline_wall_s": t_off, "pod_rank": 20}
    for inner in INNER:
        cfg = rte.SolveConfig(eps_sisa=1e-8, norm="abs", theta=theta, max_iters=500, dsa_inner=inner,
                              eps_romsad=rte.romsad_tolerance(eps_train, eps_pod))
        for label, method in (("SI-DSA", "DSA"), ("ROMSAD", "ROMSAD")):
            (_, r), t = warm(lambda: rte.sisa_solve(b, method, cfg))
            c4[label + INNER[inner]] = summary(r, t, len(test), t_set)
    out["c4_xy_pin_cell"] = c4
    del b
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# CPU reference arm: the oracle restatement of the reference's SI-DSA
# iteration (sisa.cpp:14-54: rho* = L rho + bbar, one sweep of every direction,
# transport_system.cpp:393-418; rho = rho* + DsaOperator::correct(rho* - rho),
# dsa.cpp:264-277 with the SuperLU factorization built untimed, as our arm's
# DSA setup is) on a bounded sample of the C5 workload.

def _cpu_worker(payload):
    sys.path.insert(0, ROOT)
    import numpy as np
    from oracle import rte_oracle as ro
    win, st, ss, reps = payload
    h = 1.0 / 1024
    mesh = ro.Mesh.rect_uniform(0.0, win * h, win, 0.0, win * h, win)

    def cell(x, y):
        ix = np.clip(np.floor(np.asarray(x) / h).astype(np.int64), 0, win - 1)
        iy = np.clip(np.floor(np.asarray(y) / h).astype(np.int64), 0, win - 1)
        return ix + win * iy
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: (st - ss)[cell(x, y)],
                            scattering_weight=lambda x, y: ss[cell(x, y)])
    p = ro.ProblemDefinition(ro.XY2D, [t0], lambda x, y: 1.0)
    sys_ = ro.TransportSystem(p, mesh, ro.build_dg_space(mesh), ro.chebyshev_legendre(PHI, VZ), [])
    dsa = ro.build_dsa(sys_)
    bbar = sys_.assemble_rhs()
    rho = np.zeros(sys_.n_dof())
    t = time.perf_counter()
    for _ in range(reps):
        rstar = sys_.apply_L(rho) + bbar
        rho = rstar + dsa.correct(rstar - rho)
    return time.perf_counter() - t


def cpu_reference(args, budget_s=20.0):
    import multiprocessing as mp
    from paper_2402_10488_b200 import configs
    win = 64
    st, ss = configs.c5_coefficients(1024, 1, seed=configs.SEEDS["c5"])
    st = st[0].reshape(1024, 1024)
    ss = ss[0].reshape(1024, 1024)
    cores = min(os.cpu_count() or 1, 64)
    # one calibration iteration to size the sample to ~budget_s of CPU time
    probe = _cpu_worker((win, st[:win, :win].ravel().copy(), ss[:win, :win].ravel().copy(), 1))
    reps = max(1, int(budget_s / max(probe, 1e-3) / 2))
    jobs = []
    for k in range(cores):
        oy, ox = (k * win) % 1024, ((k * win) // 1024 * win) % 1024
        jobs.append((win, st[oy:oy + win, ox:ox + win].ravel().copy(), ss[oy:oy + win, ox:ox + win].ravel().copy(),
                     reps))
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        times = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    upd = win * win * (PHI * VZ // 2) * reps * cores
    return {"value": upd / max(times), "unit": "updates/s", "cores": cores, "kind": "port",
            "value_1core": win * win * (PHI * VZ // 2) / probe,
            "sample": "%d SI-DSA iterations (one sweep of all %d directions as the reference does + SuperLU DSA "
                      "correction; updates counted over the %d unique slots as in our arm) on %d independent %dx%d "
                      "windows of C5 sample 0, one per process; one iteration %.3f s"
                      % (reps, PHI * VZ, PHI * VZ // 2, cores, win, win, probe),
            "wall_s": wall}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    cb = cpu_reference(args, budget_s=args.cpu_seconds)
    return {"metric": METRIC, "value": cb["value"], "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic (seeded mt19937_64, BASELINE configs[4])",
            "config": bench_config(args, PHI * VZ // 2),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference C++ not buildable here (Eigen3/LAPACKE absent); CPU oracle restatement timed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)  # configs[4]: a fixed 20 source iterations with DSA
    ap.add_argument("--dsa-tol", type=float, default=1e-8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--nx", type=int, default=1024)
    ap.add_argument("--samples", type=int, default=16)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the C1-C4 time-to-tolerance leg")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    args = ap.parse_args()
    rank, world, local = dist_init(init_group=args.impl != "reference")
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_b200(args, rank, world, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1 and args.impl != "reference":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
