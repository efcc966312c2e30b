"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
one process per case, every hot kernel family of librte_b200.so.

  compute-sanitizer --tool memcheck python scripts/sanitize_cases.py sweep2d_c5plan
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401

from paper_2402_10488_b200 import configs, rte
from tests.problems import homog


def cells(nx, cl, S, seed=3):
    st, ss = configs.c5_coefficients(nx, S, seed=seed)
    mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    px, _ = mesh.cell_points()
    return rte.TransportBatch.from_cells(mesh, rte.chebyshev_legendre(*cl), st, ss, mesh.project(np.ones(px.size)),
                                         inflow=(0.3, 0.1, 0.2, 0.4))


def main(case):
    rng = np.random.default_rng(0)
    if case == "sweep1d":  # K1 sweep1d + 1D DSA (block cyclic reduction) in SI-DSA, plus ROM-free kinetic sweep
        b = rte.TransportBatch(homog(rte, rte.SLAB1D, 0.01, 99.99, 1.0), rte.Mesh.slab_uniform(0, 1, 256),
                               rte.gauss_legendre(16), [[], []])
        rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, max_iters=50))
        b.kinetic_sweep(rng.uniform(0, 1, (2, b.n_dof())))
    elif case == "sweep2d_c4plan":  # CL(16,8) D = 2 plan, 4 samples, apply_L / bbar / kinetic store
        os.environ["RTE_SWEEP_DPL"] = "2"
        b = cells(64, (16, 8), 4)
        assert b.sweep_plan()[0] == 2
        rho = rng.uniform(0, 1, (4, b.n_dof()))
        b.apply_L(rho), b.assemble_rhs(), b.kinetic_sweep(rho)
    elif case == "sweep2d_c5plan":  # CL(32,16) D = 8 plan (the C5 production kernel)
        os.environ["RTE_SWEEP_DPL"] = "8"
        b = cells(64, (32, 16), 4)
        assert b.sweep_plan()[0] == 8
        rho = rng.uniform(0, 1, (4, b.n_dof()))
        b.apply_L(rho), b.fixed_point(rho)
    elif case == "dsa2d":  # multigrid-preconditioned BiCGStab: smoother, coarse cycle, history warm start
        b = cells(64, (8, 4), 2)
        d = rte.DsaOperator(b)
        rhs = rng.uniform(-1, 1, (2, b.n_dof()))
        for _ in range(3):
            d.solve_density(rhs)
        rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=1e-8, max_iters=6, fixed_iters=6))
    elif case == "offline":  # snapshots, POD, projections, ROMSAD, PGMRES on a small pin cell
        train, test = configs.c4_params(6, 4)
        mesh, quad, make = rte.Mesh.rect_uniform(0, 1, 32, 0, 1, 32), rte.chebyshev_legendre(8, 4), configs.pin_cell(rte)
        tb = rte.TransportBatch(make(32), mesh, quad, train)
        sn = rte.collect_snapshots(tb, 3, 1e-8)
        U, sv = rte.pod(rte.snapshot_matrix(tb, sn, "correction"), 8)
        cm = rte.build_reduced_model(tb, U, sv, float(np.sum(sv[8:]) / np.sum(sv)), 1e-8, "c")
        b = rte.TransportBatch(make(32), mesh, quad, test)
        rte.load_rom(b, 1, cm)
        rte.sisa_solve(b, "ROMSAD", rte.SolveConfig(eps_sisa=1e-8, theta=5, max_iters=100,
                                                    eps_romsad=rte.romsad_tolerance(1e-8, cm.discarded_fraction)))
        rte.gmres_solve(b, rte.DsaOperator(b), rte.SolveConfig(gmres_rel_tol=1e-10, max_iters=100))
    else:
        raise SystemExit("unknown case " + case)
    torch.cuda.synchronize()
    print("case", case, "ok")


if __name__ == "__main__":
    main(sys.argv[1])
