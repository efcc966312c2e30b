"""Generate tests/golden/*.npz from the CPU oracle (the reference itself cannot
be built here: Eigen3/LAPACKE absent).  The fixtures pin the oracle against
regressions and give the GPU tests fixed expected vectors.

  python tests/tools/make_golden.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np

from oracle import rte_oracle as ro
from tests.problems import homog, prob2d_const, two_region_slab

OUT = os.path.join(ROOT, "tests", "golden")


def c1():
    mesh = ro.Mesh.slab_uniform(0.0, 1.0, 256)
    sys_ = ro.TransportSystem(homog(ro, ro.SLAB1D, 100.0 * (1 - 0.9999), 100.0 * 0.9999, 1.0), mesh,
                              ro.build_dg_space(mesh), ro.gauss_legendre(16), [])
    rho, rep = ro.sisa_solve(sys_, ro.DsaStrategy(ro.build_dsa(sys_)), ro.SolveConfig(eps_sisa=1e-10))
    rng = np.random.default_rng(2024)
    probe = rng.uniform(0, 1, sys_.n_dof())
    np.savez_compressed(os.path.join(OUT, "c1_slab_si_dsa.npz"), rho=rho, history=np.array(rep.change_history),
                        iterations=rep.iterations, n_sweep=rep.n_sweep, probe=probe, L_probe=sys_.apply_L(probe),
                        bbar=sys_.assemble_rhs())


def box2d():
    mesh = ro.Mesh.rect_uniform(0.0, 1.2, 9, -0.5, 1.0, 7)
    p = prob2d_const(ro, 0.4, 0.8, lambda x, y: 1.0 + x + 0.5 * y, inflow_left=1.0, inflow_bottom=0.7,
                     inflow_right=0.2, inflow_top=0.3)
    sys_ = ro.TransportSystem(p, mesh, ro.build_dg_space(mesh), ro.chebyshev_legendre(8, 4), [])
    rng = np.random.default_rng(7)
    probe = rng.uniform(-1, 1, sys_.n_dof())
    rho, rep = ro.sisa_solve(sys_, ro.DsaStrategy(ro.build_dsa(sys_)), ro.SolveConfig(eps_sisa=1e-10))
    np.savez_compressed(os.path.join(OUT, "box2d_inflow.npz"), probe=probe, L_probe=sys_.apply_L(probe),
                        bbar=sys_.assemble_rhs(), f0=sys_.sweep_direction(0, probe), rho=rho,
                        iterations=rep.iterations, history=np.array(rep.change_history))


def c2_small():
    from paper_2402_10488_b200 import configs
    train, test = configs.c2_params(8, 4)
    mesh = ro.Mesh.slab_uniform(0.0, 1.0, 64)
    sp = ro.build_dg_space(mesh)
    quad = ro.gauss_legendre(16)
    prob = two_region_slab(ro)
    snaps = []
    for mu in train:
        s = ro.TransportSystem(prob, mesh, sp, quad, mu)
        snaps.append(ro.collect_snapshots(s, ro.build_dsa(s), window=3, eps_train=1e-8))
    pod = ro.pod_truncate(ro.correction_matrix(snaps, 3), 1e-16)
    r = 8
    eps_pod = float(np.sum(pod.singular_values[r:]) / np.sum(pod.singular_values))
    model = ro.build_reduced_model(ro.TransportSystem(prob, mesh, sp, quad, train[0]), pod.u[:, :r],
                                   pod.singular_values, eps_pod, 1e-8, "c")
    its, logs, rhos = [], [], []
    eps_r = ro.romsad_tolerance(1e-8, eps_pod)
    for mu in test:
        s = ro.TransportSystem(prob, mesh, sp, quad, mu)
        rho, rep = ro.sisa_solve(s, ro.RomsadStrategy(model, ro.build_dsa(s), 3, eps_r), ro.SolveConfig(eps_sisa=1e-8))
        its.append(rep.iterations)
        logs.append(rep.correction_log)
        rhos.append(rho)
    np.savez_compressed(os.path.join(OUT, "c2_small_romsad.npz"), train=np.array(train), test=np.array(test),
                        sigma=pod.singular_values, n_conv=np.array([s.n_conv for s in snaps]),
                        iterations=np.array(its), logs=np.array(logs), rho=np.array(rhos), eps_pod=eps_pod,
                        rank=r)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    c1()
    box2d()
    c2_small()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
