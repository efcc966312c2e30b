"""Size-independent properties at BASELINE.json's full C5 size (configs[4]:
1024 x 1024 cells, CL(32,16), 16 samples; the oracle cannot run this size):

* linearity of the transport operator L (apply_L) and of the DSA solve;
* batch consistency: a sample solved inside the 16-sample batch equals the
  same sample solved alone (different plan, same operator);
* mirror symmetry: reflecting the coefficient field in x reflects L rho
  (x-odd DG modes change sign), since the quadrature and vacuum boundaries
  are symmetric;
* SI-DSA converges and its final residual ||rho - L rho - bbar||_inf is
  consistent with the stop test.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NX, S = 1024, 16


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def c5():
    import torch
    from paper_2402_10488_b200 import configs, rte
    st, ss = configs.c5_coefficients(NX, S)
    mesh = rte.Mesh.rect_uniform(0, 1, NX, 0, 1, NX)
    quad = rte.chebyshev_legendre(32, 16)
    px, py = mesh.cell_points()
    g = mesh.project(np.ones(px.size))
    batch = rte.TransportBatch.from_cells(mesh, quad, st, ss, g)
    gen = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand((S, batch.n_dof()), dtype=torch.float64, device="cuda", generator=gen)
    y = torch.rand((S, batch.n_dof()), dtype=torch.float64, device="cuda", generator=gen) - 0.5
    return dict(rte=rte, st=st, ss=ss, mesh=mesh, quad=quad, g=g, batch=batch, x=x, y=y)


def test_c5_transport_linearity(c5):
    b, x, y = c5["batch"], c5["x"], c5["y"]
    lhs = b.apply_L(0.7 * x - 1.3 * y).cpu().numpy()
    rhs = (0.7 * b.apply_L(x) - 1.3 * b.apply_L(y)).cpu().numpy()
    assert rel(lhs, rhs) < 1e-12


def test_c5_batch_consistency(c5):
    rte, b, x = c5["rte"], c5["batch"], c5["x"]
    k = 5
    single = rte.TransportBatch.from_cells(c5["mesh"], c5["quad"], c5["st"][k:k + 1], c5["ss"][k:k + 1], c5["g"])
    a = b.apply_L(x)[k].cpu().numpy()
    s1 = single.apply_L(x[k:k + 1])[0].cpu().numpy()
    assert rel(s1, a) < 1e-13


def _mirror_x(v, nx):
    """Reflect a DOF vector [S][cells * 4] in x: cells ix -> nx-1-ix, x-odd modes (a = 1) flip sign."""
    w = v.reshape(v.shape[0], nx, nx, 4)[:, :, ::-1, :].copy()
    w[..., 1] *= -1
    w[..., 3] *= -1
    return w.reshape(v.shape)


def test_c5_mirror_symmetry(c5):
    rte = c5["rte"]
    st = c5["st"][:2].reshape(2, NX, NX)[:, :, ::-1].reshape(2, -1)
    ss = c5["ss"][:2].reshape(2, NX, NX)[:, :, ::-1].reshape(2, -1)
    b2 = rte.TransportBatch.from_cells(c5["mesh"], c5["quad"], c5["st"][:2], c5["ss"][:2], c5["g"])
    bm = rte.TransportBatch.from_cells(c5["mesh"], c5["quad"], st, ss, c5["g"])
    x = c5["x"][:2].cpu().numpy()
    a = _mirror_x(b2.apply_L(x).cpu().numpy(), NX)
    m = bm.apply_L(_mirror_x(x, NX)).cpu().numpy()
    assert rel(m, a) < 1e-12


def test_c5_dsa_linearity(c5):
    rte, b, x, y = c5["rte"], c5["batch"], c5["x"], c5["y"]
    d = rte.DsaOperator(b)
    d.set_tolerance(1e-12, 2000)
    cx, cy = d.solve_density(x), d.solve_density(y)
    cz = d.solve_density(0.7 * x - 1.3 * y)
    assert rel(cz.cpu().numpy(), (0.7 * cx - 1.3 * cy).cpu().numpy()) < 1e-8


def test_c5_si_dsa_converges_with_consistent_residual(c5):
    rte, b = c5["rte"], c5["batch"]
    d = rte.DsaOperator(b)
    d.set_tolerance(1e-10, 2000)
    eps = 1e-7
    rho, reps = rte.sisa_solve(b, "DSA", rte.SolveConfig(eps_sisa=eps, norm="rel", max_iters=40))
    rho = rho.cpu().numpy()
    for s, r in enumerate(reps):
        assert r.converged and r.n_sweep == r.iterations + 1
        assert all(h >= 0 for h in r.change_history) and r.change_history[-1] < eps
        # rho* - rho = -(residual of rho): the returned rho* has residual <= (1 + ||L||) * change
        assert r.final_residual <= 3 * eps * np.abs(rho[s]).max()


def test_c4_full_size_methods_agree():
    """configs[3] at full size (128 x 128 pin cell, CL(16,8), 40 training /
    64 test samples): device offline stage -> ROMSAD, SI-DSA and PGMRES reach
    the same fluxes; ROMSAD never takes more sweeps than SI-DSA needs + theta."""
    from paper_2402_10488_b200 import configs, rte
    from tests.problems import pin_cell
    nx = 128
    train, test = configs.c4_params(40, 64)
    mesh = rte.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
    quad = rte.chebyshev_legendre(16, 8)
    make = pin_cell(rte)
    tb = rte.TransportBatch(make(nx), mesh, quad, train)
    snaps = rte.collect_snapshots(tb, 3, 1e-8)
    assert snaps.converged.all()
    Fc = rte.snapshot_matrix(tb, snaps, "correction")
    Uc, sc = rte.pod(Fc, 20)
    eps_c = float(np.sum(sc[20:]) / np.sum(sc))
    cm = rte.build_reduced_model(tb, Uc, sc, eps_c, 1e-8, "c")
    del tb, snaps, Fc
    b = rte.TransportBatch(make(nx), mesh, quad, test)
    dsa = rte.DsaOperator(b)
    rte.load_rom(b, 1, cm)
    cfg = rte.SolveConfig(eps_sisa=1e-10, norm="rel", theta=5, eps_romsad=rte.romsad_tolerance(1e-8, eps_c),
                          max_iters=500)
    rho_d, rep_d = rte.sisa_solve(b, "DSA", cfg)
    rho_r, rep_r = rte.sisa_solve(b, "ROMSAD", cfg)
    rho_g, rep_g = rte.gmres_solve(b, dsa, rte.SolveConfig(gmres_rel_tol=1e-11, max_iters=500))
    rd, rr, rg = (t.cpu().numpy() for t in (rho_d, rho_r, rho_g))
    assert all(r.converged for r in rep_d + rep_r + rep_g)
    for s in range(len(test)):
        assert rel(rr[s], rd[s]) < 1e-7 and rel(rg[s], rd[s]) < 1e-7
        assert rep_r[s].n_sweep <= rep_d[s].n_sweep + 5


def test_c5_dsa_fast_paths_match_the_plain_solver(monkeypatch):
    """At full C5 size (4 of the samples), three SI-DSA iterations with the
    production DSA (mixed-precision recurrences, history warm start) and with
    the plain one (fp64 recurrences, cold start: RTE_DSA_SLOPPY=0,
    RTE_DSA_WARM=0) agree to the DSA tolerance: the fast paths change the
    cost of each correction, not its value."""
    import torch
    from paper_2402_10488_b200 import configs, rte
    st, ss = configs.c5_coefficients(NX, 4)
    mesh = rte.Mesh.rect_uniform(0, 1, NX, 0, 1, NX)
    g = mesh.project(np.ones(mesh.cell_points()[0].size))
    out = []
    for env in ({}, {"RTE_DSA_SLOPPY": "0", "RTE_DSA_WARM": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        b = rte.TransportBatch.from_cells(mesh, rte.chebyshev_legendre(32, 16), st, ss, g)
        rte.DsaOperator(b).set_tolerance(1e-10, 2000)
        rho, reps = rte.sisa_solve(b, "DSA", rte.SolveConfig(fixed_iters=3, max_iters=3, compute_residual=False))
        out.append((rho.cpu().numpy(), [r.change_history for r in reps]))
        del b, rho
        torch.cuda.empty_cache()
    assert rel(out[0][0], out[1][0]) < 1e-8
    np.testing.assert_allclose(out[0][1], out[1][1], rtol=1e-6)
