"""Pins the CPU oracle's DSA, source-iteration, GMRES, reduced-model and POD
restatements against the reference's own tests:
  proj/tests/unit/test_dsa.cpp, test_solvers.cpp, test_rom.cpp, test_pod.cpp,
  proj/tests/acceptance/acceptance.cpp criteria 1-2.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro


def homog_slab(sig_t, sig_s, src):  # test_dsa.cpp:12-21
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: sig_t - sig_s, scattering_weight=lambda x, y: sig_s)
    return ro.ProblemDefinition(ro.SLAB1D, [t0], lambda x, y: src)


@pytest.fixture(scope="module")
def demo_slab():  # test_dsa.cpp:24-30
    mesh = ro.Mesh.slab_uniform(0, 10, 400)
    sys = ro.TransportSystem(homog_slab(1.0, 1.0, 0.01), mesh, ro.build_dg_space(mesh), ro.gauss_legendre(16), [])
    return sys, ro.build_dsa(sys)


def test_dsa_linear_and_zero(demo_slab):  # test_dsa.cpp:34-47
    sys, dsa = demo_slab
    assert np.linalg.norm(dsa.correct(np.zeros(sys.n_dof()))) == 0.0
    rng = np.random.default_rng(7)
    a, b = rng.uniform(-1, 1, sys.n_dof()), rng.uniform(-1, 1, sys.n_dof())
    lin = dsa.correct(2.0 * a - 0.5 * b) - (2.0 * dsa.correct(a) - 0.5 * dsa.correct(b))
    assert np.max(np.abs(lin)) < 1e-12
    assert dsa.coupled_dim() == 2 * sys.n_dof()


def test_dsa_eliminated_inverts_solve(demo_slab):  # :49-56
    sys, dsa = demo_slab
    rhs = np.random.default_rng(8).uniform(-1, 1, sys.n_dof())
    back = dsa.apply_eliminated(dsa.solve_density(rhs))
    assert np.max(np.abs(back - rhs)) < 1e-9 * np.max(np.abs(rhs))


def test_dsa_step_is_preconditioned_richardson(demo_slab):  # :58-69
    sys, dsa = demo_slab
    r0 = np.random.default_rng(9).uniform(-1, 1, sys.n_dof())
    bbar = sys.assemble_rhs()
    rho_star = sys.apply_L(r0) + bbar
    step = rho_star + dsa.correct(rho_star - r0)
    resid = bbar - (r0 - sys.apply_L(r0))
    rich = r0 + resid + dsa.solve_density(sys.apply_Ms(resid))
    assert np.max(np.abs(step - rich)) < 1e-12


def test_dsa_iteration_counts(demo_slab):  # :71-93
    sys, dsa = demo_slab
    rho, rep = ro.sisa_solve(sys, ro.DsaStrategy(dsa), ro.SolveConfig(eps_sisa=1e-11))
    assert rep.converged and 10 <= rep.iterations <= 30
    assert rep.n_sweep == rep.iterations + 1
    assert rep.final_residual < 1e-9
    assert rep.initial_guess == "zero" and len(rep.change_history) == rep.iterations
    rho_g, rep_g = ro.gmres_solve(sys, dsa, ro.SolveConfig(gmres_rel_tol=1e-11))
    assert rep_g.converged and rep_g.n_sweep == rep_g.iterations + 3
    assert np.max(np.abs(rho_g - rho)) < 1e-8 * np.max(np.abs(rho))


def test_dsa_thick_diffusive_limit():  # :95-112
    mesh = ro.Mesh.slab_uniform(0, 1, 100)
    sys = ro.TransportSystem(homog_slab(100.0, 100.0, 1.0), mesh, ro.build_dg_space(mesh), ro.gauss_legendre(16), [])
    dsa = ro.build_dsa(sys)
    cfg = ro.SolveConfig(eps_sisa=1e-10, max_iters=600)
    _, rep = ro.sisa_solve(sys, ro.DsaStrategy(dsa), cfg)
    assert rep.converged and rep.n_sweep <= 30
    _, rep2 = ro.sisa_solve(sys, None, cfg)
    assert (not rep2.converged) or rep2.n_sweep > 500


def test_dsa_2d_diffusive_box():  # :114-145
    mesh = ro.Mesh.rect_uniform(0, 1, 12, 0, 1, 12)
    t0 = ro.CoefficientTerm(scattering_weight=lambda x, y: 20.0)
    p = ro.ProblemDefinition(ro.XY2D, [t0], lambda x, y: np.exp(-10 * ((x - .5) ** 2 + (y - .5) ** 2)))
    sys = ro.TransportSystem(p, mesh, ro.build_dg_space(mesh), ro.chebyshev_legendre(8, 4), [])
    dsa = ro.build_dsa(sys)
    assert dsa.coupled_dim() == 3 * sys.n_dof()
    cfg = ro.SolveConfig(eps_sisa=1e-12, max_iters=3000)
    rho, rep = ro.sisa_solve(sys, ro.DsaStrategy(dsa), cfg)
    rho2, rep2 = ro.sisa_solve(sys, None, cfg)
    assert rep.converged and rep2.converged
    assert rep.iterations * 4 < rep2.iterations
    assert np.max(np.abs(rho - rho2)) < 1e-9 * np.max(np.abs(rho))
    rho_g, rep_g = ro.gmres_solve(sys, dsa, ro.SolveConfig())
    assert rep_g.converged and np.max(np.abs(rho_g - rho)) < 1e-8 * np.max(np.abs(rho))


def test_pure_absorber_counts():  # :147-163
    mesh = ro.Mesh.slab_uniform(0, 1, 8)
    sys = ro.TransportSystem(homog_slab(1.0, 0.0, 1.0), mesh, ro.build_dg_space(mesh), ro.gauss_legendre(4), [])
    dsa = ro.build_dsa(sys)
    rho_g, rep_g = ro.gmres_solve(sys, dsa, ro.SolveConfig())
    assert rep_g.converged and rep_g.iterations == 1 and rep_g.n_sweep == 4
    rho_s, rep_s = ro.sisa_solve(sys, None, ro.SolveConfig())
    assert rep_s.iterations == 2 and rep_s.n_sweep == 3
    assert np.max(np.abs(rho_g - rho_s)) < 1e-10 * np.max(np.abs(rho_s))


# ---- test_solvers.cpp ----

@pytest.fixture(scope="module")
def scatter_slab():  # test_solvers.cpp:12-28
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: 0.3, scattering_weight=lambda x, y: 0.8 + 0.1 * x)
    p = ro.ProblemDefinition(ro.SLAB1D, [t0], lambda x, y: 1.0 + 0.2 * x, inflow_left=0.5)
    mesh = ro.Mesh.slab_uniform(0.0, 3.0, 48)
    return ro.TransportSystem(p, mesh, ro.build_dg_space(mesh), ro.gauss_legendre(8), [])


class ZeroCorrection(ro.CorrectionStrategy):  # test_solvers.cpp:30-38
    def correct(self, l, delta):
        return np.zeros(len(delta))

    def last_kind(self):
        return "Z"

    def label(self):
        return "ZERO"


def test_zero_correction_reproduces_si(scatter_slab):  # :42-62
    cfg = ro.SolveConfig(eps_sisa=1e-10)
    rho_si, rep_si = ro.sisa_solve(scatter_slab, None, cfg)
    rho_z, rep_z = ro.sisa_solve(scatter_slab, ZeroCorrection(), cfg)
    assert rep_si.converged and rep_z.converged
    assert rep_si.iterations == rep_z.iterations and rep_si.n_sweep == rep_z.n_sweep
    assert np.max(np.abs(rho_si - rho_z)) == 0.0
    assert rep_si.change_history == rep_z.change_history
    assert rep_si.strategy == "SI" and rep_z.strategy == "ZERO"
    assert rep_si.correction_log == "" and rep_z.correction_log == "Z" * (rep_z.iterations - 1)


def test_exact_guess_one_iteration(scatter_slab):  # :64-86
    cfg = ro.SolveConfig(eps_sisa=1e-10)
    rho, rep0 = ro.sisa_solve(scatter_slab, None, cfg)
    assert rep0.converged and rep0.initial_guess == "zero"
    warm = ro.SolveConfig(eps_sisa=1e-10, initial_guess=rho)
    rho1, rep1 = ro.sisa_solve(scatter_slab, None, warm)
    assert rep1.converged and rep1.iterations == 1 and rep1.n_sweep == 2 and rep1.initial_guess == "supplied"
    assert np.max(np.abs(rho1 - rho)) < 1e-9 * np.max(np.abs(rho))
    _, rep_g = ro.gmres_solve(scatter_slab, None, warm)
    assert rep_g.converged and rep_g.iterations <= 1


def test_iteration_cap(scatter_slab):  # :88-99
    _, rep = ro.sisa_solve(scatter_slab, None, ro.SolveConfig(eps_sisa=1e-13, max_iters=3))
    assert not rep.converged and rep.iterations == 3 and len(rep.change_history) == 3 and rep.final_residual > 0


def test_gmres_restart(scatter_slab):  # :101-121
    rho_si, rep_si = ro.sisa_solve(scatter_slab, None, ro.SolveConfig(eps_sisa=1e-12))
    rho_g, rep_g = ro.gmres_solve(scatter_slab, None, ro.SolveConfig(gmres_rel_tol=1e-12, gmres_restart=5))
    assert rep_g.converged and rep_g.strategy == "GMRES"
    assert np.max(np.abs(rho_g - rho_si)) < 1e-9 * np.max(np.abs(rho_si))
    assert len(rep_g.change_history) > rep_g.iterations
    assert rep_g.change_history[-1] <= 1e-12


def test_residual_consistency(scatter_slab):  # :123-132
    rho, rep = ro.sisa_solve(scatter_slab, None, ro.SolveConfig(eps_sisa=1e-11))
    r = ro.residual_inf(scatter_slab, rho)
    assert r == pytest.approx(rep.final_residual, rel=1e-12) and r < 1e-9


# ---- test_rom.cpp ----

def parametric_slab():  # test_rom.cpp:12-31
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: 0.2, scattering_weight=lambda x, y: 0.5, name="base")
    t1 = ro.CoefficientTerm(psi=lambda mu: mu[0], scattering_weight=lambda x, y: 0.3, name="mu0 scattering")
    return ro.ProblemDefinition(ro.SLAB1D, [t0, t1], lambda x, y: 1.0, inflow_left=0.3, n_params=1,
                                param_ranges=[(0.0, 1.0)])


class Tiny:  # test_rom.cpp:33-41
    def __init__(self):
        self.mesh = ro.Mesh.slab_uniform(0.0, 2.0, 8)
        self.space = ro.build_dg_space(self.mesh)
        self.quad = ro.gauss_legendre(4)
        self.prob = parametric_slab()

    def at(self, mu0):
        return ro.TransportSystem(self.prob, self.mesh, self.space, self.quad, [mu0])


def dense_kinetic_solve(sys):
    return np.linalg.solve(sys.materialize_kinetic(), sys.kinetic_rhs())


def qr_basis(a):
    q, _ = np.linalg.qr(a)
    return q


def dense_term_matrix(sys, k):
    m = sys.kinetic_dim()
    return np.stack([sys.apply_term_kinetic(k, e) for e in np.eye(m)], axis=1)


def test_projections_match_dense():  # test_rom.cpp:74-124
    t = Tiny()
    sys = t.at(0.4)
    u = qr_basis(np.random.default_rng(99).uniform(-1, 1, (sys.kinetic_dim(), 3)))
    sv = np.array([1.0, 0.1, 0.01, 1e-13, 1e-14])
    model = ro.build_reduced_model(sys, u, sv, 1e-9, 1e-11, "p", 0.5)
    assert model.rank == 3 and model.k_affine == 2 and model.n_v == 4 and model.n_dof == sys.n_dof()
    assert model.discarded_fraction == pytest.approx((1e-13 + 1e-14) / sv.sum(), rel=1e-12)
    for k in range(2):
        assert np.max(np.abs(model.a_r[k] - u.T @ dense_term_matrix(sys, k) @ u)) < 1e-12
    assert np.max(np.abs(model.b_r - u.T @ sys.kinetic_rhs())) < 1e-13
    n = sys.n_dof()
    urho = sum(t.quad.weights[j] * u[j * n:(j + 1) * n] for j in range(4))
    uiso = sum(u[j * n:(j + 1) * n] for j in range(4))
    assert np.max(np.abs(model.u_rho - urho)) < 1e-14
    assert np.max(np.abs(model.u_iso - uiso)) < 1e-14
    assert np.max(np.abs(model.assemble(sys) - (model.a_r[0] + 0.4 * model.a_r[1]))) < 1e-13


def test_non_orthonormal_rejected():  # :126-135
    t = Tiny()
    sys = t.at(0.4)
    u = qr_basis(np.random.default_rng(100).uniform(-1, 1, (sys.kinetic_dim(), 3)))
    u[:, 1] *= 1.1
    with pytest.raises(RuntimeError):
        ro.build_reduced_model(sys, u, np.ones(3), 1e-9, 1e-11, "p", 0.0)


def _span_model(t, at, kind):
    snaps = np.stack([dense_kinetic_solve(t.at(m)) for m in (0.2, 0.5, 0.8)], axis=1)
    u = qr_basis(snaps)
    return u, ro.build_reduced_model(t.at(at), u, np.array([1.0, 0.5, 0.25]), 1e-9, 1e-11, kind, 0.0)


def test_reduced_solve_exact_in_span():  # :137-167
    t = Tiny()
    u, model = _span_model(t, 0.5, "p")
    sys05 = t.at(0.5)
    rho_exact = sys05.density_of(dense_kinetic_solve(sys05))
    rho_rom = ro.romig(model, sys05)
    assert np.max(np.abs(rho_rom - rho_exact)) < 1e-10 * np.max(np.abs(rho_exact))
    a_mu = dense_term_matrix(sys05, 0) + 0.5 * dense_term_matrix(sys05, 1)
    c = ro.FullPivLU(model.assemble(sys05)).solve(model.b_r)
    resid = sys05.kinetic_rhs() - a_mu @ (u @ c)
    assert np.max(np.abs(u.T @ resid)) < 1e-11 * np.linalg.norm(sys05.kinetic_rhs())


def test_romig_rejects_singular():  # :169-193
    t = Tiny()
    sys = t.at(0.4)
    broken = ro.ReducedModel(0, 4, sys.n_dof(), 1, 2, "p")
    broken.a_r = [np.zeros((1, 1)), np.zeros((1, 1))]
    broken.u_rho = np.zeros((sys.n_dof(), 1))
    broken.u_iso = np.zeros((sys.n_dof(), 1))
    broken.b_r = np.zeros(1)
    broken.singular_values = np.ones(1)
    with pytest.raises(RuntimeError):
        ro.romig(broken, sys)
    strat = ro.RomsaStrategy(broken)
    strat.setup(sys)
    assert strat.singular
    corr = strat.correct(1, np.full(sys.n_dof(), 0.7))
    assert np.max(np.abs(corr)) == 0.0 and strat.last_kind() == "S"


def test_romsa_matches_dense_formula():  # :195-224
    t = Tiny()
    _, model = _span_model(t, 0.33, "c")
    sys = t.at(0.33)
    strat = ro.RomsaStrategy(model)
    strat.setup(sys)
    delta = np.random.default_rng(17).uniform(-1, 1, sys.n_dof())
    corr = strat.correct(1, delta)
    assert strat.last_kind() == "R"
    rhs_r = model.u_iso.T @ sys.apply_Ms(delta)
    manual = model.u_rho @ np.linalg.solve(model.assemble(sys), rhs_r)
    assert np.max(np.abs(corr - manual)) < 1e-12 * (np.max(np.abs(manual)) + 1.0)
    assert np.max(np.abs(strat.correct(2, np.zeros(sys.n_dof())))) == 0.0


def test_romsad_switching():  # :226-272
    t = Tiny()
    _, model = _span_model(t, 0.5, "c")
    sys = t.at(0.5)
    dsa = ro.build_dsa(sys)
    big = np.ones(sys.n_dof())
    tiny = np.full(sys.n_dof(), 1e-14)
    s = ro.RomsadStrategy(model, dsa, 2, 1e-10, "ROMSAD-test")
    s.setup(sys)
    s.correct(1, big)
    assert s.last_kind() == "R"
    s.correct(2, big)
    assert s.last_kind() == "R"
    corr = s.correct(3, big)
    assert s.last_kind() == "D" and np.max(np.abs(corr - dsa.correct(big))) < 1e-14
    s.correct(1, big)
    assert s.last_kind() == "D"
    s = ro.RomsadStrategy(model, dsa, 10, 1e-10)
    s.setup(sys)
    s.correct(1, tiny)
    assert s.last_kind() == "D"
    s = ro.RomsadStrategy(model, dsa, 10, 1e10)
    s.setup(sys)
    s.correct(1, big)
    assert s.last_kind() == "D"
    assert ro.romsad_tolerance(1e-11, 1e-9) == pytest.approx(1e-10)
    assert ro.romsad_tolerance(1e-9, 1e-11) == pytest.approx(1e-10)
    assert ro.romsad_tolerance(1e-12, 1e-10, 0.5) == pytest.approx(5e-11)


def test_snapshot_correction_identity():  # :274-366
    t = Tiny()
    snaps = []
    for m in (0.3, 0.7):
        sys = t.at(m)
        s = ro.collect_snapshots(sys, ro.build_dsa(sys), window=3, eps_train=1e-12)
        assert s.converged and s.w_mu == 3 and s.n_conv > 3 and s.mu == [m]
        n = sys.n_dof()
        for l in range(1, 4):
            lhs = sys.apply_kinetic(s.converged_f - s.iterates[l - 1])
            msd = sys.apply_Ms(s.delta_rho[l - 1])
            for j in range(4):
                assert np.max(np.abs(lhs[j * n:(j + 1) * n] - msd)) < 1e-9
        snaps.append(s)
    assert ro.primary_matrix(snaps).shape[1] == 2
    assert ro.correction_matrix(snaps).shape[1] == 6
    assert ro.correction_matrix(snaps, 1).shape[1] == 2
    sys = t.at(0.9)
    bad = ro.collect_snapshots(sys, ro.build_dsa(sys), window=3, eps_train=1e-12, max_iters=2)
    assert not bad.converged
    assert ro.primary_matrix(snaps + [bad]).shape[1] == 2


def test_rom_file_round_trip(tmp_path):  # :368-401
    t = Tiny()
    sys = t.at(0.4)
    u = qr_basis(np.random.default_rng(5).uniform(-1, 1, (sys.kinetic_dim(), 2)))
    model = ro.build_reduced_model(sys, u, np.array([2.0, 1.0, 1e-12, 1e-13]), 1e-8, 1e-10, "c", 1.25)
    p = str(tmp_path / "m.rom")
    model.save(p)
    back = ro.ReducedModel.load(p)
    for attr in ("geometry", "n_v", "n_dof", "rank", "k_affine", "kind", "eps_pod", "eps_train",
                 "discarded_fraction", "basis_seconds"):
        assert getattr(back, attr) == getattr(model, attr)
    assert np.array_equal(back.u_rho, model.u_rho) and np.array_equal(back.u_iso, model.u_iso)
    assert all(np.array_equal(a, b) for a, b in zip(back.a_r, model.a_r))
    assert np.array_equal(back.b_r, model.b_r) and np.array_equal(back.singular_values, model.singular_values)
    with pytest.raises(RuntimeError):
        ro.ReducedModel.load(str(tmp_path / "missing.rom"))


# ---- test_pod.cpp ----

def test_truncation_kats():  # test_pod.cpp:56-70
    hs = np.array([0.9, 0.09, 0.009, 0.001])
    assert ro.truncation_rank(hs, 0.01) == 2
    assert ro.truncation_rank(hs, 1e-4) == 4
    gs = np.array([4, 2, 1, 0.5, 0.25])
    assert ro.truncation_rank(gs, 0.5) == 1
    assert ro.truncation_rank(gs, 0.1) == 3
    assert ro.truncation_rank(gs, 1e-16) == 5
    with pytest.raises(ValueError):
        ro.truncation_rank(np.zeros(3), 1e-9)


def synthetic_spectrum():  # test_pod.cpp:15-36 (3000x40, sigma_k = 10^(-k/2))
    rng = np.random.default_rng(42)
    qa, _ = np.linalg.qr(rng.standard_normal((3000, 40)))
    qb, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    s = 10.0 ** (-0.5 * np.arange(40))
    return (qa * s) @ qb.T, s


def test_dense_pod_recovers_spectrum():  # :72-81
    a, s = synthetic_spectrum()
    d = ro.pod_truncate(a, 1e-9)
    assert d.rank == 18 and d.singular_values.size == 40 and d.u.shape[1] == 18
    for k in range(30):
        assert abs(d.singular_values[k] - s[k]) < 1e-12 * s[k] + 1e-15
    assert np.max(np.abs(d.u.T @ d.u - np.eye(18))) < 1e-13


def test_gram_cross_check():  # :146-158
    small = np.random.default_rng(7).standard_normal((50, 10))
    lam = np.linalg.eigvalsh(small.T @ small)[::-1]
    sp = ro.pod_truncate(small, 1e-12)
    assert np.max(np.abs(np.sqrt(np.maximum(lam, 0)) - sp.singular_values)) < 1e-12


def test_rank_deficient():  # :160-175
    base = np.random.default_rng(11).standard_normal((200, 3))
    dup = np.hstack([base, base])
    r = ro.pod_truncate(dup, 1e-15)
    assert r.rank == 3
    assert np.all(r.singular_values[3:] < 1e-13 * r.singular_values[0])
    assert np.linalg.norm(dup - r.u @ (r.u.T @ dup)) < 1e-12 * np.linalg.norm(dup)


def test_degenerate_and_wide():  # :177-193
    with pytest.raises(ValueError, match="zero"):
        ro.pod_truncate(np.zeros((5, 3)), 1e-9)
    with pytest.raises(ValueError):
        ro.pod_truncate(np.zeros((0, 0)), 1e-9)
    wide = np.random.default_rng(3).standard_normal((8, 20))
    r = ro.pod_truncate(wide, 1e-14)
    assert r.rank == 8
    assert np.linalg.norm(wide - r.u @ (r.u.T @ wide)) < 1e-12 * np.linalg.norm(wide)


# ---- acceptance.cpp criteria 1-2 (tiny-instance oracle equivalence) ----

def tiny_problem(geom):  # acceptance.cpp:100-116
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: 0.25, scattering_weight=lambda x, y: 0.6)
    t1 = ro.CoefficientTerm(psi=lambda mu: mu[0], scattering_weight=lambda x, y: 0.2 + 0.1 * x)
    return ro.ProblemDefinition(geom, [t0, t1], lambda x, y: 1.0 + 0.3 * x + 0.1 * y, inflow_left=0.4,
                                n_params=1, param_ranges=[(0.0, 1.0)])


class TinyInstance:  # acceptance.cpp:118-134
    def __init__(self, geom, c1, c2):
        self.mesh = ro.Mesh.slab_uniform(0.0, 1.0, c1) if geom == ro.SLAB1D else \
            ro.Mesh.rect_uniform(0.0, 1.0, c2, 0.0, 1.0, c2)
        self.space = ro.build_dg_space(self.mesh)
        self.quad = ro.gauss_legendre(2) if geom == ro.SLAB1D else ro.chebyshev_legendre(4, 2)
        self.prob = tiny_problem(geom)

    def at(self, mu0):
        return ro.TransportSystem(self.prob, self.mesh, self.space, self.quad, [mu0])


def tiny_correction_model(t):  # acceptance.cpp:141-172
    snaps = []
    for m in (0.2, 0.5, 0.8):
        sys = t.at(m)
        snaps.append(ro.collect_snapshots(sys, ro.build_dsa(sys), window=3, eps_train=1e-12))
    pod = ro.pod_truncate(ro.correction_matrix(snaps, 3), 1e-12)
    return ro.build_reduced_model(t.at(0.2), pod.u, pod.singular_values, 1e-12, 1e-12, "c")


@pytest.mark.parametrize("geom", [ro.SLAB1D, ro.XY2D])
def test_criterion1_tiny_oracle_equivalence(geom):  # acceptance.cpp:182-224
    t = TinyInstance(geom, 4, 3)
    sys = t.at(0.4)
    rho_exact = sys.density_of(dense_kinetic_solve(sys))
    dsa = ro.build_dsa(sys)
    corr = tiny_correction_model(t)
    cfg = ro.SolveConfig(eps_sisa=1e-11)
    tol = 10 * 1e-11
    err = lambda r: np.max(np.abs(r - rho_exact))
    rho_d, rep_d = ro.sisa_solve(sys, None, cfg)
    rho_a, rep_a = ro.sisa_solve(sys, ro.DsaStrategy(dsa), cfg)
    rho_r, rep_r = ro.sisa_solve(sys, ro.RomsadStrategy(corr, dsa, 3, ro.romsad_tolerance(1e-12, 1e-12)), cfg)
    rho_g, rep_g = ro.gmres_solve(sys, dsa, ro.SolveConfig(gmres_rel_tol=1e-12))
    assert rep_d.converged and err(rho_d) < tol
    assert rep_a.converged and err(rho_a) < tol
    assert rep_r.converged and err(rho_r) < tol
    assert rep_g.converged and err(rho_g) < tol


class ExactCorrection(ro.CorrectionStrategy):  # acceptance.cpp:230-255
    def setup(self, system):
        self.sys = system
        self.A = system.materialize_kinetic()

    def correct(self, l, delta):
        n, nv = self.sys.n_dof(), self.sys.quad.n()
        rhs = np.tile(self.sys.apply_Ms(delta), nv)
        return self.sys.density_of(np.linalg.solve(self.A, rhs))

    def last_kind(self):
        return "X"

    def label(self):
        return "EXACT"


@pytest.mark.parametrize("geom", [ro.SLAB1D, ro.XY2D])
def test_criterion2_exact_correction_two_steps(geom):  # acceptance.cpp:257-285
    t = TinyInstance(geom, 16, 4)
    sys = t.at(0.9)
    cfg = ro.SolveConfig(eps_sisa=1e-11)
    rho_si, rep_si = ro.sisa_solve(sys, None, cfg)
    rho_x, rep_x = ro.sisa_solve(sys, ExactCorrection(), cfg)
    assert rep_x.converged and rep_x.iterations <= 2 < rep_si.iterations
    assert np.max(np.abs(rho_x - rho_si)) < 100 * 1e-11
