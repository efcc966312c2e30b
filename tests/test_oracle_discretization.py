"""Pins the CPU oracle against the reference's own known-answer tests for the
discretization and the transport operator.

Restates, in pytest form, the checks in
  proj/tests/unit/test_quadrature.cpp, test_dg_space.cpp, test_sweep.cpp,
  test_assembly.cpp
against oracle/rte_oracle (the C++ restatement).  Tolerances are the
reference's.
"""
import numpy as np
import pytest

from oracle import rte_oracle as ro

# test_quadrature.cpp:14-21 -- published 16-point GL table (positive abscissas).
GL16_NODES = [0.0950125098376374, 0.2816035507792589, 0.4580167776572274, 0.6178762444026438,
              0.7554044083550030, 0.8656312023878318, 0.9445750230732326, 0.9894009349916499]
GL16_WEIGHTS = [0.1894506104550685, 0.1826034150449236, 0.1691565193950025, 0.1495959888165767,
                0.1246289712555339, 0.0951585116824928, 0.0622535239386479, 0.0271524594117541]


def moment(q, px, py, pz):
    d = q.directions
    return float(np.sum(q.weights * d[:, 0] ** px * d[:, 1] ** py * d[:, 2] ** pz))


def test_slab_rule_matches_published_table():  # test_quadrature.cpp:33-51
    q = ro.gauss_legendre(16)
    assert q.n() == 16 and q.geometry == ro.SLAB1D
    for j in range(16):
        v, w = q.vx(j), q.weights[j]
        k = [i for i in range(8) if abs(abs(v) - GL16_NODES[i]) < 1e-10]
        assert len(k) == 1
        k = k[0]
        assert abs(abs(v) - GL16_NODES[k]) < 1e-13
        assert abs(w - 0.5 * GL16_WEIGHTS[k]) < 1e-13
        assert q.vy(j) == 0.0 and q.vz(j) == 0.0


def test_raw_nodes_sum_and_symmetry():  # :53-62
    x, w = ro.gauss_legendre_nodes(16)
    assert abs(w.sum() - 2.0) < 1e-14
    for i in range(16):
        assert abs(x[i] + x[15 - i]) < 1e-14
        assert abs(w[i] - w[15 - i]) < 1e-14


def test_cl42_corner_directions():  # :64-82
    q = ro.chebyshev_legendre(4, 2)
    assert q.n() == 8 and q.geometry == ro.XY2D
    c = 1.0 / np.sqrt(3.0)
    seen = [0] * 8
    for j in range(8):
        assert abs(q.weights[j] - 0.125) < 1e-15
        for comp in range(3):
            assert abs(abs(q.directions[j, comp]) - c) < 1e-14
        seen[int(q.vx(j) > 0) + 2 * int(q.vy(j) > 0) + 4 * int(q.vz(j) > 0)] += 1
    assert seen == [1] * 8


def test_product_rule_orders_azimuth_fastest():  # :84-95
    q = ro.chebyshev_legendre(4, 2)
    for j in range(1, 4):
        assert q.vz(j) == q.vz(0)
    assert q.vz(4) != q.vz(0)
    for j in range(4):
        assert q.vx(j) == q.vx(j + 4) and q.vy(j) == q.vy(j + 4)
        assert abs(q.vz(j) + q.vz(j + 4)) < 1e-15


@pytest.mark.parametrize("rule", [("gl", 16), ("gl", 8), ("cl", 30, 6), ("cl", 16, 4), ("cl", 40, 6),
                                  ("cl", 16, 8), ("cl", 32, 16)])
def test_moment_identities(rule):  # :97-122 (+ the BASELINE CL(16,8), CL(32,16))
    q = ro.gauss_legendre(rule[1]) if rule[0] == "gl" else ro.chebyshev_legendre(rule[1], rule[2])
    assert abs(moment(q, 0, 0, 0) - 1.0) < 1e-13
    assert abs(moment(q, 1, 0, 0)) < 1e-13
    assert abs(moment(q, 2, 0, 0) - 1.0 / 3.0) < 1e-13
    if q.geometry == ro.XY2D:
        assert abs(moment(q, 0, 1, 0)) < 1e-13
        assert abs(moment(q, 0, 0, 1)) < 1e-13
        assert abs(moment(q, 0, 2, 0) - 1.0 / 3.0) < 1e-13
        assert abs(moment(q, 0, 0, 2) - 1.0 / 3.0) < 1e-13
        assert abs(moment(q, 1, 1, 0)) < 1e-13
        assert abs(moment(q, 1, 0, 1)) < 1e-13
        r = np.sum(q.directions ** 2, axis=1)
        assert np.max(np.abs(r - 1.0)) < 1e-13
    assert abs(moment(q, 4, 0, 0) - 0.2) < 1e-13


def test_weights_positive():  # :124-130
    for q in (ro.gauss_legendre(2), ro.gauss_legendre(16), ro.chebyshev_legendre(4, 2),
              ro.chebyshev_legendre(30, 6)):
        assert np.all(q.weights > 0)


# ---- dg space (test_dg_space.cpp) ----

def test_projection_affine_slab():  # test_dg_space.cpp:34-51
    mesh = ro.Mesh.slab([0.0, 0.3, 0.7, 1.2, 2.0])
    sp = ro.build_dg_space(mesh)
    f = lambda x, y: 2.0 - 3.0 * x
    c = ro.project(mesh, sp, f)
    for cell in range(4):
        a, h = mesh.left(cell), mesh.width(cell)
        for t in (0.1, 0.5, 0.93):
            x = a + t * h
            assert abs(ro.evaluate(mesh, sp, c, cell, x) - f(x, 0)) < 1e-13
    avg = ro.cell_averages(mesh, sp, c)
    for cell in range(4):
        assert abs(avg[cell] - f(mesh.center(cell), 0)) < 1e-13


def test_projection_bilinear_2d():  # :53-71
    mesh = ro.Mesh.rect_uniform(0.0, 1.2, 3, -0.5, 1.0, 2)
    sp = ro.build_dg_space(mesh)
    assert sp.n_local == 4 and sp.n_dof == 24
    f = lambda x, y: 1.0 + 2.0 * x - y + 0.5 * x * y
    c = ro.project(mesh, sp, f)
    for iy in range(2):
        for ix in range(3):
            cell = ix + 3 * iy
            for tx in (0.2, 0.8):
                for ty in (0.3, 0.6):
                    x = mesh.cell_x0(ix) + tx * mesh.hx()
                    y = mesh.cell_y0(iy) + ty * mesh.hy()
                    assert abs(ro.evaluate(mesh, sp, c, cell, x, y) - f(x, y)) < 1e-13


def test_constant_projects_onto_first_mode():  # :73-82
    mesh = ro.Mesh.slab_uniform(0.0, 3.0, 3)
    sp = ro.build_dg_space(mesh)
    c = ro.project(mesh, sp, lambda x, y: 5.0)
    assert np.max(np.abs(c[0::2] - 5.0)) < 1e-14
    assert np.max(np.abs(c[1::2])) < 1e-14


def test_local_layout_2d():  # :84-96
    mesh = ro.Mesh.rect_uniform(0.0, 1.0, 1, 0.0, 1.0, 1)
    sp = ro.build_dg_space(mesh)
    cx = ro.project(mesh, sp, lambda x, y: x)
    assert abs(cx[2]) < 1e-14 and abs(cx[3]) < 1e-14 and abs(cx[1]) > 1e-3
    cy = ro.project(mesh, sp, lambda x, y: y)
    assert abs(cy[1]) < 1e-14 and abs(cy[3]) < 1e-14 and abs(cy[2]) > 1e-3


def test_quadratic_rejected():  # :98-101
    with pytest.raises(ValueError):
        ro.build_dg_space(ro.Mesh.slab_uniform(0.0, 1.0, 2), 2)


# ---- sweep (test_sweep.cpp) ----

def homogeneous(geom, sig_a, sig_s, src):
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: sig_a, scattering_weight=lambda x, y: sig_s)
    return ro.ProblemDefinition(geometry=geom, terms=[t0], source=lambda x, y: src)


def test_sweep_inverts_forward_operator():  # test_sweep.cpp:26-53
    rng = np.random.default_rng(1)
    mesh = ro.Mesh.slab([0.0, 0.2, 0.9, 1.4, 2.0, 2.3])
    sys = ro.TransportSystem(homogeneous(ro.SLAB1D, 0.4, 0.8, 1.0), mesh, ro.build_dg_space(mesh),
                             ro.gauss_legendre(4), [])
    for j in range(4):
        rhs = rng.uniform(-1, 1, sys.n_dof())
        back = sys.apply_streaming_collision(j, sys.sweep_direction(j, rhs))
        assert np.max(np.abs(back - rhs)) < 1e-12
    mesh = ro.Mesh.rect_uniform(0.0, 1.0, 4, 0.0, 1.5, 3)
    sys = ro.TransportSystem(homogeneous(ro.XY2D, 0.4, 0.8, 1.0), mesh, ro.build_dg_space(mesh),
                             ro.chebyshev_legendre(4, 2), [])
    for j in range(8):
        rhs = rng.uniform(-1, 1, sys.n_dof())
        back = sys.apply_streaming_collision(j, sys.sweep_direction(j, rhs))
        assert np.max(np.abs(back - rhs)) < 1e-12


def test_sweep_counter():  # :55-72
    mesh = ro.Mesh.slab_uniform(0.0, 1.0, 8)
    sys = ro.TransportSystem(homogeneous(ro.SLAB1D, 0.5, 0.5, 1.0), mesh, ro.build_dg_space(mesh),
                             ro.gauss_legendre(4), [])
    sc = ro.SweepCounter()
    rho = np.random.default_rng(2).uniform(-1, 1, sys.n_dof())
    sys.apply_L(rho, sc)
    assert sc.sweeps == 1
    sys.assemble_rhs(sc)
    assert sc.sweeps == 2
    sys.kinetic_sweep(rho, sc)
    assert sc.sweeps == 3
    sys.apply_L(rho, None)
    assert sc.sweeps == 3


def test_pure_absorber_analytic_attenuation():  # :74-99
    sig, g_in = 2.0, 1.5
    mesh = ro.Mesh.slab_uniform(0.0, 1.0, 64)
    sp = ro.build_dg_space(mesh)
    p = homogeneous(ro.SLAB1D, sig, 0.0, 0.0)
    p.inflow_left = g_in
    quad = ro.gauss_legendre(4)
    sys = ro.TransportSystem(p, mesh, sp, quad, [])
    for j in range(4):
        v = quad.vx(j)
        f = sys.sweep_direction(j, sys.boundary_source(j))
        avg = ro.cell_averages(mesh, sp, f)
        if v < 0:
            assert np.max(np.abs(avg)) == 0.0
        else:
            for i in range(0, 64, 13):
                x0, h = mesh.left(i), mesh.width(i)
                exact = g_in * v / (sig * h) * (np.exp(-sig * x0 / v) - np.exp(-sig * (x0 + h) / v))
                assert abs(avg[i] - exact) < 1e-3 * g_in


def test_upwind_causality_2d():  # :101-125
    mesh = ro.Mesh.rect_uniform(0.0, 1.0, 8, 0.0, 1.0, 8)
    sp = ro.build_dg_space(mesh)
    quad = ro.chebyshev_legendre(4, 2)
    sys = ro.TransportSystem(homogeneous(ro.XY2D, 1.0, 0.0, 0.0), mesh, sp, quad, [])
    sx, sy = 3, 4
    rhs = np.zeros(sys.n_dof())
    rhs[sp.dof(sx + 8 * sy, 0)] = 1.0
    for j in range(quad.n()):
        f = sys.sweep_direction(j, rhs)
        dx = 1 if quad.vx(j) > 0 else -1
        dy = 1 if quad.vy(j) > 0 else -1
        for iy in range(8):
            for ix in range(8):
                down = (ix >= sx if dx > 0 else ix <= sx) and (iy >= sy if dy > 0 else iy <= sy)
                if not down:
                    cell = ix + 8 * iy
                    assert np.all(f[4 * cell:4 * cell + 4] == 0.0)


def test_symmetric_slab_symmetric_density():  # :127-149
    n = 40
    mesh = ro.Mesh.slab_uniform(0.0, 1.0, n)
    sp = ro.build_dg_space(mesh)
    p = homogeneous(ro.SLAB1D, 0.3, 1.2, 0.0)
    p.source = lambda x, y: np.exp(-30.0 * (x - 0.5) * (x - 0.5))
    p.inflow_left = 0.8
    p.inflow_right = 0.8
    sys = ro.TransportSystem(p, mesh, sp, ro.gauss_legendre(8), [])
    bbar = sys.assemble_rhs()
    rho = np.zeros(sys.n_dof())
    for _ in range(4000):
        nxt = sys.apply_L(rho) + bbar
        d = np.max(np.abs(nxt - rho))
        rho = nxt
        if d < 1e-13:
            break
    avg = ro.cell_averages(mesh, sp, rho)
    for i in range(n // 2):
        assert abs(avg[i] - avg[n - 1 - i]) < 1e-11


# ---- assembly (test_assembly.cpp) ----

def prob1d():  # test_assembly.cpp:11-22
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: 0.3, scattering_weight=lambda x, y: 0.6 + 0.1 * x)
    return ro.ProblemDefinition(ro.SLAB1D, [t0], lambda x, y: 1.0 + x, inflow_left=2.0, inflow_right=0.5)


def prob2d():  # :24-37
    t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: 0.2 + 0.1 * x * y,
                            scattering_weight=lambda x, y: 0.5 + 0.2 * x + 0.1 * y)
    return ro.ProblemDefinition(ro.XY2D, [t0], lambda x, y: 1.0 + x + 0.5 * y, inflow_left=1.0,
                                inflow_bottom=0.7)


def prob_affine(geom):  # :40-55
    p = prob1d() if geom == ro.SLAB1D else prob2d()
    p.n_params = 2
    p.param_ranges = [(0.1, 2.0), (0.1, 2.0)]
    p.terms.append(ro.CoefficientTerm(psi=lambda mu: mu[0], absorption_weight=lambda x, y: 0.05 + 0.02 * x,
                                      name="abs"))
    p.terms.append(ro.CoefficientTerm(psi=lambda mu: mu[1] * mu[1],
                                      scattering_weight=lambda x, y: 0.3 + 0.1 * y + 0.05 * x, name="scat"))
    return p


def make_instance(two_d):  # :65-77
    if two_d:
        mesh = ro.Mesh.rect_uniform(0.0, 1.2, 3, -0.5, 1.0, 3)
        return ro.TransportSystem(prob2d(), mesh, ro.build_dg_space(mesh), ro.chebyshev_legendre(4, 2), [])
    mesh = ro.Mesh.slab([0.0, 0.3, 0.7, 1.2, 2.0])
    return ro.TransportSystem(prob1d(), mesh, ro.build_dg_space(mesh), ro.gauss_legendre(4), [])


@pytest.mark.parametrize("two_d", [False, True])
def test_fixed_point_matches_dense_kinetic_solve(two_d):  # :81-107
    sys = make_instance(two_d)
    A = sys.materialize_kinetic()
    b = sys.kinetic_rhs()
    f = np.linalg.solve(A, b)
    rho_exact = sys.density_of(f)
    bbar = sys.assemble_rhs()
    rho = np.zeros(sys.n_dof())
    for _ in range(4000):
        nxt = sys.apply_L(rho) + bbar
        d = np.max(np.abs(nxt - rho))
        rho = nxt
        if d < 1e-14:
            break
    assert np.max(np.abs(rho - rho_exact)) < 1e-11
    fk = sys.kinetic_sweep(rho)
    assert np.max(np.abs(sys.apply_kinetic(fk) - b)) < 1e-11


def test_dense_matches_operator():  # :109-119
    sys = make_instance(False)
    A = sys.materialize_kinetic()
    rng = np.random.default_rng(3)
    for _ in range(3):
        u = rng.uniform(-1, 1, sys.kinetic_dim())
        assert np.max(np.abs(sys.apply_kinetic(u) - A @ u)) < 1e-12


@pytest.mark.parametrize("geom", [ro.SLAB1D, ro.XY2D])
def test_affine_reconstruction(geom):  # :121-146
    p = prob_affine(geom)
    mesh = ro.Mesh.slab([0.0, 0.5, 1.0, 2.0]) if geom == ro.SLAB1D else ro.Mesh.rect_uniform(0, 1, 2, 0, 1, 2)
    quad = ro.gauss_legendre(4) if geom == ro.SLAB1D else ro.chebyshev_legendre(4, 2)
    rng = np.random.default_rng(4)
    for mu in ([0.3, 1.4], [1.7, 0.2]):
        sys = ro.TransportSystem(p, mesh, ro.build_dg_space(mesh), quad, mu)
        assert sys.n_terms() == 3 and sys.psi(0) == 1.0 and sys.psi(1) == mu[0] and sys.psi(2) == mu[1] * mu[1]
        u = rng.uniform(-1, 1, sys.kinetic_dim())
        acc = sum(sys.psi(k) * sys.apply_term_kinetic(k, u) for k in range(3))
        assert np.max(np.abs(acc - sys.apply_kinetic(u))) < 1e-12


def test_density_and_mass_operators():  # :148-176
    sys = make_instance(True)
    nd, nv = sys.n_dof(), sys.quad.n()
    rng = np.random.default_rng(5)
    f = rng.uniform(-1, 1, nv * nd)
    expect = sum(sys.quad.weights[j] * f[j * nd:(j + 1) * nd] for j in range(nv))
    assert np.max(np.abs(sys.density_of(f) - expect)) < 1e-13
    r = rng.uniform(-1, 1, nd)
    ms, mt = sys.apply_Ms(r), sys.apply_Mt(r)
    for cell in range(sys.mesh.cell_count()):
        seg = r[4 * cell:4 * cell + 4]
        assert np.linalg.norm(ms[4 * cell:4 * cell + 4] - sys.Ms_block(cell) @ seg) < 1e-13
        assert np.linalg.norm(mt[4 * cell:4 * cell + 4] - sys.Mt_block(cell) @ seg) < 1e-13
    assert r @ ms <= r @ mt + 1e-12


@pytest.mark.parametrize("two_d", [False, True])
def test_single_direction_forward_block(two_d):  # :178-193
    sys = make_instance(two_d)
    nd, n = sys.n_dof(), sys.kinetic_dim()
    u = np.random.default_rng(6).uniform(-1, 1, nd)
    out = sys.apply_streaming_collision(0, u)
    full = np.zeros(n)
    full[:nd] = u
    prod = sys.apply_kinetic(full)
    ms = sys.apply_Ms(sys.density_of(full))
    assert np.max(np.abs(out - (prod[:nd] + ms))) < 1e-12


def test_psi0_must_be_one():  # transport_system.cpp:98-101
    p = prob1d()
    p.terms[0].psi = lambda mu: 2.0
    mesh = ro.Mesh.slab_uniform(0, 1, 4)
    with pytest.raises(ValueError):
        ro.TransportSystem(p, mesh, ro.build_dg_space(mesh), ro.gauss_legendre(2), [])
