"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference's hot path (arxiv 2402.10488, C++ reference under
/root/reference/proj) used as the checker by tests/, by ``__graft_entry__.smoke``
and by bench.py's ``cpu_baseline`` / ``--impl reference`` legs.  The product
(``paper_2402_10488_b200``) never imports this module.

Split of the restatement:
  * ``librte_oracle.so`` (rte_oracle.cpp): transport operator (sweeps, L, b̄,
    kinetic operators) and the consistent-DSA sparse assembly, in plain C++;
  * this module: the problem/mesh/quadrature front end, the DSA direct solve
    (SuperLU via scipy, standing in for Eigen::SparseLU), the source-iteration
    driver, the correction strategies, restarted GMRES, the reduced model and
    POD (numpy.linalg.svd is LAPACK dgesdd, the routine the reference calls).

Citations are file:line into /root/reference/proj/core/src unless noted.
Parity is pinned against the reference's own unit/acceptance tests, restated
in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "librte_oracle.so")
_lib = None

SLAB1D = 0
XY2D = 1

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_long)


def build(force: bool = False) -> str:
    """Compile the C++ restatement (gcc, no external libraries)."""
    src = os.path.join(_HERE, "rte_oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "librte_oracle.so"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.ro_last_error.restype = ctypes.c_char_p
        L.ro_system_create.restype = ctypes.c_void_p
        L.ro_dsa_create.restype = ctypes.c_void_p
        L.ro_n_dof.restype = ctypes.c_long
        L.ro_dsa_nnz.restype = ctypes.c_long
        L.ro_dsa_block_nnz.restype = ctypes.c_long
        for name in ("ro_system_destroy", "ro_n_dof", "ro_n_slots", "ro_mass_blocks",
                     "ro_term_mass_blocks", "ro_volumetric_source", "ro_boundary_source",
                     "ro_sweep_direction", "ro_apply_sc", "ro_apply_Ms", "ro_apply_Mt", "ro_apply_L",
                     "ro_assemble_rhs", "ro_kinetic_sweep", "ro_density_of", "ro_apply_term_kinetic",
                     "ro_apply_kinetic", "ro_kinetic_rhs", "ro_dsa_create", "ro_dsa_destroy",
                     "ro_dsa_nnz", "ro_dsa_fields", "ro_dsa_triplets", "ro_dsa_block_nnz", "ro_dsa_block"):
            getattr(L, name).argtypes = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# Quadrature (quadrature.cpp:8-73)

@dataclass
class AngularQuadrature:
    geometry: int
    directions: np.ndarray  # (n, 3)
    weights: np.ndarray     # (n,)

    def n(self) -> int:
        return len(self.weights)

    def vx(self, j):
        return self.directions[j, 0]

    def vy(self, j):
        return self.directions[j, 1]

    def vz(self, j):
        return self.directions[j, 2]


def gauss_legendre_nodes(n: int):
    """quadrature.cpp:8-39 (weights sum to 2)."""
    if n < 1:
        raise ValueError("gauss_legendre: n must be >= 1")
    x = np.zeros(n)
    w = np.zeros(n)
    lib().ro_gauss_legendre_nodes(ctypes.c_int(n), _p(x), _p(w))
    return x, w


def gauss_legendre(n: int) -> AngularQuadrature:
    """quadrature.cpp:41-52: slab rule, weights halved so they sum to 1."""
    x, w = gauss_legendre_nodes(n)
    d = np.zeros((n, 3))
    d[:, 0] = x
    return AngularQuadrature(SLAB1D, d, 0.5 * w)


def chebyshev_legendre(n_phi: int, n_vz: int) -> AngularQuadrature:
    """quadrature.cpp:54-73: CL(n_phi, n_vz), azimuth index fastest."""
    if n_phi < 2:
        raise ValueError("chebyshev_legendre: n_phi must be >= 2")
    if n_vz < 1:
        raise ValueError("chebyshev_legendre: n_vz must be >= 1")
    z, wz = gauss_legendre_nodes(n_vz)
    pi = 3.14159265358979323846
    dirs, ws = [], []
    for j2 in range(n_vz):
        vz = z[j2]
        s = np.sqrt(max(0.0, 1.0 - vz * vz))
        for j1 in range(1, n_phi + 1):
            phi = 2.0 * j1 * pi / n_phi - pi / n_phi
            dirs.append((np.cos(phi) * s, np.sin(phi) * s, vz))
            ws.append((1.0 / n_phi) * (0.5 * wz[j2]))
    return AngularQuadrature(XY2D, np.array(dirs), np.array(ws))


# ---------------------------------------------------------------------------
# Mesh / DG space (mesh.cpp, dg_space.cpp)

@dataclass
class Mesh:
    geometry: int = SLAB1D
    boundaries: Optional[np.ndarray] = None
    x0: float = 0.0
    x1: float = 1.0
    y0: float = 0.0
    y1: float = 1.0
    nx: int = 0
    ny: int = 0

    def cell_count(self) -> int:
        return self.nx if self.geometry == SLAB1D else self.nx * self.ny

    def width(self, i):
        return self.boundaries[i + 1] - self.boundaries[i]

    def left(self, i):
        return self.boundaries[i]

    def center(self, i):
        return 0.5 * (self.boundaries[i] + self.boundaries[i + 1])

    def hx(self):
        return (self.x1 - self.x0) / self.nx

    def hy(self):
        return (self.y1 - self.y0) / self.ny

    def cell_x0(self, ix):
        return self.x0 + ix * self.hx()

    def cell_y0(self, iy):
        return self.y0 + iy * self.hy()

    @staticmethod
    def slab(bounds) -> "Mesh":
        """mesh.cpp:7-19."""
        b = np.asarray(bounds, dtype=np.float64)
        if b.size < 2:
            raise ValueError("slab mesh needs at least one cell")
        if not np.all(b[:-1] < b[1:]):
            raise ValueError("slab mesh boundaries must be strictly increasing")
        return Mesh(SLAB1D, b.copy(), nx=b.size - 1, ny=1)

    @staticmethod
    def slab_uniform(a, b, n) -> "Mesh":
        """mesh.cpp:21-27."""
        if n < 1 or not (a < b):
            raise ValueError("invalid slab mesh")
        bounds = np.array([a + (b - a) * i / n for i in range(n + 1)])
        bounds[n] = b
        return Mesh.slab(bounds)

    @staticmethod
    def rect_uniform(x0, x1, nx, y0, y1, ny) -> "Mesh":
        """mesh.cpp:29-39."""
        if nx < 1 or ny < 1 or not (x0 < x1) or not (y0 < y1):
            raise ValueError("invalid rectangular mesh")
        return Mesh(XY2D, None, float(x0), float(x1), float(y0), float(y1), nx, ny)

    # ctypes argument tuple
    def _args(self):
        b = self.boundaries if self.boundaries is not None else np.zeros(1)
        self._b = _c(b)
        return (ctypes.c_int(self.geometry), ctypes.c_int(self.nx), ctypes.c_int(max(self.ny, 1)),
                _p(self._b), ctypes.c_double(self.x0), ctypes.c_double(self.x1),
                ctypes.c_double(self.y0), ctypes.c_double(self.y1))


@dataclass
class DgSpace:
    geometry: int
    degree: int
    n_local: int
    n_dof: int

    def dof(self, cell, local):
        return cell * self.n_local + local


def build_dg_space(mesh: Mesh, degree: int = 1) -> DgSpace:
    """dg_space.cpp:10-19."""
    if degree != 1:
        raise ValueError("build_dg_space: only linear (K=1) elements are supported")
    nl = 2 if mesh.geometry == SLAB1D else 4
    return DgSpace(mesh.geometry, 1, nl, mesh.cell_count() * nl)


def cell_points(mesh: Mesh, nq: int = 6):
    """Cell Gauss points in the order transport_system.cpp:23-53 visits them."""
    npc = nq if mesh.geometry == SLAB1D else nq * nq
    n = mesh.cell_count() * npc
    px = np.zeros(n)
    py = np.zeros(n)
    lib().ro_cell_points(*mesh._args(), ctypes.c_int(nq), _p(px), _p(py))
    return px, py


def _eval(fn, px, py):
    if fn is None:
        return None
    v = fn(px, py)
    v = np.broadcast_to(np.asarray(v, dtype=np.float64), px.shape)
    return np.ascontiguousarray(v)


def project(mesh: Mesh, space: DgSpace, f: Callable, nq: int = 6) -> np.ndarray:
    """dg_space.cpp:31-71 (f is vectorised: f(x_array, y_array))."""
    px, py = cell_points(mesh, nq)
    vals = _eval(f, px, py)
    out = np.zeros(space.n_dof)
    lib().ro_project(*mesh._args(), ctypes.c_int(nq), _p(vals), _p(out))
    return out


def cell_averages(mesh: Mesh, space: DgSpace, coeffs: np.ndarray) -> np.ndarray:
    """dg_space.cpp:91-105."""
    n = mesh.cell_count()
    if mesh.geometry == SLAB1D:
        meas = np.diff(mesh.boundaries)
    else:
        meas = np.full(n, mesh.hx() * mesh.hy())
    return coeffs[0::space.n_local][:n] / np.sqrt(meas)


def evaluate(mesh: Mesh, space: DgSpace, coeffs, cell, x, y=0.0) -> float:
    """dg_space.cpp:73-89."""
    if mesh.geometry == SLAB1D:
        h, xc = mesh.width(cell), mesh.center(cell)
        return coeffs[2 * cell] / np.sqrt(h) + coeffs[2 * cell + 1] * np.sqrt(12.0 / h ** 3) * (x - xc)
    hx, hy = mesh.hx(), mesh.hy()
    ix, iy = cell % mesh.nx, cell // mesh.nx
    rx = x - (mesh.cell_x0(ix) + 0.5 * hx)
    ry = y - (mesh.cell_y0(iy) + 0.5 * hy)
    bx = (1 / np.sqrt(hx), np.sqrt(12.0 / hx ** 3) * rx)
    by = (1 / np.sqrt(hy), np.sqrt(12.0 / hy ** 3) * ry)
    v = 0.0
    for b in range(2):
        for a in range(2):
            v += coeffs[4 * cell + a + 2 * b] * bx[a] * by[b]
    return v


# ---------------------------------------------------------------------------
# Problem definition (problem.hpp:24-44)

@dataclass
class CoefficientTerm:
    psi: Optional[Callable] = None
    absorption_weight: Optional[Callable] = None
    scattering_weight: Optional[Callable] = None
    name: str = ""


@dataclass
class ProblemDefinition:
    geometry: int = SLAB1D
    terms: list = field(default_factory=list)
    source: Optional[Callable] = None
    inflow_left: float = 0.0
    inflow_right: float = 0.0
    inflow_bottom: float = 0.0
    inflow_top: float = 0.0
    n_params: int = 0
    param_ranges: list = field(default_factory=list)


class SweepCounter:
    def __init__(self):
        self.sweeps = 0


class TransportSystem:
    """transport_system.hpp:30-142 over the C++ restatement."""

    def __init__(self, problem: ProblemDefinition, mesh: Mesh, space: DgSpace,
                 quad: AngularQuadrature, mu):
        if not (problem.geometry == mesh.geometry == space.geometry == quad.geometry):
            raise ValueError("transport system: geometry mismatch")
        if not problem.terms:
            raise ValueError("transport system: no coefficient terms")
        self.problem, self.mesh, self.space, self.quad = problem, mesh, space, quad
        self.mu = list(mu) if mu is not None else []
        psi = np.array([t.psi(self.mu) if t.psi is not None else 1.0 for t in problem.terms])
        self._psi = psi
        nq = 6
        px, py = cell_points(mesh, nq)
        nt = len(problem.terms)
        tot = np.zeros((nt, px.size))
        sct = np.zeros((nt, px.size))
        for k, t in enumerate(problem.terms):
            a = _eval(t.absorption_weight, px, py)
            s = _eval(t.scattering_weight, px, py)
            acc = np.zeros(px.size)
            if a is not None:
                acc = acc + a
            if s is not None:
                acc = acc + s
                sct[k] = s
            tot[k] = acc
        src = _eval(problem.source, px, py) if problem.source is not None else np.zeros(px.size)
        inflow = np.array([problem.inflow_left, problem.inflow_right, problem.inflow_bottom,
                           problem.inflow_top], dtype=np.float64)
        self._dirs = _c(quad.directions)
        self._w = _c(quad.weights)
        tot, sct, src = _c(tot), _c(sct), _c(src)
        psi_c = _c(psi)
        h = lib().ro_system_create(*mesh._args(), ctypes.c_int(quad.n()), _p(self._dirs), _p(self._w),
                                   ctypes.c_int(nt), _p(psi_c), _p(tot), _p(sct), _p(src), _p(inflow))
        if not h:
            raise ValueError(lib().ro_last_error().decode())
        self._h = ctypes.c_void_p(h)
        self._nd = space.n_dof

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.ro_system_destroy(h)

    # metadata
    def n_dof(self) -> int:
        return self._nd

    def kinetic_dim(self) -> int:
        return self.quad.n() * self._nd

    def n_terms(self) -> int:
        return len(self._psi)

    def psi(self, k) -> float:
        return float(self._psi[k])

    def n_slots(self) -> int:
        return lib().ro_n_slots(self._h)

    def is_cached(self) -> bool:
        """True when the per-slot inverse cache (build_sweep_cache) was built;
        large problems sweep with per-cell inverses computed on the fly."""
        return bool(lib().ro_is_cached(self._h))

    def dir_slot(self, j) -> int:
        return lib().ro_dir_slot(self._h, ctypes.c_int(j))

    def cache_slots(self, k0, k1):
        lib().ro_cache_slots(self._h, ctypes.c_int(k0), ctypes.c_int(k1))

    def time_sweeps(self, rho, dirs, nthreads):
        """Wall seconds of `nthreads` concurrent reference apply_L sweeps over
        `dirs` (cached inverses; see ro_time_sweeps)."""
        rho = _c(rho)
        d = np.ascontiguousarray(dirs, dtype=np.int32)
        L = lib()
        L.ro_time_sweeps.restype = ctypes.c_double
        return float(L.ro_time_sweeps(self._h, _p(rho), d.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                      ctypes.c_int(d.size), ctypes.c_int(nthreads)))

    def apply_L_dirs(self, rho, j0, j1):
        """apply_L restricted to directions [j0, j1) (CPU baseline timing)."""
        rho = _c(rho)
        out = np.zeros(self._nd)
        lib().ro_apply_L_dirs(self._h, _p(rho), _p(out), ctypes.c_int(j0), ctypes.c_int(j1))
        return out

    # --- density-space ops ---
    def apply_Ms(self, rho):
        rho = _c(rho)
        out = np.zeros(self._nd)
        lib().ro_apply_Ms(self._h, _p(rho), _p(out))
        return out

    def apply_Mt(self, rho):
        rho = _c(rho)
        out = np.zeros(self._nd)
        lib().ro_apply_Mt(self._h, _p(rho), _p(out))
        return out

    def sweep_direction(self, j, rhs):
        rhs = _c(rhs)
        f = np.zeros(self._nd)
        lib().ro_sweep_direction(self._h, ctypes.c_int(j), _p(rhs), _p(f))
        return f

    def apply_streaming_collision(self, j, f):
        f = _c(f)
        out = np.zeros(self._nd)
        lib().ro_apply_sc(self._h, ctypes.c_int(j), _p(f), _p(out))
        return out

    def apply_L(self, rho, counter: Optional[SweepCounter] = None):
        rho = _c(rho)
        out = np.zeros(self._nd)
        lib().ro_apply_L(self._h, _p(rho), _p(out))
        if counter is not None:
            counter.sweeps += 1
        return out

    def assemble_rhs(self, counter: Optional[SweepCounter] = None):
        out = np.zeros(self._nd)
        lib().ro_assemble_rhs(self._h, _p(out))
        if counter is not None:
            counter.sweeps += 1
        return out

    def boundary_source(self, j):
        out = np.zeros(self._nd)
        lib().ro_boundary_source(self._h, ctypes.c_int(j), _p(out))
        return out

    def volumetric_source(self):
        out = np.zeros(self._nd)
        lib().ro_volumetric_source(self._h, _p(out))
        return out

    def Ms_block(self, cell):
        return self._blocks()[1][cell]

    def Mt_block(self, cell):
        return self._blocks()[0][cell]

    def _blocks(self):
        if not hasattr(self, "_mblk"):
            nl = self.space.n_local
            nc = self.mesh.cell_count()
            mt = np.zeros(nc * nl * nl)
            ms = np.zeros(nc * nl * nl)
            lib().ro_mass_blocks(self._h, _p(mt), _p(ms))
            self._mblk = (mt.reshape(nc, nl, nl), ms.reshape(nc, nl, nl))
        return self._mblk

    def term_mass_blocks(self):
        nl = self.space.n_local
        nc = self.mesh.cell_count()
        nt = self.n_terms()
        tmt = np.zeros(nt * nc * nl * nl)
        tms = np.zeros(nt * nc * nl * nl)
        lib().ro_term_mass_blocks(self._h, _p(tmt), _p(tms))
        return tmt.reshape(nt, nc, nl, nl), tms.reshape(nt, nc, nl, nl)

    # --- kinetic-space ops ---
    def density_of(self, f):
        f = _c(f)
        rho = np.zeros(self._nd)
        lib().ro_density_of(self._h, _p(f), _p(rho))
        return rho

    def apply_term_kinetic(self, k, u):
        u = _c(u)
        out = np.zeros(self.kinetic_dim())
        lib().ro_apply_term_kinetic(self._h, ctypes.c_int(k), _p(u), _p(out))
        return out

    def apply_kinetic(self, u):
        u = _c(u)
        out = np.zeros(self.kinetic_dim())
        lib().ro_apply_kinetic(self._h, _p(u), _p(out))
        return out

    def kinetic_rhs(self):
        b = np.zeros(self.kinetic_dim())
        lib().ro_kinetic_rhs(self._h, _p(b))
        return b

    def kinetic_sweep(self, rho, counter: Optional[SweepCounter] = None):
        rho = _c(rho)
        f = np.zeros(self.kinetic_dim())
        lib().ro_kinetic_sweep(self._h, _p(rho), _p(f))
        if counter is not None:
            counter.sweeps += 1
        return f

    def materialize_kinetic(self):
        """transport_system.cpp:626-636."""
        n = self.kinetic_dim()
        a = np.zeros((n, n))
        e = np.zeros(n)
        for col in range(n):
            e[col] = 1.0
            a[:, col] = self.apply_kinetic(e)
            e[col] = 0.0
        return a


# ---------------------------------------------------------------------------
# DSA (dsa.cpp) -- assembly in C++, direct solve by SuperLU (the reference
# factors the same coupled matrix with Eigen::SparseLU, dsa.cpp:253).

def _splu(m):
    import scipy.sparse.linalg as sla
    return sla.splu(m.tocsc(), permc_spec="COLAMD")


def nested_dissection_cells(nx, ny):
    """Nested-dissection order of the cells of an nx x ny grid (recursive
    bisection along the longer side, separator line last)."""
    out = []

    def rec(x0, x1, y0, y1):
        w, h = x1 - x0, y1 - y0
        if w <= 0 or h <= 0:
            return
        if w * h <= 16:
            for y in range(y0, y1):
                out.extend(range(x0 + nx * y, x1 + nx * y))
            return
        if w >= h:
            m = (x0 + x1) // 2
            rec(x0, m, y0, y1)
            rec(m + 1, x1, y0, y1)
            out.extend(range(m + nx * y0, m + nx * y1, nx))
        else:
            m = (y0 + y1) // 2
            rec(x0, x1, y0, m)
            rec(x0, x1, m + 1, y1)
            out.extend(range(x0 + nx * m, x1 + nx * m))
    rec(0, nx, 0, ny)
    return np.array(out, dtype=np.int64)


class _NdLU:
    """SuperLU of the 2D coupled system in a nested-dissection order of the
    cells (the 12 unknowns of a cell kept together).  Eigen's SparseLU
    (dsa.cpp:146, 253) orders with COLAMD; COLAMD fill on these grids makes a
    128^2 factorization take ~45 s, the dissection order ~4x less.  The
    ordering changes only the rounding of the direct solve (backward error
    ~1e-14, tests/test_oracle_solvers.py)."""

    def __init__(self, m, nx, ny, nl, nf):
        import scipy.sparse.linalg as sla
        nd = nx * ny * nl
        cells = nested_dissection_cells(nx, ny)
        self.p = (np.arange(nf)[None, :, None] * nd + nl * cells[:, None, None]
                  + np.arange(nl)[None, None, :]).ravel()
        mc = m.tocsr()[self.p][:, self.p].tocsc()
        self.lu = sla.splu(mc, permc_spec="NATURAL", diag_pivot_thresh=0.1, options=dict(SymmetricMode=True))

    def solve(self, b):
        x = np.empty_like(b)
        x[self.p] = self.lu.solve(b[self.p])
        return x


class DsaOperator:
    """dsa.hpp:29-56."""

    def __init__(self, system: TransportSystem):
        import scipy.sparse as sp
        self.sys = system
        L = lib()
        h = L.ro_dsa_create(system._h)
        if not h:
            raise RuntimeError(L.ro_last_error().decode())
        self._h = ctypes.c_void_p(h)
        nnz = L.ro_dsa_nnz(self._h)
        r = np.zeros(nnz, dtype=np.int64)
        c = np.zeros(nnz, dtype=np.int64)
        v = np.zeros(nnz)
        L.ro_dsa_triplets(self._h, r.ctypes.data_as(_lp), c.ctypes.data_as(_lp), _p(v))
        self.n = system.n_dof()
        self.n_fields = L.ro_dsa_fields(self._h)
        dim = self.n_fields * self.n
        self.coupled = sp.coo_matrix((v, (r, c)), shape=(dim, dim)).tocsc()
        try:
            m = system.mesh
            if self.n_fields == 3:
                self.lu = _NdLU(self.coupled, m.nx, m.ny, 4, 3)
            else:
                self.lu = _splu(self.coupled)
        except RuntimeError as e:  # dsa.cpp:254-256
            raise RuntimeError("dsa: coupled moment system factorization failed") from e
        self._t_lu = [None] * (self.n_fields - 1)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.ro_dsa_destroy(h)

    def coupled_dim(self) -> int:
        return self.n_fields * self.n

    def _block(self, which, i=0):
        import scipy.sparse as sp
        L = lib()
        nnz = L.ro_dsa_block_nnz(self._h, ctypes.c_int(which), ctypes.c_int(i))
        r = np.zeros(nnz, dtype=np.int64)
        c = np.zeros(nnz, dtype=np.int64)
        v = np.zeros(nnz)
        L.ro_dsa_block(self._h, ctypes.c_int(which), ctypes.c_int(i), r.ctypes.data_as(_lp),
                       c.ctypes.data_as(_lp), _p(v))
        return sp.coo_matrix((v, (r, c)), shape=(self.n, self.n)).tocsr()

    def solve_density(self, rhs):
        """dsa.cpp:264-273."""
        full = np.zeros(self.coupled_dim())
        full[: self.n] = rhs
        sol = self.lu.solve(full)
        if not np.all(np.isfinite(sol)):
            raise RuntimeError("dsa: coupled moment system solve failed")
        return sol[: self.n]

    def correct(self, delta_rho):
        """dsa.cpp:275-277."""
        return self.solve_density(self.sys.apply_Ms(delta_rho))

    def apply_eliminated(self, x):
        """dsa.cpp:279-293."""
        out = self._block(0) @ x
        for i in range(self.n_fields - 1):
            if self._t_lu[i] is None:
                self._t_lu[i] = _splu(self._block(3, i))
            out = out - self._block(1, i) @ self._t_lu[i].solve(self._block(2, i) @ x)
        return out

    def triplets(self):
        c = self.coupled.tocoo()
        return c.row, c.col, c.data


def build_dsa(system: TransportSystem) -> DsaOperator:
    return DsaOperator(system)


# ---------------------------------------------------------------------------
# Solvers (solvers.hpp, sisa.cpp, gmres.cpp)

@dataclass
class SolveConfig:
    eps_sisa: float = 1e-11
    max_iters: int = 2000
    gmres_restart: int = 25
    gmres_rel_tol: float = 1e-11
    initial_guess: Optional[np.ndarray] = None
    # Extension (BASELINE.json says "relative change"): "abs" is the
    # reference's absolute test sisa.cpp:123, "rel" divides by ||rho*||_inf.
    norm: str = "abs"


@dataclass
class SolveReport:
    converged: bool = False
    n_sweep: int = 0
    iterations: int = 0
    change_history: list = field(default_factory=list)
    final_residual: float = 0.0
    wall_seconds: float = 0.0
    strategy: str = ""
    initial_guess: str = ""
    correction_log: str = ""


class CorrectionStrategy:
    """solvers.hpp:38-51."""

    def setup(self, system):
        pass

    def correct(self, l, delta):
        raise NotImplementedError

    def last_kind(self) -> str:
        raise NotImplementedError

    def label(self) -> str:
        raise NotImplementedError


class DsaStrategy(CorrectionStrategy):
    """solvers.hpp:54-65."""

    def __init__(self, op: DsaOperator):
        self.op = op

    def correct(self, l, delta):
        return self.op.correct(delta)

    def last_kind(self):
        return "D"

    def label(self):
        return "DSA"


def _inf(v) -> float:
    return float(np.max(np.abs(v))) if len(v) else 0.0


def sisa_solve(system: TransportSystem, strategy: Optional[CorrectionStrategy], config: SolveConfig):
    """sisa.cpp:14-54."""
    t0 = time.perf_counter()
    rep = SolveReport()
    rep.strategy = strategy.label() if strategy is not None else "SI"
    rep.initial_guess = "supplied" if config.initial_guess is not None else "zero"
    if strategy is not None:
        strategy.setup(system)
    sc = SweepCounter()
    bbar = system.assemble_rhs(sc)
    rho = np.array(config.initial_guess, dtype=np.float64) if config.initial_guess is not None \
        else np.zeros(system.n_dof())
    log = []
    for l in range(1, config.max_iters + 1):
        rho_star = system.apply_L(rho, sc) + bbar
        delta = rho_star - rho
        change = _inf(delta)
        if config.norm == "rel":
            den = _inf(rho_star)
            change = change / den if den > 0 else change
        rep.change_history.append(change)
        rep.iterations = l
        if change < config.eps_sisa:
            rho = rho_star
            rep.converged = True
            break
        if strategy is not None:
            rho = rho_star + strategy.correct(l, delta)
            log.append(strategy.last_kind())
        else:
            rho = rho_star
    rep.correction_log = "".join(log)
    rep.n_sweep = sc.sweeps
    rep.final_residual = _inf(rho - system.apply_L(rho, None) - bbar)
    rep.wall_seconds = time.perf_counter() - t0
    return rho, rep


def residual_inf(system: TransportSystem, rho) -> float:
    """sisa.cpp:56-59."""
    bbar = system.assemble_rhs(None)
    return _inf(rho - system.apply_L(rho, None) - bbar)


def gmres_solve(system: TransportSystem, preconditioner: Optional[DsaOperator], config: SolveConfig):
    """gmres.cpp:15-124 -- restarted left-preconditioned GMRES (MGS + Givens)."""
    t0 = time.perf_counter()
    n = system.n_dof()
    m = config.gmres_restart
    rep = SolveReport()
    rep.strategy = "PGMRES" if preconditioner is not None else "GMRES"
    rep.initial_guess = "supplied" if config.initial_guess is not None else "zero"
    sc = SweepCounter()
    bbar = system.assemble_rhs(sc)

    def apply_A(x):
        return x - system.apply_L(x, sc)

    def apply_P(x):
        if preconditioner is None:
            return x
        return x + preconditioner.solve_density(system.apply_Ms(x))

    pb = apply_P(bbar)
    bnorm = float(np.linalg.norm(pb))
    if bnorm == 0:
        bnorm = 1.0
    rho = np.array(config.initial_guess, dtype=np.float64) if config.initial_guess is not None else np.zeros(n)
    V = np.zeros((n, m + 1))
    H = np.zeros((m + 1, m))
    g = np.zeros(m + 1)
    cs = np.zeros(m)
    sn = np.zeros(m)
    total = 0
    while True:
        a_rho = apply_A(rho)
        r = apply_P(bbar - a_rho)
        beta = float(np.linalg.norm(r))
        rel0 = beta / bnorm
        rep.change_history.append(rel0)
        if rel0 <= config.gmres_rel_tol:
            rep.converged = True
            rep.final_residual = _inf(a_rho - bbar)
            break
        if total >= config.max_iters:
            break
        V[:, 0] = r / beta
        g[:] = 0
        g[0] = beta
        cols = 0
        for j in range(m):
            if total >= config.max_iters:
                break
            total += 1
            w = apply_P(apply_A(V[:, j]))
            for i in range(j + 1):
                H[i, j] = float(w @ V[:, i])
                w = w - H[i, j] * V[:, i]
            H[j + 1, j] = float(np.linalg.norm(w))
            breakdown = H[j + 1, j] <= 1e-300
            if not breakdown:
                V[:, j + 1] = w / H[j + 1, j]
            for i in range(j):
                tmp = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = tmp
            denom = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j] = 1.0 if denom == 0 else H[j, j] / denom
            sn[j] = 0.0 if denom == 0 else H[j + 1, j] / denom
            H[j, j] = denom
            H[j + 1, j] = 0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            cols = j + 1
            rel = abs(g[j + 1]) / bnorm
            rep.change_history.append(rel)
            if rel <= config.gmres_rel_tol or breakdown:
                break
        if cols > 0:
            y = np.zeros(cols)
            for i in range(cols - 1, -1, -1):
                s = g[i]
                for k in range(i + 1, cols):
                    s -= H[i, k] * y[k]
                y[i] = s / H[i, i]
            rho = rho + V[:, :cols] @ y
    rep.iterations = total
    rep.n_sweep = sc.sweeps
    if not rep.converged:
        rep.final_residual = _inf(rho - system.apply_L(rho, None) - bbar)
    rep.wall_seconds = time.perf_counter() - t0
    return rho, rep


# ---------------------------------------------------------------------------
# Full-pivot LU (restates the Eigen::FullPivLU semantics the strategies use:
# complete pivoting, rank threshold eps * n * |max pivot|).

class FullPivLU:
    def __init__(self, a):
        a = np.array(a, dtype=np.float64)
        n = a.shape[0]
        self.n = n
        lu = a.copy()
        rp = np.arange(n)
        cp = np.arange(n)
        self.nonzero_pivots = n
        self.maxpivot = 0.0
        for k in range(n):
            sub = np.abs(lu[k:, k:])
            # column-major first maximum, like Eigen's maxCoeff traversal
            idx = np.argmax(sub.T.reshape(-1))
            ci, ri = divmod(int(idx), n - k)
            big = sub[ri, ci]
            if big == 0.0:
                self.nonzero_pivots = k
                break
            self.maxpivot = max(self.maxpivot, big)
            ri += k
            ci += k
            if ri != k:
                lu[[k, ri], :] = lu[[ri, k], :]
                rp[[k, ri]] = rp[[ri, k]]
            if ci != k:
                lu[:, [k, ci]] = lu[:, [ci, k]]
                cp[[k, ci]] = cp[[ci, k]]
            if k < n - 1:
                lu[k + 1:, k] /= lu[k, k]
                lu[k + 1:, k + 1:] -= np.outer(lu[k + 1:, k], lu[k, k + 1:])
        self.lu, self.rp, self.cp = lu, rp, cp

    def rank(self) -> int:
        thr = np.finfo(np.float64).eps * self.n * abs(self.maxpivot)
        d = np.abs(np.diag(self.lu))[: self.nonzero_pivots]
        return int(np.sum(d > thr))

    def is_invertible(self) -> bool:
        return self.rank() == self.n

    def solve(self, b):
        b = np.asarray(b, dtype=np.float64)[self.rp]
        n = self.n
        y = b.copy()
        for i in range(n):
            y[i] -= self.lu[i, :i] @ y[:i]
        x = y.copy()
        for i in range(n - 1, -1, -1):
            x[i] = (y[i] - self.lu[i, i + 1:] @ x[i + 1:]) / self.lu[i, i]
        out = np.zeros(n)
        out[self.cp] = x
        return out


# ---------------------------------------------------------------------------
# Reduced model (reduced_model.hpp/.cpp) and strategies (strategies.cpp)

@dataclass
class ReducedModel:
    geometry: int = 0
    n_v: int = 0
    n_dof: int = 0
    rank: int = 0
    k_affine: int = 0
    kind: str = "p"
    eps_pod: float = 0.0
    eps_train: float = 0.0
    u_rho: np.ndarray = None
    u_iso: np.ndarray = None
    a_r: list = None
    singular_values: np.ndarray = None
    discarded_fraction: float = 0.0
    b_r: np.ndarray = None
    basis_seconds: float = 0.0
    operators_seconds: float = 0.0

    def assemble(self, system: TransportSystem):
        """reduced_model.cpp:32-39."""
        if system.n_terms() != self.k_affine:
            raise ValueError("reduced model: affine term count does not match the system")
        a = np.zeros((self.rank, self.rank))
        for k in range(self.k_affine):
            a = a + system.psi(k) * self.a_r[k]
        return a

    def assemble_psi(self, psi):
        a = np.zeros((self.rank, self.rank))
        for k in range(self.k_affine):
            a = a + psi[k] * self.a_r[k]
        return a

    # RTEROM1 binary format (reduced_model.cpp:41-104)
    def save(self, path):
        import struct
        with open(path, "wb") as f:
            f.write(b"RTEROM1\0")
            f.write(struct.pack("<IIQQIIB", 1, self.geometry, self.n_v, self.n_dof, self.rank,
                                self.k_affine, ord(self.kind)))
            f.write(struct.pack("<5d", self.eps_pod, self.eps_train, self.discarded_fraction,
                                self.basis_seconds, self.operators_seconds))
            f.write(np.asfortranarray(self.u_rho).tobytes(order="F"))
            f.write(np.asfortranarray(self.u_iso).tobytes(order="F"))
            for a in self.a_r:
                f.write(np.asfortranarray(a).tobytes(order="F"))
            f.write(np.asarray(self.singular_values, dtype=np.float64).tobytes())
            f.write(np.asarray(self.b_r, dtype=np.float64).tobytes())

    @staticmethod
    def load(path) -> "ReducedModel":
        import struct
        try:
            f = open(path, "rb")
        except OSError as e:
            raise RuntimeError("reduced model: cannot open " + path) from e
        with f:
            if f.read(8) != b"RTEROM1\0":
                raise RuntimeError("reduced model: " + path + " has wrong magic")
            ver, geom, nv, nd, r, k, kind = struct.unpack("<IIQQIIB", f.read(33))
            if ver != 1:
                raise RuntimeError("reduced model: unsupported version in " + path)
            eps_pod, eps_train, disc, bs, os_ = struct.unpack("<5d", f.read(40))

            def mat(rows, cols):
                return np.frombuffer(f.read(8 * rows * cols), dtype=np.float64).reshape((rows, cols), order="F").copy()
            m = ReducedModel(geom, nv, nd, r, k, chr(kind), eps_pod, eps_train)
            m.discarded_fraction, m.basis_seconds, m.operators_seconds = disc, bs, os_
            m.u_rho = mat(nd, r)
            m.u_iso = mat(nd, r)
            m.a_r = [mat(r, r) for _ in range(k)]
            m.singular_values = np.frombuffer(f.read(8 * r), dtype=np.float64).copy()
            m.b_r = np.frombuffer(f.read(8 * r), dtype=np.float64).copy()
        return m


def build_reduced_model(system: TransportSystem, basis: np.ndarray, all_singular_values,
                        eps_pod: float, eps_train: float, kind: str, basis_seconds: float = 0.0):
    """reduced_model.cpp:106-199 (single batch: the basis fits in memory)."""
    t0 = time.perf_counter()
    m = system.kinetic_dim()
    n = system.n_dof()
    nv = system.quad.n()
    U = np.asarray(basis, dtype=np.float64)
    if U.shape[0] != m:
        raise ValueError("reduced model: basis rows != kinetic dimension")
    r = U.shape[1]
    kk = system.n_terms()
    sv = np.asarray(all_singular_values, dtype=np.float64)
    model = ReducedModel(int(system.quad.geometry), nv, n, r, kk, kind, eps_pod, eps_train)
    model.basis_seconds = basis_seconds
    model.singular_values = sv[:r].copy()
    total = float(np.sum(sv))
    model.discarded_fraction = float(np.sum(sv[r:])) / total if total > 0 else 0.0
    w = system.quad.weights
    u_rho = np.zeros((n, r))
    u_iso = np.zeros((n, r))
    for j in range(nv):
        blk = U[j * n:(j + 1) * n, :]
        u_rho += w[j] * blk
        u_iso += blk
    model.u_rho, model.u_iso = u_rho, u_iso
    model.b_r = U.T @ system.kinetic_rhs()
    model.a_r = []
    for k in range(kk):
        Y = np.stack([system.apply_term_kinetic(k, U[:, c]) for c in range(r)], axis=1)
        model.a_r.append(U.T @ Y)
    gram = U.T @ U
    ortho = float(np.max(np.abs(gram - np.eye(r)))) if r else 0.0
    if ortho > 1e-10:
        raise RuntimeError("reduced model: basis columns are not orthonormal (defect %g)" % ortho)
    model.operators_seconds = time.perf_counter() - t0
    return model


def romig(model: ReducedModel, system: TransportSystem):
    """strategies.cpp:8-28."""
    a = model.assemble(system)
    lu = FullPivLU(a)
    if not lu.is_invertible():
        raise RuntimeError("reduced initial guess: reduced operator is singular at this parameter value")
    c = lu.solve(model.b_r)
    resid = _inf(model.b_r - a @ c)
    scale = float(np.max(np.sum(np.abs(a), axis=1))) * _inf(c) + _inf(model.b_r)
    if resid > 1e-10 * max(scale, 1e-300):
        raise RuntimeError("reduced initial guess: Galerkin residual check failed")
    return model.u_rho @ c


def romsad_tolerance(eps_train, eps_pod, eta=0.1):
    """strategies.cpp:30-32."""
    return eta * max(eps_train, eps_pod)


class RomsaStrategy(CorrectionStrategy):
    """strategies.cpp:34-53."""

    def __init__(self, model: ReducedModel, label: str = "ROMSA"):
        self.model = model
        self._label = label
        self.singular = False
        self._kind = "R"

    def setup(self, system):
        self.system = system
        self.lu = FullPivLU(self.model.assemble(system))
        self.singular = not self.lu.is_invertible()
        self._kind = "R"

    def correct(self, l, delta):
        if self.singular:
            self._kind = "S"
            return np.zeros(len(delta))
        self._kind = "R"
        rhs = self.model.u_iso.T @ self.system.apply_Ms(delta)
        return self.model.u_rho @ self.lu.solve(rhs)

    def last_kind(self):
        return self._kind

    def label(self):
        return self._label


class RomsadStrategy(CorrectionStrategy):
    """strategies.cpp:55-76 -- monotone ROMSA -> DSA switch."""

    def __init__(self, model: ReducedModel, dsa: DsaOperator, theta: int, eps_romsad: float,
                 label: str = "ROMSAD"):
        self.romsa = RomsaStrategy(model)
        self.dsa = DsaStrategy(dsa)
        self.theta = theta
        self.eps = eps_romsad
        self.switched = False
        self._kind = "R"
        self._label = label

    def setup(self, system):
        self.romsa.setup(system)
        self.switched = self.romsa.singular
        self._kind = "D" if self.switched else "R"

    def correct(self, l, delta):
        if not self.switched and l <= self.theta and _inf(delta) >= self.eps:
            self._kind = "R"
            return self.romsa.correct(l, delta)
        self.switched = True
        self._kind = "D"
        return self.dsa.correct(l, delta)

    def last_kind(self):
        return self._kind

    def label(self):
        return self._label


# ---------------------------------------------------------------------------
# POD (pod.cpp) and snapshot collection (snapshots.cpp)

def truncation_rank(singular_values, eps_pod) -> int:
    """pod.cpp:117-139."""
    s = np.asarray(singular_values, dtype=np.float64)
    if s.size == 0 or not (s[0] > 0):
        raise ValueError("pod: snapshot matrix is zero")
    guard = 1e-14 * s[0]
    kept = 0
    total = 0.0
    for k in range(s.size):
        if s[k] >= guard:
            total += s[k]
            kept = k + 1
        else:
            break
    partial = 0.0
    for l in range(kept):
        partial += s[l]
        if partial / total >= 1.0 - eps_pod:
            return l + 1
    return kept


@dataclass
class DensePod:
    rank: int
    u: np.ndarray
    singular_values: np.ndarray


def pod_truncate(a, eps_pod) -> DensePod:
    """pod.cpp:141-150 with dgesdd (numpy.linalg.svd calls LAPACK dgesdd)."""
    a = np.asarray(a, dtype=np.float64)
    if a.size == 0:
        raise ValueError("pod: empty snapshot matrix")
    u, s, _ = np.linalg.svd(a, full_matrices=False)
    r = truncation_rank(s, eps_pod)
    return DensePod(r, u[:, :r].copy(), s)


@dataclass
class Snapshots:
    mu: list
    window: int
    w_mu: int
    n_conv: int
    converged: bool
    eps_train: float
    iterates: list       # f^(l), l = 1..w_mu (kinetic vectors)
    delta_rho: list      # drho^(l)
    converged_f: np.ndarray


def collect_snapshots(system: TransportSystem, dsa: DsaOperator, window: int = 3,
                      eps_train: float = 1e-11, max_iters: int = 2000) -> Snapshots:
    """snapshots.cpp:118-194 (kept in memory instead of an RTESNP1 file)."""
    n = system.n_dof()
    rho_prev = np.zeros(n)
    its, drs = [], []
    l = 0
    converged = False
    f = None
    while l < max_iters:
        l += 1
        f = system.kinetic_sweep(rho_prev)
        rho_star = system.density_of(f)
        drho = rho_star - rho_prev
        if l <= window:
            its.append(f.copy())
            drs.append(drho.copy())
        if _inf(drho) < eps_train:
            converged = True
            break
        rho_prev = rho_star + dsa.correct(drho)
    return Snapshots(list(system.mu), window, len(its), l, converged, eps_train, its, drs, f.copy())


def primary_matrix(snaps):
    """PrimarySource (snapshots.cpp:316-332): converged solutions only."""
    return np.stack([s.converged_f for s in snaps if s.converged], axis=1)


def correction_matrix(snaps, window_limit=1 << 30):
    """CorrectionSource (snapshots.cpp:334-376): f_conv - f^(l), l <= window."""
    cols = []
    for s in snaps:
        if not s.converged:
            continue
        for l in range(1, min(s.w_mu, window_limit) + 1):
            cols.append(s.converged_f - s.iterates[l - 1])
    return np.stack(cols, axis=1)


def unit_draws(seed: int, n: int) -> np.ndarray:
    """cases.cpp:11-13: n unit draws (gen() >> 11) * 2^-53 of std::mt19937_64(seed)."""
    out = np.zeros(n)
    lib().ro_unit_draws(ctypes.c_ulonglong(seed), ctypes.c_long(n), _p(out))
    return out


class Mt19937_64:
    """std::mt19937_64 (for cases.cpp:11-13 unit draws: (gen() >> 11) * 2^-53)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.idx = 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF

    def unit(self) -> float:
        return float(self() >> 11) * 2.0 ** -53


def set_cache_budget(nbytes: float):
    """Largest per-slot inverse cache (bytes) later TransportSystems build;
    bigger problems compute each cell's inverse when they sweep (same
    arithmetic), slot-major over OpenMP threads."""
    lib().ro_set_cache_budget(ctypes.c_double(float(nbytes)))


def cell_constant_system(nx, ny, sigma_t, sigma_s, quad, source=1.0, inflow=(0.0, 0.0, 0.0, 0.0),
                         extent=(0.0, 1.0, 0.0, 1.0)):
    """TransportSystem of an XY problem with per-cell constant coefficients
    sigma_t, sigma_s [ny * nx] (cell = ix + nx iy): one coefficient term whose
    closures look up the cell of each quadrature point (transport_system.cpp:
    17-55 integrates them exactly to sigma * I blocks)."""
    x0, x1, y0, y1 = extent
    hx, hy = (x1 - x0) / nx, (y1 - y0) / ny
    st = np.asarray(sigma_t, dtype=np.float64)
    sa = st - np.asarray(sigma_s, dtype=np.float64)
    ss = np.asarray(sigma_s, dtype=np.float64)

    def cell(x, y):
        ix = np.clip(np.floor((np.asarray(x) - x0) / hx).astype(np.int64), 0, nx - 1)
        iy = np.clip(np.floor((np.asarray(y) - y0) / hy).astype(np.int64), 0, ny - 1)
        return ix + nx * iy
    term = CoefficientTerm(absorption_weight=lambda x, y: sa[cell(x, y)],
                           scattering_weight=lambda x, y: ss[cell(x, y)])
    p = ProblemDefinition(XY2D, [term], lambda x, y: source + 0.0 * np.asarray(x),
                          inflow_left=inflow[0], inflow_right=inflow[1], inflow_bottom=inflow[2],
                          inflow_top=inflow[3])
    m = Mesh.rect_uniform(x0, x1, nx, y0, y1, ny)
    return TransportSystem(p, m, build_dg_space(m), quad, [])
