"""Host-side mirror of the reference's solver API for the B200 path.

Names and argument meaning follow the reference core library (namespace rte,
/root/reference/proj/core/include/rte): quadratures, meshes, DG space,
ProblemDefinition/CoefficientTerm, TransportSystem (here batched over
parameter samples: ``TransportBatch``), DsaOperator, ReducedModel, romig,
romsad_tolerance and sisa_solve.  Every numerical operation on the hot path
runs in librte_b200.so (hand-written sm_100a kernels) through the C-ABI of
include/rte_b200.h; this module only marshals arguments.

Device vectors are torch float64 CUDA tensors of shape [S, n_dof]
(per-sample reference layout) -- torch is used for device memory and
streams only.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import capi

SLAB1D = capi.RTE_SLAB1D
XY2D = capi.RTE_XY2D
NQ = 6  # per-axis Gauss points of the cell rules (transport_system.cpp:18)


def _torch():
    import torch
    return torch


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# Quadrature (quadrature.cpp:8-73), mesh (mesh.cpp), DG space (dg_space.cpp)

@dataclass
class AngularQuadrature:
    geometry: int
    directions: np.ndarray
    weights: np.ndarray

    def n(self) -> int:
        return len(self.weights)


def gauss_legendre_nodes(n: int):
    if n < 1:
        raise ValueError("gauss_legendre: n must be >= 1")
    x, w = np.zeros(n), np.zeros(n)
    capi.check(capi.load().rte_gauss_legendre_nodes(n, capi.dptr(x), capi.dptr(w)))
    return x, w


def gauss_legendre(n: int) -> AngularQuadrature:
    x, w = gauss_legendre_nodes(n)
    d = np.zeros((n, 3))
    d[:, 0] = x
    return AngularQuadrature(SLAB1D, d, 0.5 * w)


def chebyshev_legendre(n_phi: int, n_vz: int) -> AngularQuadrature:
    if n_phi < 2 or n_vz < 1:
        raise ValueError("chebyshev_legendre: invalid sizes")
    z, wz = gauss_legendre_nodes(n_vz)
    pi = 3.14159265358979323846
    dirs, ws = [], []
    for j2 in range(n_vz):
        s = np.sqrt(max(0.0, 1.0 - z[j2] * z[j2]))
        for j1 in range(1, n_phi + 1):
            phi = 2.0 * j1 * pi / n_phi - pi / n_phi
            dirs.append((np.cos(phi) * s, np.sin(phi) * s, z[j2]))
            ws.append((1.0 / n_phi) * (0.5 * wz[j2]))
    return AngularQuadrature(XY2D, np.array(dirs), np.array(ws))


@dataclass
class Mesh:
    geometry: int = SLAB1D
    boundaries: Optional[np.ndarray] = None
    x0: float = 0.0
    x1: float = 1.0
    y0: float = 0.0
    y1: float = 1.0
    nx: int = 0
    ny: int = 1

    def cell_count(self) -> int:
        return self.nx if self.geometry == SLAB1D else self.nx * self.ny

    def n_local(self) -> int:
        return 2 if self.geometry == SLAB1D else 4

    def n_dof(self) -> int:
        return self.cell_count() * self.n_local()

    @staticmethod
    def slab(bounds) -> "Mesh":
        b = _c(bounds)
        if b.size < 2 or not np.all(b[:-1] < b[1:]):
            raise ValueError("slab mesh boundaries must be strictly increasing")
        return Mesh(SLAB1D, b, nx=b.size - 1, ny=1)

    @staticmethod
    def slab_uniform(a, b, n) -> "Mesh":
        if n < 1 or not (a < b):
            raise ValueError("invalid slab mesh")
        bounds = np.array([a + (b - a) * i / n for i in range(n + 1)])
        bounds[n] = b
        return Mesh.slab(bounds)

    @staticmethod
    def rect_uniform(x0, x1, nx, y0, y1, ny) -> "Mesh":
        if nx < 1 or ny < 1 or not (x0 < x1) or not (y0 < y1):
            raise ValueError("invalid rectangular mesh")
        return Mesh(XY2D, None, float(x0), float(x1), float(y0), float(y1), nx, ny)

    def _geo(self):
        b = self.boundaries if self.boundaries is not None else np.zeros(2)
        self._bk = _c(b)
        return (self.geometry, self.nx, max(self.ny, 1), capi.dptr(self._bk), self.x0, self.x1, self.y0, self.y1)

    def cell_points(self, nq: int = NQ):
        npc = nq if self.geometry == SLAB1D else nq * nq
        px, py = np.zeros(self.cell_count() * npc), np.zeros(self.cell_count() * npc)
        capi.check(capi.load().rte_cell_points(*self._geo(), nq, capi.dptr(px), capi.dptr(py)))
        return px, py

    def _check_points(self, vals, nq):
        npc = nq if self.geometry == SLAB1D else nq * nq
        if vals.size != self.cell_count() * npc:
            raise ValueError("expected %d quadrature-point values (cell_points(%d)), got %d"
                             % (self.cell_count() * npc, nq, vals.size))

    def weighted_mass(self, wvals, nq: int = NQ):
        """weighted_mass (transport_system.cpp:17-55) from values at the cell
        points, or from one constant (a scalar: same arithmetic, no array)."""
        nl = self.n_local()
        out = np.empty(self.cell_count() * nl * nl)
        if np.ndim(wvals) == 0:
            capi.check(capi.load().rte_weighted_mass_const(*self._geo(), nq, float(wvals), capi.dptr(out)))
        else:
            w = _c(wvals)
            self._check_points(w, nq)
            capi.check(capi.load().rte_weighted_mass(*self._geo(), nq, capi.dptr(w), capi.dptr(out)))
        return out.reshape(self.cell_count(), nl, nl)

    def project(self, fvals, nq: int = NQ):
        """project (dg_space.cpp:31-71) from values at the cell points or a constant."""
        out = np.empty(self.n_dof())
        if np.ndim(fvals) == 0:
            capi.check(capi.load().rte_project_const(*self._geo(), nq, float(fvals), capi.dptr(out)))
        else:
            f = _c(fvals)
            self._check_points(f, nq)
            capi.check(capi.load().rte_project(*self._geo(), nq, capi.dptr(f), capi.dptr(out)))
        return out


@dataclass
class CoefficientTerm:
    """problem.hpp:24-29."""
    psi: Optional[Callable] = None
    absorption_weight: Optional[Callable] = None
    scattering_weight: Optional[Callable] = None
    name: str = ""


@dataclass
class ProblemDefinition:
    """problem.hpp:31-44 (coefficient closures are vectorised f(x, y))."""
    geometry: int = SLAB1D
    terms: list = field(default_factory=list)
    source: Optional[Callable] = None
    inflow_left: float = 0.0
    inflow_right: float = 0.0
    inflow_bottom: float = 0.0
    inflow_top: float = 0.0
    n_params: int = 0
    param_ranges: list = field(default_factory=list)


def _vals(fn, px, py):
    """Closure values at the cell points; a closure returning one scalar for
    the whole array (a constant coefficient) stays a scalar."""
    if fn is None:
        return 0.0
    v = np.asarray(fn(px, py), dtype=np.float64)
    if v.ndim == 0:
        return float(v)
    return np.ascontiguousarray(np.broadcast_to(v, px.shape))


# ---------------------------------------------------------------------------

class TransportBatch:
    """TransportSystem (transport_system.hpp:30-142) for S parameter samples.

    Construct either from a ProblemDefinition + parameter list (the
    reference's constructor; mass blocks via the 6x6 Gauss rule of
    transport_system.cpp:17-55) or with ``from_cells`` from per-cell constant
    coefficients (the B200-native bulk input).
    """

    def __init__(self, problem: ProblemDefinition, mesh: Mesh, quad: AngularQuadrature,
                 mus: Sequence[Sequence[float]], device: int = 0, force_full_blocks: bool = False):
        """transport_system.cpp:82-109 for a batch of parameter samples.  XY
        problems whose mass blocks are sigma I per cell use the closed-form
        cell solves; intra-cell-varying coefficients (or force_full_blocks)
        use full 4x4 per-cell blocks."""
        if not (problem.geometry == mesh.geometry == quad.geometry):
            raise ValueError("transport system: geometry mismatch")
        if not problem.terms:
            raise ValueError("transport system: no coefficient terms")
        mus = [list(m) for m in mus]
        S = len(mus)
        psi = np.array([[t.psi(m) if t.psi is not None else 1.0 for t in problem.terms] for m in mus])
        if np.any(psi[:, 0] != 1.0):
            raise ValueError("transport system: term 0 must be parameter independent (psi == 1)")
        px, py = mesh.cell_points()
        K = len(problem.terms)
        tmt, tms = [], []
        for t in problem.terms:
            a = _vals(t.absorption_weight, px, py)
            sc = _vals(t.scattering_weight, px, py)
            tot = 0.0  # transport_system.cpp:125-130 (scalars stay scalars)
            if t.absorption_weight is not None:
                tot = tot + a
            if t.scattering_weight is not None:
                tot = tot + sc
            tmt.append(mesh.weighted_mass(tot))
            tms.append(mesh.weighted_mass(sc))
        tmt, tms = np.stack(tmt), np.stack(tms)  # [K][cells][nl][nl]

        def combine(terms):  # build_masses accumulation order (transport_system.cpp:136-137)
            t = np.ascontiguousarray(terms)
            out = np.empty((S,) + t.shape[1:])
            ps = np.ascontiguousarray(psi)
            capi.check(capi.load().rte_combine_terms(S, K, t[0].size, capi.dptr(ps), capi.dptr(t), capi.dptr(out)))
            return out
        g = mesh.project(_vals(problem.source, px, py)) if problem.source is not None else np.zeros(mesh.n_dof())
        inflow = (problem.inflow_left, problem.inflow_right, problem.inflow_bottom, problem.inflow_top)
        if mesh.geometry == XY2D:
            tmt_s = None
            if not force_full_blocks:
                try:
                    # every term sigma I per cell -> so is every combination: the
                    # samples' scalars are combined from the K term scalars (the
                    # same arithmetic, in the same order, as combining the blocks)
                    tmt_s, tms_s = _scalar_blocks(tmt), _scalar_blocks(tms)
                except capi.RteError:
                    tmt_s = None
            if tmt_s is not None:
                self._create(mesh, quad, combine(tmt_s), combine(tms_s), g, True, inflow, 1, device)
                self._affine(K, tmt_s, tms_s, psi)
            else:
                mt, ms = combine(tmt), combine(tms)
                # intra-cell-varying coefficients: full 4x4 blocks per cell (block = 16)
                self._create(mesh, quad, mt.reshape(S, -1, 16), ms.reshape(S, -1, 16), g, True, inflow, 16, device)
                self._affine(K, tmt.reshape(K, -1, 16), tms.reshape(K, -1, 16), psi)
        else:
            mt, ms = combine(tmt), combine(tms)
            self._create(mesh, quad, mt.reshape(S, -1, 4), ms.reshape(S, -1, 4), g, True, inflow, 4, device)
            self._affine(K, tmt.reshape(K, -1, 4), tms.reshape(K, -1, 4), psi)
        self.problem, self.mus = problem, mus

    @classmethod
    def from_cells(cls, mesh: Mesh, quad: AngularQuadrature, sigma_t, sigma_s, source, inflow=(0, 0, 0, 0),
                   device: int = 0, psi=None, term_sigma_t=None, term_sigma_s=None) -> "TransportBatch":
        """Per-cell constant coefficients: sigma_t/sigma_s [S][cells]; source is
        a DOF load vector [n_dof] (shared) or [S][n_dof]."""
        self = cls.__new__(cls)
        st, ss = _c(sigma_t), _c(sigma_s)
        if st.ndim == 1:
            st, ss = st[None], ss[None]
        g = _c(source)
        shared = g.ndim == 1
        self._create(mesh, quad, st, ss, g, shared, inflow, 1, device)
        if psi is not None:
            self._affine(np.asarray(psi).shape[1], _c(term_sigma_t), _c(term_sigma_s), _c(psi))
        self.problem, self.mus = None, None
        return self

    def _create(self, mesh, quad, mt, ms, g, shared, inflow, block, device):
        L = capi.load()
        self.mesh, self.quad, self.device = mesh, quad, device
        S = mt.shape[0]
        self._keep = [_c(mt), _c(ms), _c(g), _c(quad.directions), _c(quad.weights)]
        p = capi.Problem()
        geo = mesh._geo()
        p.geometry, p.nx, p.ny, p.bounds = geo[0], geo[1], geo[2], geo[3]
        p.x0, p.x1, p.y0, p.y1 = mesh.x0, mesh.x1, mesh.y0, mesh.y1
        p.n_dirs = quad.n()
        p.dirs = capi.dptr(self._keep[3])
        p.weights = capi.dptr(self._keep[4])
        p.inflow = (ctypes.c_double * 4)(*[float(v) for v in inflow])
        p.n_samples = S
        p.block = block
        p.mt, p.ms, p.source = capi.dptr(self._keep[0]), capi.dptr(self._keep[1]), capi.dptr(self._keep[2])
        p.source_shared = 1 if shared else 0
        h = ctypes.c_void_p()
        capi.check(L.rte_create(ctypes.byref(p), device, ctypes.byref(h)))
        self._h = h
        self.S = S
        self.nd = L.rte_n_dof(h)
        self.sigma_t_cells = mt if block == 1 else None
        self.k_terms = 0

    def _affine(self, K, tmt, tms, psi):
        self._akeep = [_c(tmt), _c(tms), _c(psi)]
        a = capi.Affine(K, capi.dptr(self._akeep[0]), capi.dptr(self._akeep[1]), capi.dptr(self._akeep[2]))
        capi.check(capi.load().rte_set_affine(self._h, ctypes.byref(a)), self._h)
        self.k_terms = K
        self.psi = self._akeep[2]

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(capi, "_lib", None) if capi is not None else None
        if h is not None and lib is not None:
            lib.rte_destroy(h)
            self._h = None

    # -- helpers --
    def n_dof(self) -> int:
        return self.nd

    def n_samples(self) -> int:
        return self.S

    def kinetic_dim(self) -> int:
        return self.quad.n() * self.nd

    def n_slots(self) -> int:
        return capi.load().rte_n_slots(self._h)

    def sweep_plan(self):
        """(directions per lane, direction groups per quadrant) of the XY
        sweep kernel for this batch ((0, 0) for slabs)."""
        d, g = ctypes.c_int(), ctypes.c_int()
        capi.check(capi.load().rte_sweep_plan(self._h, ctypes.byref(d), ctypes.byref(g)), self._h)
        return d.value, g.value

    def _dev(self, x, shape=None):
        torch = _torch()
        t = torch.as_tensor(x, dtype=torch.float64, device="cuda:%d" % self.device).contiguous()
        if shape is not None:
            t = t.reshape(shape)
        return t

    def _out(self, *shape):
        torch = _torch()
        return torch.empty(*shape, dtype=torch.float64, device="cuda:%d" % self.device)

    def _stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def _call(self, fn, *args):
        capi.check(fn(self._h, *args), self._h)

    # -- transport operator (batched over samples) --
    def apply_L(self, rho):
        rho = self._dev(rho, (self.S, self.nd))
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_apply_L, rho.data_ptr(), out.data_ptr(), self._stream())
        return out

    def assemble_rhs(self):
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_assemble_rhs, out.data_ptr(), self._stream())
        return out

    def fixed_point(self, rho):
        rho = self._dev(rho, (self.S, self.nd))
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_fixed_point, rho.data_ptr(), out.data_ptr(), self._stream())
        return out

    def sweep_direction(self, j, rhs):
        rhs = self._dev(rhs, (self.S, self.nd))
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_sweep_direction, int(j), rhs.data_ptr(), out.data_ptr(), self._stream())
        return out

    def kinetic_sweep(self, rho):
        rho = self._dev(rho, (self.S, self.nd))
        out = self._out(self.S, self.quad.n() * self.nd)
        self._call(capi.load().rte_kinetic_sweep, rho.data_ptr(), out.data_ptr(), self._stream())
        return out

    def density_of(self, f):
        f = self._dev(f, (self.S, self.quad.n() * self.nd))
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_density_of, f.data_ptr(), out.data_ptr(), self._stream())
        return out

    def apply_kinetic(self, u):
        """A_mu u = sum_k psi_k(mu) A_k u per sample (transport_system.cpp:598-613)."""
        u = self._dev(u, (self.S, self.kinetic_dim()))
        out = self._out(self.S, self.kinetic_dim())
        self._call(capi.load().rte_apply_kinetic, u.data_ptr(), out.data_ptr(), self._stream())
        return out

    def apply_streaming_collision(self, j, f):
        """(D_j + Sigma_t) f per sample, zero inflow (transport_system.cpp:482-558)."""
        f = self._dev(f, (self.S, self.nd))
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_apply_streaming_collision, int(j), f.data_ptr(), out.data_ptr(), self._stream())
        return out

    def kinetic_rhs(self):
        """Stacked kinetic right-hand side, block j = G + g_j^bc (transport_system.cpp:615-624)."""
        out = self._out(self.S, self.kinetic_dim())
        self._call(capi.load().rte_kinetic_rhs, out.data_ptr(), self._stream())
        return out

    def apply_term_kinetic(self, k, u):
        """A_k u (transport_system.cpp:560-596) for kinetic columns u [n, kdim]
        (term operators are parameter independent)."""
        u = self._dev(u)
        if u.dim() == 1:
            u = u.reshape(1, -1)
        out = self._out(u.shape[0], self.kinetic_dim())
        self._call(capi.load().rte_apply_term_kinetic, int(k), int(u.shape[0]), u.data_ptr(), out.data_ptr(),
                   self._stream())
        return out

    def apply_Ms(self, x):
        x = self._dev(x, (self.S, self.nd))
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_apply_Ms, x.data_ptr(), out.data_ptr(), self._stream())
        return out

    def apply_Mt(self, x):
        x = self._dev(x, (self.S, self.nd))
        out = self._out(self.S, self.nd)
        self._call(capi.load().rte_apply_Mt, x.data_ptr(), out.data_ptr(), self._stream())
        return out


def _scalar_blocks(m):
    """Per-cell mass blocks -> scalar sigma (the B200 2D path needs sigma*I);
    rte_scalar_blocks (OpenMP) raises RTE_ERR_UNSUPPORTED otherwise."""
    nl = m.shape[-1]
    f = np.ascontiguousarray(m).reshape(-1, nl * nl)
    out = np.empty(f.shape[0])
    rc = capi.load().rte_scalar_blocks(f.shape[0], nl, capi.dptr(f), capi.dptr(out))
    if rc == capi.RTE_ERR_UNSUPPORTED:
        raise capi.RteError(capi.RTE_ERR_UNSUPPORTED,
                            "xy geometry: coefficients must be constant per cell in this build")
    capi.check(rc)
    return out.reshape(m.shape[:-2])


class DsaOperator:
    """DsaOperator (dsa.hpp:29-56), one factorization per sample."""

    def __init__(self, batch: TransportBatch):
        self.batch = batch
        batch._call(capi.load().rte_dsa_setup, batch._stream())

    def coupled_dim(self) -> int:
        return capi.load().rte_dsa_coupled_dim(self.batch._h)

    def set_tolerance(self, tol: float, max_iters: int = 0) -> None:
        """XY only: relative residual of the iterative coupled solve."""
        self.batch._call(capi.load().rte_dsa_set_tolerance, float(tol), int(max_iters))

    def reset_history(self) -> None:
        """Clear the XY warm-start history (rte_dsa_reset_history): the next
        direct solve starts from zero.  rte_si_solve / rte_gmres_solve clear
        it themselves."""
        self.batch._call(capi.load().rte_dsa_reset_history, None)

    def last_iterations(self) -> int:
        return capi.load().rte_dsa_last_iterations(self.batch._h)

    def iteration_log(self, cap: int = 4096):
        """Krylov iteration counts (max over the samples) of the XY DSA solves
        of the last sisa_solve / gmres_solve, one per correction."""
        import ctypes
        buf = (ctypes.c_int * cap)()
        n = capi.load().rte_dsa_iteration_log(self.batch._h, buf, cap)
        if n < 0:
            raise capi.RteError("rte_dsa_iteration_log failed")
        return [int(buf[i]) for i in range(min(n, cap))]

    def solve_density(self, rhs):
        b = self.batch
        rhs = b._dev(rhs, (b.S, b.nd))
        out = b._out(b.S, b.nd)
        b._call(capi.load().rte_dsa_solve_density, rhs.data_ptr(), out.data_ptr(), b._stream())
        return out

    def correct(self, delta):
        b = self.batch
        d = b._dev(delta, (b.S, b.nd))
        out = b._out(b.S, b.nd)
        b._call(capi.load().rte_dsa_correct, d.data_ptr(), out.data_ptr(), b._stream())
        return out

    def apply_eliminated(self, x):
        """dsa.cpp:279-293: S x = A_rr x - A_rJ T^-1 A_Jr x per sample (the
        current block is factored lazily on first use)."""
        b = self.batch
        xd = b._dev(x, (b.S, b.nd))
        out = b._out(b.S, b.nd)
        b._call(capi.load().rte_dsa_apply_eliminated, xd.data_ptr(), out.data_ptr(), b._stream())
        return out


def build_dsa(batch: TransportBatch) -> DsaOperator:
    return DsaOperator(batch)


# ---------------------------------------------------------------------------
# Reduced models and the solver driver

@dataclass
class ReducedModel:
    """reduced_model.hpp:19-44 (host copy; column-major storage)."""
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

    _MAGIC = b"RTEROM1\0"

    def save(self, path: str) -> None:
        """RTEROM1 writer (reduced_model.cpp:41-64): header, then u_rho, u_iso,
        a_r[k] column-major, singular values, b_r -- all little-endian."""
        import struct
        try:
            f = open(path, "wb")
        except OSError as e:
            raise RuntimeError("reduced model: cannot create " + path) from e
        with f:
            f.write(self._MAGIC)
            f.write(struct.pack("<IIQQIIB", 1, int(self.geometry), int(self.n_v), int(self.n_dof), int(self.rank),
                                int(self.k_affine), ord(self.kind)))
            f.write(struct.pack("<5d", self.eps_pod, self.eps_train, self.discarded_fraction, self.basis_seconds,
                                self.operators_seconds))
            for a in [self.u_rho, self.u_iso] + list(self.a_r):
                f.write(np.asarray(a, dtype=np.float64).tobytes(order="F"))
            f.write(np.asarray(self.singular_values, dtype=np.float64).tobytes())
            f.write(np.asarray(self.b_r, dtype=np.float64).tobytes())

    @staticmethod
    def load(path: str) -> "ReducedModel":
        """RTEROM1 reader (reduced_model.cpp:66-104), same error messages."""
        import struct
        try:
            f = open(path, "rb")
        except OSError as e:
            raise RuntimeError("reduced model: cannot open " + path) from e
        with f:
            def raw(n):
                b = f.read(n)
                if len(b) != n:
                    raise RuntimeError("reduced model: truncated file")
                return b
            if raw(8) != ReducedModel._MAGIC:
                raise RuntimeError("reduced model: " + path + " has wrong magic")
            if struct.unpack("<I", raw(4))[0] != 1:
                raise RuntimeError("reduced model: unsupported version in " + path)
            geom, nv, nd, r, k, kind = struct.unpack("<IQQIIB", raw(29))
            eps_pod, eps_train, disc, bs, os_ = struct.unpack("<5d", raw(40))

            def mat(rows, cols):
                return np.frombuffer(raw(8 * rows * cols), dtype=np.float64).reshape((rows, cols), order="F").copy()
            m = ReducedModel(geom, nv, nd, r, k, chr(kind), eps_pod, eps_train)
            m.discarded_fraction, m.basis_seconds, m.operators_seconds = disc, bs, os_
            m.u_rho = mat(nd, r)
            m.u_iso = mat(nd, r)
            m.a_r = [mat(r, r) for _ in range(k)]
            m.singular_values = np.frombuffer(raw(8 * r), dtype=np.float64).copy()
            m.b_r = np.frombuffer(raw(8 * r), dtype=np.float64).copy()
        return m


def load_rom(batch: TransportBatch, which: int, model) -> None:
    """Upload a reduced model (which: 0 primary / 1 correction)."""
    keep = [_c(np.asarray(model.u_rho).T), _c(np.asarray(model.u_iso).T),
            _c(np.stack([np.asarray(a).T for a in model.a_r])), _c(model.b_r)]
    r = capi.Rom(int(model.rank), int(model.k_affine), capi.dptr(keep[0]), capi.dptr(keep[1]), capi.dptr(keep[2]),
                 capi.dptr(keep[3]), float(model.eps_pod), float(model.eps_train))
    capi.check(capi.load().rte_rom_load(batch._h, which, ctypes.byref(r)), batch._h)
    batch.__dict__.setdefault("_romkeep", {})[which] = keep


def romig(batch: TransportBatch):
    """strategies.cpp:8-28 for every sample; returns (rho0 [S,n_dof], status)."""
    out = batch._out(batch.S, batch.nd)
    status = (ctypes.c_int * batch.S)()
    batch._call(capi.load().rte_romig, out.data_ptr(), status, batch._stream())
    return out, np.array(status[:], dtype=np.int32)


def romsad_tolerance(eps_train, eps_pod, eta=0.1):
    """strategies.cpp:30-32."""
    return eta * max(eps_train, eps_pod)


@dataclass
class SolveConfig:
    """solvers.hpp:13-19 plus the batch extensions of rte_si_config."""
    eps_sisa: float = 1e-11
    max_iters: int = 2000
    norm: str = "abs"
    fixed_iters: int = 0
    theta: int = 3
    eps_romsad: float = 0.0
    initial_guess: Optional[object] = None
    compute_residual: bool = True
    check_every: int = 4
    gmres_restart: int = 25       # solvers.hpp:16
    gmres_rel_tol: float = 1e-11  # solvers.hpp:17
    dsa_inner: float = 0.0        # xy DSA: 0 = DSA tolerance; c > 0: relative c * eps / change per iteration
    dsa_floor: float = 0.0        # xy DSA: c > 0: relative min(0.1, c u ||rho*|| / ||delta||) per iteration (round-off floor)


@dataclass
class SolveReport:
    """solvers.hpp:21-33 (per sample)."""
    converged: bool
    n_sweep: int
    iterations: int
    change_history: list
    final_residual: float
    strategy: str
    initial_guess: str
    correction_log: str
    switch_iter: int
    singular: bool
    wall_seconds: float = 0.0  # wall time of the whole batched solve (shared by its samples)
    dsa_status: int = 0  # worst rte_dsa_status of the sample's DSA solves (0 = every solve met its tolerance)


_METHODS = {"SI": capi.RTE_SI, "DSA": capi.RTE_DSA, "ROMSA": capi.RTE_ROMSA, "ROMSAD": capi.RTE_ROMSAD,
            "ROMIG": capi.RTE_ROMIG}


class CorrectionStrategy:
    """The reference's plugin point (solvers.hpp:38-51), batched: ``setup`` is
    called once before the solve; ``correct(l, delta, active, out)`` once per
    SI iteration with ``delta`` = rho* - rho and ``out`` torch CUDA views
    [S, n_dof] and ``active`` a bool array of the samples to correct; it fills
    ``out`` for those samples and returns one kind letter per sample
    (``last_kind()``; '' = no correction).  ``label`` names the strategy in the
    reports."""

    def setup(self, batch: "TransportBatch") -> None:
        pass

    def correct(self, l: int, delta, active, out):
        raise NotImplementedError

    def label(self) -> str:
        return "CUSTOM"


class _DevArray:
    """Zero-copy torch view of a device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr, False), "version": 2}


def _custom_callback(batch, strategy, errors):
    torch = _torch()

    def cb(user, l, S, nd, active_p, delta_p, corr_p, kinds_p, stream):
        try:
            act = np.array([bool(active_p[s]) for s in range(S)])
            delta = torch.as_tensor(_DevArray(delta_p, (S, nd)), device=batch.device)
            out = torch.as_tensor(_DevArray(corr_p, (S, nd)), device=batch.device)
            kinds = strategy.correct(int(l), delta, act, out)
            torch.cuda.synchronize(batch.device)
            for s in range(S):
                k = kinds[s] if kinds is not None else ""
                kinds_p[s] = (k.encode()[:1] if k else b"\0")
            return 0
        except Exception as e:  # reported by rte_si_solve as RTE_ERR_RUNTIME
            errors.append(e)
            return 1
    return capi.CORRECTION_FN(cb)


def si_config(config: SolveConfig, method_code: int, callback=None) -> "capi.SiConfig":
    """SolveConfig -> rte_si_config (include/rte_b200.h); raises ValueError for
    settings the reference would reject (solvers.hpp:13-19)."""
    if config.norm not in ("abs", "rel"):
        raise ValueError("solve config: norm must be 'abs' or 'rel'")
    if config.max_iters < 1 or config.fixed_iters < 0 or config.check_every < 0:
        raise ValueError("solve config: max_iters >= 1, fixed_iters >= 0, check_every >= 0")
    if config.fixed_iters > config.max_iters:
        raise ValueError("solve config: fixed_iters must not exceed max_iters")
    if not 0.0 <= config.dsa_inner < 1.0:
        raise ValueError("solve config: dsa_inner must be in [0, 1)")
    if not config.dsa_floor >= 0.0:
        raise ValueError("solve config: dsa_floor must be >= 0")
    return capi.SiConfig(method_code, float(config.eps_sisa),
                         capi.RTE_NORM_REL if config.norm == "rel" else capi.RTE_NORM_ABS,
                         int(config.max_iters), int(config.fixed_iters), int(config.theta),
                         float(config.eps_romsad), 1 if config.initial_guess is not None else 0,
                         1 if config.compute_residual else 0, int(config.check_every),
                         callback if callback is not None else capi.CORRECTION_FN(), None, float(config.dsa_inner),
                         float(config.dsa_floor))


def sisa_solve(batch: TransportBatch, method, config: SolveConfig):
    """Batched sisa_solve (sisa.cpp:14-54): returns (rho [S, n_dof], reports).
    ``method`` is a built-in strategy name ("SI", "DSA", "ROMSA", "ROMSAD",
    "ROMIG") or a CorrectionStrategy object (RTE_CUSTOM)."""
    L = capi.load()
    custom = None if isinstance(method, str) else method
    m = capi.RTE_CUSTOM if custom is not None else _METHODS[method]
    errors = []
    cb = capi.CORRECTION_FN() if custom is None else _custom_callback(batch, custom, errors)
    if custom is not None:
        custom.setup(batch)
    cfg = si_config(config, m, cb)
    if config.initial_guess is not None:
        rho = batch._dev(config.initial_guess, (batch.S, batch.nd)).clone()
    else:
        rho = batch._out(batch.S, batch.nd)
    S, mi = batch.S, config.max_iters
    reps = (capi.SiReport * S)()
    hist = np.empty(S * mi)  # only the rows' first max(iterations) entries are written
    log = np.empty(S * mi, dtype=np.uint8)
    _torch().cuda.synchronize(batch.device)
    import time as _time
    t0 = _time.perf_counter()
    rc = L.rte_si_solve(batch._h, ctypes.byref(cfg), ctypes.c_void_p(rho.data_ptr()), reps, capi.dptr(hist),
                        log.ctypes.data_as(ctypes.c_char_p))
    wall = _time.perf_counter() - t0
    if rc != 0 and errors:
        raise errors[0]
    if rc != 0:
        # a failed DSA correction still fills the reports (attached to the error)
        try:
            capi.check(rc, batch._h)
        except capi.RteError as e:
            e.dsa_status = [int(reps[s].dsa_status) for s in range(S)]
            raise
    raw = log.tobytes()
    out = []
    label = custom.label() if custom is not None else method
    width = max((reps[s].iterations for s in range(S)), default=0)
    rows = hist.reshape(S, mi)[:, :width].tolist()  # one conversion for the batch
    for s in range(S):
        r = reps[s]
        it = r.iterations
        lg = raw[s * mi:s * mi + it].replace(b"\0", b"").decode()
        out.append(SolveReport(bool(r.converged), int(r.n_sweep), int(it), rows[s][:it],
                               float(r.final_residual), label,
                               "supplied" if (config.initial_guess is not None or m == capi.RTE_ROMIG) else "zero",
                               lg, int(r.switch_iter), bool(r.singular), wall, int(r.dsa_status)))
    return rho, out


def gmres_solve(batch: TransportBatch, preconditioner, config: SolveConfig, romig_guess: bool = False):
    """Batched gmres_solve (gmres.cpp:15-124): restarted GMRES on (I - L) rho =
    bbar, left-preconditioned with P = I + C Ms when ``preconditioner`` is a
    DsaOperator (PGMRES) or None (GMRES).  ``romig_guess`` = PGMRES-ROMIG
    (runner.cpp:202-205: the primary model's romig guess).  Returns
    (rho [S, n_dof], reports)."""
    L = capi.load()
    if romig_guess:
        guess = capi.RTE_GUESS_ROMIG
    elif config.initial_guess is not None:
        guess = capi.RTE_GUESS_SUPPLIED
    else:
        guess = capi.RTE_GUESS_ZERO
    cfg = capi.GmresConfig(1 if preconditioner is not None else 0, int(config.gmres_restart),
                           float(config.gmres_rel_tol), int(config.max_iters), guess)
    if guess == capi.RTE_GUESS_SUPPLIED:
        rho = batch._dev(config.initial_guess, (batch.S, batch.nd)).clone()
    else:
        rho = batch._out(batch.S, batch.nd)
    S = batch.S
    cap = 2 * int(config.max_iters) + 2
    reps = (capi.GmresReport * S)()
    hist = np.zeros(S * cap)
    _torch().cuda.synchronize(batch.device)
    import time as _time
    t0 = _time.perf_counter()
    capi.check(L.rte_gmres_solve(batch._h, ctypes.byref(cfg), ctypes.c_void_p(rho.data_ptr()), reps,
                                 capi.dptr(hist), cap), batch._h)
    wall = _time.perf_counter() - t0
    out = []
    for s in range(S):
        r = reps[s]
        n = min(int(r.history_len), cap)
        out.append(SolveReport(bool(r.converged), int(r.n_sweep), int(r.iterations), list(hist[s * cap:s * cap + n]),
                               float(r.final_residual), "PGMRES" if preconditioner is not None else "GMRES",
                               "zero" if guess == capi.RTE_GUESS_ZERO else "supplied", "", -1, False, wall,
                               int(r.dsa_status)))
    return rho, out


# ---------------------------------------------------------------------------
# Offline stage on the device: snapshots (snapshots.cpp:118-194), POD
# (pod.cpp), Galerkin projections (reduced_model.cpp:106-199).

@dataclass
class Snapshots:
    window: int
    f_iter: object        # torch [S, window, kdim]
    f_conv: object        # torch [S, kdim]
    drho: object          # torch [S, window, n_dof]
    converged: np.ndarray
    n_iter: np.ndarray

    @property
    def w_mu(self):
        return np.minimum(self.n_iter, self.window)


def collect_snapshots(batch: TransportBatch, window: int = 3, eps_train: float = 1e-11,
                      max_iters: int = 2000) -> Snapshots:
    kdim = batch.kinetic_dim()
    f_iter = batch._out(batch.S, window, kdim)
    f_iter.zero_()
    f_conv = batch._out(batch.S, kdim)
    drho = batch._out(batch.S, window, batch.nd)
    drho.zero_()
    conv = (ctypes.c_int * batch.S)()
    nit = (ctypes.c_int * batch.S)()
    _torch().cuda.synchronize(batch.device)
    batch._call(capi.load().rte_collect_snapshots, int(window), float(eps_train), int(max_iters),
                f_iter.data_ptr(), f_conv.data_ptr(), drho.data_ptr(), conv, nit)
    return Snapshots(window, f_iter, f_conv, drho, np.array(conv[:], dtype=np.int32),
                     np.array(nit[:], dtype=np.int32))


# RTESNP1 snapshot files (snapshots.cpp:15-78, 224-314): one file per
# training parameter, header | w_mu records (f^(l), delta_rho^(l)) | f_conv.
_SNAP_MAGIC = b"RTESNP1\0"


def snapshot_header_bytes(n_params: int) -> int:
    """snapshots.cpp:57 -- the first stored iterate starts here."""
    return 58 + 8 * n_params


def snapshot_patch_offset(n_params: int) -> int:
    """snapshots.cpp:58 -- w_mu, n_conv, converged (patched after the solve)."""
    return 49 + 8 * n_params


def write_snapshot_file(path: str, geometry: int, n_v: int, n_dof: int, mu, window: int, eps_train: float,
                        f_iter, drho, f_conv, n_conv: int, converged: bool, float32: bool = False) -> None:
    """One training parameter in the reference's RTESNP1 layout (the writer
    sequence of snapshots.cpp:128-176): f_iter [w_mu, n_v*n_dof] and drho
    [w_mu, n_dof] are the stored iterates (w_mu = min(n_conv, window))."""
    import struct
    mu = [float(v) for v in mu]
    f_iter = np.asarray(f_iter, dtype=np.float64)
    drho = np.asarray(drho, dtype=np.float64)
    w_mu = min(int(n_conv), int(window))
    kd = np.float32 if float32 else np.float64
    try:
        f = open(path, "wb")
    except OSError as e:
        raise RuntimeError("snapshots: cannot create " + path) from e
    with f:
        f.write(_SNAP_MAGIC)
        f.write(struct.pack("<IIQQI", 1, int(geometry), int(n_v), int(n_dof), len(mu)))
        f.write(struct.pack("<%dd" % len(mu), *mu))
        f.write(struct.pack("<IdBIIB", int(window), float(eps_train), 4 if float32 else 8, w_mu, int(n_conv),
                            1 if converged else 0))
        for l in range(w_mu):
            f.write(f_iter[l].astype(kd).tobytes())
            f.write(drho[l].tobytes())
        f.write(np.asarray(f_conv, dtype=np.float64).astype(kd).tobytes())


def read_snapshot_file(path: str) -> dict:
    """Header and data of one RTESNP1 file (snapshots.cpp:60-78, 270-314)."""
    import struct
    try:
        f = open(path, "rb")
    except OSError as e:
        raise RuntimeError("snapshots: cannot open " + path) from e
    with f:
        def raw(n):
            b = f.read(n)
            if len(b) != n:
                raise RuntimeError("snapshots: truncated file")
            return b
        if raw(8) != _SNAP_MAGIC:
            raise RuntimeError("snapshots: " + path + " is not a snapshot file")
        if struct.unpack("<I", raw(4))[0] != 1:
            raise RuntimeError("snapshots: unsupported version in " + path)
        geom, nv, nd, npar = struct.unpack("<IQQI", raw(24))
        mu = list(struct.unpack("<%dd" % npar, raw(8 * npar)))
        window, eps_train, dsize, w_mu, n_conv, conv = struct.unpack("<IdBIIB", raw(22))
        kd = np.float32 if dsize == 4 else np.float64
        kdim = nv * nd
        f_iter = np.zeros((w_mu, kdim))
        drho = np.zeros((w_mu, nd))
        for l in range(w_mu):
            f_iter[l] = np.frombuffer(raw(dsize * kdim), dtype=kd)
            drho[l] = np.frombuffer(raw(8 * nd), dtype=np.float64)
        f_conv = np.frombuffer(raw(dsize * kdim), dtype=kd).astype(np.float64)
    return dict(geometry=geom, n_v=nv, n_dof=nd, mu=mu, window=window, eps_train=eps_train, dsize=dsize,
                w_mu=w_mu, n_conv=n_conv, converged=bool(conv), f_iter=f_iter, drho=drho, f_conv=f_conv)


def save_snapshots(batch: TransportBatch, snaps: Snapshots, directory: str, eps_train: float,
                   float32: bool = False) -> list:
    """Write the device snapshots as the reference's per-parameter store
    (runner.cpp:44-48 names: snap_%03d.snap); returns the paths."""
    import os
    os.makedirs(directory, exist_ok=True)
    mus = batch.mus
    paths = []
    fi = snaps.f_iter.cpu().numpy()
    dr = snaps.drho.cpu().numpy()
    fc = snaps.f_conv.cpu().numpy()
    for s in range(batch.S):
        p = os.path.join(directory, "snap_%03d.snap" % s)
        w = int(snaps.w_mu[s])
        write_snapshot_file(p, int(batch.mesh.geometry), batch.quad.n(), batch.nd, mus[s] if mus else [],
                            snaps.window, eps_train, fi[s, :w], dr[s, :w], fc[s], int(snaps.n_iter[s]),
                            bool(snaps.converged[s]), float32)
        paths.append(p)
    return paths


def load_snapshots(directory: str, device: int = 0) -> Snapshots:
    """SnapshotStore::open (snapshots.cpp:224-254): every *.snap file of the
    directory in sorted order, one discretization; returns device Snapshots
    usable by snapshot_matrix / pod (e.g. a store written by the reference)."""
    import os
    torch = _torch()
    paths = sorted(os.path.join(directory, p) for p in os.listdir(directory) if p.endswith(".snap"))
    if not paths:
        raise RuntimeError("snapshots: no .snap files in " + directory)
    recs = [read_snapshot_file(p) for p in paths]
    g0 = recs[0]
    for p, r in zip(paths, recs):
        if (r["geometry"], r["n_v"], r["n_dof"]) != (g0["geometry"], g0["n_v"], g0["n_dof"]):
            raise RuntimeError("snapshots: mixed discretizations in one store (" + p + ")")
    window = max(r["window"] for r in recs)
    S, kdim, nd = len(recs), g0["n_v"] * g0["n_dof"], g0["n_dof"]
    f_iter = np.zeros((S, window, kdim))
    drho = np.zeros((S, window, nd))
    f_conv = np.zeros((S, kdim))
    for s, r in enumerate(recs):
        f_iter[s, :r["w_mu"]] = r["f_iter"]
        drho[s, :r["w_mu"]] = r["drho"]
        f_conv[s] = r["f_conv"]
    dev = "cuda:%d" % device
    return Snapshots(window, torch.from_numpy(f_iter).to(dev), torch.from_numpy(f_conv).to(dev),
                     torch.from_numpy(drho).to(dev), np.array([r["converged"] for r in recs], dtype=np.int32),
                     np.array([r["n_conv"] for r in recs], dtype=np.int32))


def snapshot_matrix(batch: TransportBatch, snaps: Snapshots, kind: str, window_limit: int = 0):
    """'primary' or 'correction' columns as a torch tensor [n_cols, kdim]
    (i.e. column-major kdim x n_cols)."""
    L = capi.load()
    k = 0 if kind == "primary" else 1
    conv = (ctypes.c_int * batch.S)(*snaps.converged.tolist())
    nit = (ctypes.c_int * batch.S)(*snaps.n_iter.tolist())
    n = ctypes.c_int()
    batch._call(L.rte_snapshot_columns, snaps.window, snaps.f_iter.data_ptr(), snaps.f_conv.data_ptr(), nit, conv,
                k, int(window_limit), None, ctypes.byref(n))
    out = batch._out(n.value, batch.kinetic_dim())
    batch._call(L.rte_snapshot_columns, snaps.window, snaps.f_iter.data_ptr(), snaps.f_conv.data_ptr(), nit, conv,
                k, int(window_limit), out.data_ptr(), ctypes.byref(n))
    return out


def truncation_rank(singular_values, eps_pod) -> int:
    s = np.ascontiguousarray(singular_values, dtype=np.float64)
    r = capi.load().rte_truncation_rank(capi.dptr(s), int(s.size), float(eps_pod))
    if r < 0:
        raise ValueError("pod: snapshot matrix is zero")
    return r


def pod(F, rank_max: int, device: int = 0):
    """POD of F [n_cols, m] (column-major m x n_cols) on the device: returns
    (U [rank_max, m] torch, all singular values numpy)."""
    torch = _torch()
    n, m = F.shape
    U = torch.empty((rank_max, m), dtype=torch.float64, device=F.device)
    sig = np.zeros(n)
    torch.cuda.synchronize(device)
    capi.check(capi.load().rte_pod(device, m, n, ctypes.c_void_p(F.data_ptr()), int(rank_max),
                                   ctypes.c_void_p(U.data_ptr()), capi.dptr(sig), None))
    return U, sig


def build_reduced_model(batch: TransportBatch, U, all_singular_values, eps_pod: float, eps_train: float,
                        kind: str) -> ReducedModel:
    """build_reduced_model (reduced_model.cpp:106-199) with the projections on
    the device; U: torch [r, kdim] (column-major basis)."""
    r = U.shape[0]
    nd, K = batch.nd, batch.k_terms
    u_rho = np.zeros(r * nd)
    u_iso = np.zeros(r * nd)
    a_r = np.zeros(K * r * r)
    b_r = np.zeros(r)
    _torch().cuda.synchronize(batch.device)
    batch._call(capi.load().rte_build_rom, int(r), ctypes.c_void_p(U.data_ptr()), capi.dptr(u_rho),
                capi.dptr(u_iso), capi.dptr(a_r), capi.dptr(b_r))
    sv = np.asarray(all_singular_values, dtype=np.float64)
    total = float(np.sum(sv))
    m = ReducedModel(int(batch.mesh.geometry), batch.quad.n(), nd, r, K, kind, eps_pod, eps_train)
    m.u_rho = u_rho.reshape(r, nd).T.copy()
    m.u_iso = u_iso.reshape(r, nd).T.copy()
    m.a_r = [a_r[k * r * r:(k + 1) * r * r].reshape(r, r).T.copy() for k in range(K)]
    m.b_r = b_r
    m.singular_values = sv[:r].copy()
    m.discarded_fraction = float(np.sum(sv[r:])) / total if total > 0 else 0.0
    return m
