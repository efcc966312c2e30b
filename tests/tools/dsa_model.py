"""Numpy model of the 2D DSA multigrid in the C5 regime (research tool, not a test).

Builds the coupled P1 DSA matrix of a thin random-coefficient problem with the
oracle (sigma_t h in [1e-4, 0.1] like configs[4]), the nested DG prolongation,
and a red-black 12x12 block Gauss-Seidel V-cycle mirroring dsa2d.cu, then
measures BiCGStab/GMRES preconditioner applications and analyses the slow
modes.  DESIGN.md section 6 quotes its results.

  python tests/tools/dsa_model.py NX LEVELS [plain|aux] [mode|gmres|lines N|smoothedP W|spectrum|semicoarse|patch N|bicgstabl|idrs]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spl
from oracle import rte_oracle as ro

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 32
rng = np.random.default_rng(1)
st = np.exp(np.log(0.1) + (np.log(100.0) - np.log(0.1)) * rng.uniform(size=(nx, nx))) * nx / 1024
c = rng.uniform(0.5, 0.99, size=(nx, nx))
if os.environ.get("HOMOG"):  # homogeneous field at a given sigma_t (same c draw mean)
    st = np.full((nx, nx), float(os.environ["HOMOG"]) * nx / 1024); c = np.full((nx, nx), 0.745)
ss = c * st
h = 1.0 / nx
def cell(x, y):
    ix = np.clip(np.floor(np.asarray(x) / h).astype(int), 0, nx - 1)
    iy = np.clip(np.floor(np.asarray(y) / h).astype(int), 0, nx - 1)
    return iy, ix
t0 = ro.CoefficientTerm(absorption_weight=lambda x, y: (st - ss)[cell(x, y)], scattering_weight=lambda x, y: ss[cell(x, y)])
p = ro.ProblemDefinition(ro.XY2D, [t0], lambda x, y: 1.0)
m = ro.Mesh.rect_uniform(0, 1, nx, 0, 1, nx)
o = ro.TransportSystem(p, m, ro.build_dg_space(m), ro.chebyshev_legendre(16, 8), [])
A = ro.build_dsa(o).coupled.tocsr()
n = o.n_dof(); nc = nx * nx
print("dim", A.shape, "nnz", A.nnz)

# unknown index: f*n + cell*4 + local ; cell = iy*nx + ix ; local = a + 2b
def idx(f, ix, iy, loc, nxl):
    return f * (nxl * nxl * 4) + (iy * nxl + ix) * 4 + loc

# nested prolongation coarse (nx/2) -> fine (nx)
a_, b_, c_ = 1 / np.sqrt(2), np.sqrt(6) / 4, 1 / (2 * np.sqrt(2))
def Emat(pos):
    return np.array([[a_, b_ if pos else -b_], [0.0, c_]])
def prolong(nxf):
    nxc = nxf // 2
    rows, cols, vals = [], [], []
    for f in range(3):
        for iy in range(nxf):
            for ix in range(nxf):
                Ex, Ey = Emat(ix & 1), Emat(iy & 1)
                for fa in range(2):
                    for fb in range(2):
                        for ca in range(2):
                            for cb in range(2):
                                v = Ey[fb, cb] * Ex[fa, ca]
                                if v != 0:
                                    rows.append(idx(f, ix, iy, fa + 2 * fb, nxf))
                                    cols.append(idx(f, ix // 2, iy // 2, ca + 2 * cb, nxc))
                                    vals.append(v)
    return sp.csr_matrix((vals, (rows, cols)), shape=(3 * nxf * nxf * 4, 3 * nxc * nxc * 4))

# cell blocks (12 unknowns per cell) and red-black block GS
def cell_perm(nxl):
    perm = []
    for iy in range(nxl):
        for ix in range(nxl):
            for f in range(3):
                for loc in range(4):
                    perm.append(idx(f, ix, iy, loc, nxl))
    return np.array(perm)

class Level:
    def __init__(self, A, nxl):
        self.A = A.tocsr(); self.nxl = nxl
        self.perm = cell_perm(nxl)
        Ap = self.A[self.perm][:, self.perm]
        ncl = nxl * nxl
        self.Dinv = [np.linalg.inv(Ap[12*k:12*k+12, 12*k:12*k+12].toarray()) for k in range(ncl)]
        col = np.array([(k % nxl + k // nxl) % 2 for k in range(ncl)])
        self.colors = [np.where(col == cc)[0] for cc in (0, 1)]
        self.Ap = Ap
    def gs(self, b, x, order=(0, 1)):
        # block GS in cell ordering
        bp, xp = b[self.perm], x[self.perm].copy()
        for cc in order:
            r = bp - self.Ap @ xp
            for k in self.colors[cc]:
                sl = slice(12 * k, 12 * k + 12)
                xp[sl] += self.Dinv[k] @ r[sl]
        out = np.empty_like(x); out[self.perm] = xp
        return out

def build_hier(A, nxl, nlev):
    levs = [Level(A, nxl)]; Ps = []
    for l in range(nlev - 1):
        P = prolong(nxl); Ac = (P.T @ levs[-1].A @ P).tocsr()
        nxl //= 2; Ps.append(P); levs.append(Level(Ac, nxl))
    return levs, Ps

levs, Ps = build_hier(A, nx, int(sys.argv[2]) if len(sys.argv) > 2 else 3)
coarse_lu = spl.splu(levs[-1].A.tocsc())
NU, NUC = 6, 2

# curl auxiliary space on a level: psi at vertices -> (Jx, Jy) = (dpsi/dy, -dpsi/dx)
def curl_map(nxl):
    hl = 1.0 / nxl
    nv = (nxl + 1) ** 2
    rows, cols, vals = [], [], []
    s3 = np.sqrt(3.0)
    for iy in range(nxl):
        for ix in range(nxl):
            v00, v10 = iy * (nxl + 1) + ix, iy * (nxl + 1) + ix + 1
            v01, v11 = (iy + 1) * (nxl + 1) + ix, (iy + 1) * (nxl + 1) + ix + 1
            # psi = sum psi_v N_v (bilinear).  dpsi/dy = ((1-xi)(p01-p00) + xi (p11-p10))/h
            # Legendre orthonormal on the cell: phi0 = 1/h, phi1 = sqrt3 (2xi-1)/h (per axis product, scaled)
            # coefficient of mode (a,b) = <f, phi_ab> with phi_ab orthonormal over the cell (area h^2):
            # phi_00 = 1/h ; phi_10 = sqrt3(2xi-1)/h ; phi_01 = sqrt3(2eta-1)/h
            # f = dpsi/dy linear in xi: f = A0 + A1 xi ; <f,phi_00> = h (A0 + A1/2) ; <f, phi_10> = h*A1*sqrt3/6
            for (f, g) in ((1, 'y'), (2, 'x')):
                if g == 'y':
                    # dpsi/dy = ((p01-p00) + xi((p11-p10)-(p01-p00)))/h
                    A0 = {v01: 1 / hl, v00: -1 / hl}
                    A1 = {v11: 1 / hl, v10: -1 / hl, v01: -1 / hl, v00: 1 / hl}
                    sign = 1.0; lin_loc = 1  # linear in xi -> mode a=1,b=0
                else:
                    # Jy = -dpsi/dx = -((p10-p00) + eta((p11-p01)-(p10-p00)))/h
                    A0 = {v10: -1 / hl, v00: 1 / hl}
                    A1 = {v11: -1 / hl, v01: 1 / hl, v10: 1 / hl, v00: -1 / hl}
                    sign = 1.0; lin_loc = 2  # linear in eta -> mode a=0,b=1
                for vtx in set(A0) | set(A1):
                    a0 = A0.get(vtx, 0.0); a1 = A1.get(vtx, 0.0)
                    c0 = hl * (a0 + a1 / 2); c1 = hl * a1 * s3 / 6
                    if c0: rows.append(idx(f, ix, iy, 0, nxl)); cols.append(vtx); vals.append(c0)
                    if c1: rows.append(idx(f, ix, iy, lin_loc, nxl)); cols.append(vtx); vals.append(c1)
    return sp.csr_matrix((vals, (rows, cols)), shape=(3 * nxl * nxl * 4, nv))

AUX = len(sys.argv) > 3 and sys.argv[3] == "aux"
if AUX:
    for L in levs[:1]:
        G = curl_map(L.nxl)
        L.G = G; L.Apsi = (G.T @ L.A @ G).tocsr()
        d = L.Apsi.diagonal(); L.dpsi = np.where(np.abs(d) > 0, 1.0 / d, 0.0)
        print("aux dim", L.Apsi.shape, "min diag", np.abs(d).min())

def aux_smooth(L, b, x, sweeps=2):
    # Jacobi-like GS on the potential space (forward + backward Gauss-Seidel via triangular solves)
    r = b - L.A @ x
    rp = L.G.T @ r
    Lo = sp.tril(L.Apsi).tocsr(); Up = sp.triu(L.Apsi).tocsr()
    dp = np.zeros(L.Apsi.shape[0])
    for _ in range(sweeps):
        dp = dp + spl.spsolve_triangular(Lo, rp - L.Apsi @ dp, lower=True)
        dp = dp + spl.spsolve_triangular(Up, rp - L.Apsi @ dp, lower=False)
    return x + L.G @ dp

def vcycle(l, b):
    L = levs[l]
    if l == len(levs) - 1:
        return coarse_lu.solve(b)
    nu = NU if l == 0 else NUC
    x = np.zeros_like(b)
    for _ in range(nu):
        x = L.gs(b, x, (0, 1))
    if AUX and l == 0:
        x = aux_smooth(L, b, x)
    r = b - L.A @ x
    xc = vcycle(l + 1, Ps[l].T @ r)
    x = x + Ps[l] @ xc
    if AUX and l == 0:
        x = aux_smooth(L, b, x)
    for _ in range(nu):
        x = L.gs(b, x, (1, 0))
    return x

N = A.shape[0]
M = spl.LinearOperator((N, N), matvec=lambda v: vcycle(0, v))
b = np.zeros(N); b[:n] = rng.uniform(-1, 1, n)
its = [0]
def cb(xk): its[0] += 1
t = time.time()
x, info = spl.bicgstab(A, b, M=M, rtol=1e-8, maxiter=500, callback=cb)
print("levels", len(levs), "aux" if AUX else "plain", "bicgstab its", its[0], "info", info,
      "relres %.2e" % (np.linalg.norm(b - A @ x) / np.linalg.norm(b)), "%.1f s" % (time.time() - t))

def bicgstab_l(Bop, b, ell, tol=1e-8, maxit=400):
    """BiCGStab(ell) (Sleijpen-Fokkema) on B y = b; returns (y, B applications)."""
    y = np.zeros_like(b); r = [b.copy()] + [None] * ell; u = [np.zeros_like(b)] + [None] * ell
    rt = b.copy(); rho0, alpha, omega = 1.0, 0.0, 1.0
    nb = np.linalg.norm(b); napp = 0
    while napp < maxit:
        rho0 = -omega * rho0
        for j in range(ell):
            rho1 = r[j] @ rt; beta = alpha * rho1 / rho0; rho0 = rho1
            for i in range(j + 1):
                u[i] = r[i] - beta * u[i]
            u[j + 1] = Bop(u[j]); napp += 1
            alpha = rho0 / (u[j + 1] @ rt)
            for i in range(j + 1):
                r[i] = r[i] - alpha * u[i + 1]
            r[j + 1] = Bop(r[j]); napp += 1
            y = y + alpha * u[0]
        tau = np.zeros((ell + 1, ell + 1)); sig = np.zeros(ell + 1); gp = np.zeros(ell + 1)
        for j in range(1, ell + 1):
            for i in range(1, j):
                tau[i, j] = (r[j] @ r[i]) / sig[i]
                r[j] = r[j] - tau[i, j] * r[i]
            sig[j] = r[j] @ r[j]; gp[j] = (r[0] @ r[j]) / sig[j]
        g = np.zeros(ell + 1); g[ell] = gp[ell]; omega = g[ell]
        for j in range(ell - 1, 0, -1):
            g[j] = gp[j] - sum(tau[j, i] * g[i] for i in range(j + 1, ell + 1))
        gpp = np.zeros(ell + 1)
        for j in range(1, ell):
            gpp[j] = g[j + 1] + sum(tau[j, i] * g[i + 1] for i in range(j + 1, ell))
        y = y + g[1] * r[0]; r[0] = r[0] - gp[ell] * r[ell]; u[0] = u[0] - g[ell] * u[ell]
        for j in range(1, ell):
            u[0] = u[0] - g[j] * u[j]; y = y + gpp[j] * r[j]; r[0] = r[0] - gp[j] * r[j]
        if np.linalg.norm(r[0]) <= tol * nb:
            break
    return y, napp

if len(sys.argv) > 4 and sys.argv[4] == "bicgstabl":
    Bop = lambda v: A @ vcycle(0, v)
    for ell in (1, 2, 4):
        yv, napp = bicgstab_l(Bop, b, ell)
        xv = vcycle(0, yv)
        print("BiCGStab(%d): %d preconditioner applications, true relres %.2e" %
              (ell, napp, np.linalg.norm(b - A @ xv) / np.linalg.norm(b)), flush=True)

def idrs(Bop, b, s, tol=1e-8, maxit=400):
    """IDR(s), bi-orthogonal variant (van Gijzen & Sonneveld 2011) on B y = b; returns (y, B applications)."""
    nloc = b.size
    y = np.zeros(nloc); r = b.copy(); nb = np.linalg.norm(b)
    Pm = np.linalg.qr(np.random.default_rng(5).standard_normal((nloc, s)))[0]
    G = np.zeros((nloc, s)); U = np.zeros((nloc, s)); Mm = np.eye(s); om = 1.0
    napp = 0
    while np.linalg.norm(r) > tol * nb and napp < maxit:
        f = Pm.T @ r
        done = False
        for k in range(s):
            cvec = np.linalg.solve(Mm[k:, k:], f[k:])
            v = r - G[:, k:] @ cvec
            U[:, k] = U[:, k:] @ cvec + om * v
            G[:, k] = Bop(U[:, k]); napp += 1
            for i in range(k):
                al = (Pm[:, i] @ G[:, k]) / Mm[i, i]
                G[:, k] -= al * G[:, i]; U[:, k] -= al * U[:, i]
            Mm[k:, k] = Pm[:, k:].T @ G[:, k]
            beta = f[k] / Mm[k, k]
            r = r - beta * G[:, k]; y = y + beta * U[:, k]
            if np.linalg.norm(r) <= tol * nb:
                done = True
                break
            if k + 1 < s:
                f[k + 1:] = f[k + 1:] - beta * Mm[k + 1:, k]
        if done:
            break
        t = Bop(r); napp += 1
        tr = t @ r; tn = np.linalg.norm(t); rn = np.linalg.norm(r)
        om = tr / (tn * tn)
        rho = abs(tr) / (tn * rn)
        if rho < 0.7:
            om *= 0.7 / rho
        y = y + om * r; r = r - om * t
    return y, napp

if len(sys.argv) > 4 and sys.argv[4] == "idrs":
    Bop = lambda v: A @ vcycle(0, v)
    for sdim in (1, 2, 4, 8):
        yv, napp = idrs(Bop, b, sdim)
        xv = vcycle(0, yv)
        print("IDR(%d): %d preconditioner applications, true relres %.2e" %
              (sdim, napp, np.linalg.norm(b - A @ xv) / np.linalg.norm(b)), flush=True)

if len(sys.argv) > 4 and sys.argv[4] == "mode":
    e = rng.standard_normal(N)
    rates = []
    for k in range(40):
        e_new = e - vcycle(0, A @ e)
        rates.append(np.linalg.norm(e_new) / np.linalg.norm(e))
        e = e_new / np.linalg.norm(e_new)
    print("stationary rates (last 5):", ["%.3f" % r for r in rates[-5:]])
    fn = [np.linalg.norm(e[f * n:(f + 1) * n]) for f in range(3)]
    print("field norms rho/Jx/Jy:", ["%.3f" % v for v in fn])
    # per-cell energy vs sigma_t h
    E = np.zeros(nc)
    for f in range(3):
        E += (e[f * n:(f + 1) * n].reshape(nc, 4) ** 2).sum(1)
    sth = (st * h).ravel()
    order = np.argsort(sth)
    q = np.array_split(order, 5)
    print("energy share by sigma_t h quintile (thin->thick):", ["%.3f" % (E[i].sum() / E.sum()) for i in q])
    # smoothness: fraction of e captured by the coarse space (least squares projection)
    P = Ps[0]
    coef = spl.lsqr(P, e, atol=1e-12, btol=1e-12)[0]
    print("coarse-space fraction of the slow mode: %.3f" % (np.linalg.norm(P @ coef) / np.linalg.norm(e)))
    # mode shares within rho: mean (a=b=0) vs slopes
    rr = e[:n].reshape(nc, 4)
    print("rho mode energy shares (00,10,01,11):", ["%.3f" % v for v in (rr ** 2).sum(0) / (rr ** 2).sum()])
    jj = e[n:2*n].reshape(nc, 4)
    print("Jx mode energy shares:", ["%.3f" % v for v in (jj ** 2).sum(0) / (jj ** 2).sum()])

if len(sys.argv) > 4 and sys.argv[4] == "gmres":
    for restart in (20, 40):
        cnt = [0]
        def mv(v):
            cnt[0] += 1
            return vcycle(0, v)
        M2 = spl.LinearOperator((N, N), matvec=mv)
        x, info = spl.gmres(A, b, M=M2, rtol=1e-8, restart=restart, maxiter=500)
        print("gmres(%d): precond applications %d info %d relres %.2e" % (restart, cnt[0], info, np.linalg.norm(b - A @ x) / np.linalg.norm(b)))
    cnt = [0]
    def mv2(v):
        cnt[0] += 1
        return vcycle(0, v)
    x, info = spl.bicgstab(A, b, M=spl.LinearOperator((N, N), matvec=mv2), rtol=1e-8, maxiter=500)
    print("bicgstab: precond applications %d" % cnt[0])

if len(sys.argv) > 4 and sys.argv[4] == "lines":
    # zebra line Gauss-Seidel (x-lines then y-lines) on the finest level
    L0 = levs[0]
    nxl = L0.nxl
    Ap = L0.Ap  # cell-ordered (12 per cell, cell = iy*nx + ix)
    def line_sets(axis):
        sets = []
        for par in (0, 1):
            idx_list = []
            for line in range(par, nxl, 2):
                cells = [line * nxl + i for i in range(nxl)] if axis == 0 else [i * nxl + line for i in range(nxl)]
                idx_list.append(np.concatenate([np.arange(12 * c, 12 * c + 12) for c in cells]))
            sets.append(idx_list)
        return sets
    LX, LY = line_sets(0), line_sets(1)
    facs = {}
    for nm, S_ in (("x", LX), ("y", LY)):
        for par in (0, 1):
            for k, ids in enumerate(S_[par]):
                facs[(nm, par, k)] = spl.splu(Ap[ids][:, ids].tocsc())
    def line_gs(b, x, order):
        bp, xp = b[L0.perm], x[L0.perm].copy()
        for nm in order:
            S_ = LX if nm == "x" else LY
            for par in (0, 1):
                r = bp - Ap @ xp
                for k, ids in enumerate(S_[par]):
                    xp[ids] += facs[(nm, par, k)].solve(r[ids])
        out = np.empty_like(x); out[L0.perm] = xp
        return out
    NL = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    def vcycle_l(l, b):
        L = levs[l]
        if l == len(levs) - 1:
            return coarse_lu.solve(b)
        x = np.zeros_like(b)
        if l == 0:
            for _ in range(NL):
                x = line_gs(b, x, ("x", "y"))
        else:
            for _ in range(NUC):
                x = L.gs(b, x, (0, 1))
        r = b - L.A @ x
        x = x + Ps[l] @ vcycle(l + 1, Ps[l].T @ r)
        if l == 0:
            for _ in range(NL):
                x = line_gs(b, x, ("y", "x"))
        else:
            for _ in range(NUC):
                x = L.gs(b, x, (1, 0))
        return x
    cnt = [0]
    def mv3(v):
        cnt[0] += 1
        return vcycle_l(0, v)
    x, info = spl.bicgstab(A, b, M=spl.LinearOperator((N, N), matvec=mv3), rtol=1e-8, maxiter=500)
    print("line smoother NL=%d: precond applications %d info %d" % (NL, cnt[0], info))

if len(sys.argv) > 4 and sys.argv[4] == "smoothedP":
    # two-grid with a block-Jacobi-smoothed prolongator P_s = (I - w Dinv A) P
    om = float(sys.argv[5]) if len(sys.argv) > 5 else 0.6
    L0 = levs[0]
    # block-diagonal inverse in original ordering
    Dinv_blocks = sp.block_diag(L0.Dinv).tocsr()
    perm = L0.perm
    Pm = sp.csr_matrix((np.ones(len(perm)), (perm, np.arange(len(perm)))), shape=(len(perm), len(perm)))  # cell->orig
    Dinv = Pm @ Dinv_blocks @ Pm.T
    P0 = Ps[0]
    Psm = (P0 - om * (Dinv @ (A @ P0))).tocsr()
    Ac = (Psm.T @ A @ Psm).tocsc()
    lu = spl.splu(Ac)
    def tg(bv):
        x = np.zeros_like(bv)
        for _ in range(NU):
            x = L0.gs(bv, x, (0, 1))
        r = bv - A @ x
        x = x + Psm @ lu.solve(Psm.T @ r)
        for _ in range(NU):
            x = L0.gs(bv, x, (1, 0))
        return x
    cnt = [0]
    def mv4(v):
        cnt[0] += 1
        return tg(v)
    x, info = spl.bicgstab(A, b, M=spl.LinearOperator((N, N), matvec=mv4), rtol=1e-8, maxiter=500)
    print("two-grid smoothed P (w=%.2f): precond applications %d info %d, coarse nnz %d" % (om, cnt[0], info, Ac.nnz))

if len(sys.argv) > 4 and sys.argv[4] == "spectrum":
    # dense preconditioned operator I - E, E = two/three-level error propagator
    Ad = A.toarray()
    Mi = np.zeros_like(Ad)
    for i in range(N):
        e = np.zeros(N); e[i] = 1.0
        Mi[:, i] = vcycle(0, e)
    T = Mi @ Ad
    ev = np.linalg.eigvals(T)
    mu = np.abs(1 - ev)
    print("spectral radius of I - M^-1 A: %.4f" % mu.max())
    srt = np.sort(mu)[::-1]
    print("largest |1 - lambda|:", ["%.3f" % v for v in srt[:12]])
    print("count > 0.5: %d, > 0.3: %d, > 0.1: %d of %d" % ((mu > 0.5).sum(), (mu > 0.3).sum(), (mu > 0.1).sum(), N))
    print("min |lambda| %.3e, max |lambda| %.3f, max |imag| %.3f" % (np.abs(ev).min(), np.abs(ev).max(), np.abs(ev.imag).max()))

if len(sys.argv) > 4 and sys.argv[4] == "semicoarse":
    # two-grid with x-semicoarsening (coarse grid nx/2 x ny) and an exact coarse solve
    nxf = nx
    rows, cols, vals = [], [], []
    nxc = nxf // 2
    def idx2(f, ix, iy, loc, nxl, nyl):
        return f * (nxl * nyl * 4) + (iy * nxl + ix) * 4 + loc
    for f in range(3):
        for iy in range(nxf):
            for ix in range(nxf):
                Ex = Emat(ix & 1)
                for fa in range(2):
                    for fb in range(2):
                        for ca in range(2):
                            v = Ex[fa, ca]
                            if v != 0:
                                rows.append(idx2(f, ix, iy, fa + 2 * fb, nxf, nxf))
                                cols.append(idx2(f, ix // 2, iy, ca + 2 * fb, nxc, nxf))
                                vals.append(v)
    Pxs = sp.csr_matrix((vals, (rows, cols)), shape=(3 * nxf * nxf * 4, 3 * nxc * nxf * 4))
    Acs = (Pxs.T @ A @ Pxs).tocsc()
    lus = spl.splu(Acs)
    L0 = levs[0]
    def tg2(bv):
        x = np.zeros_like(bv)
        for _ in range(NU):
            x = L0.gs(bv, x, (0, 1))
        r = bv - A @ x
        x = x + Pxs @ lus.solve(Pxs.T @ r)
        for _ in range(NU):
            x = L0.gs(bv, x, (1, 0))
        return x
    cnt = [0]
    def mv5(v):
        cnt[0] += 1
        return tg2(v)
    x, info = spl.bicgstab(A, b, M=spl.LinearOperator((N, N), matvec=mv5), rtol=1e-8, maxiter=500)
    print("two-grid x-semicoarsening: precond applications %d info %d" % (cnt[0], info))

if len(sys.argv) > 4 and sys.argv[4] == "patch":
    # red-black block GS over 2x2-cell patches (48 unknowns) on the finest level
    L0 = levs[0]
    nxl = L0.nxl
    Ap = L0.Ap
    pats = []
    for py in range(0, nxl, 2):
        for px in range(0, nxl, 2):
            cells = [(py + a) * nxl + px + b_ for a in range(2) for b_ in range(2)]
            ids = np.concatenate([np.arange(12 * c, 12 * c + 12) for c in cells])
            pats.append(((px // 2 + py // 2) % 2, ids, np.linalg.inv(Ap[ids][:, ids].toarray())))
    def patch_gs(bv, x, order):
        bp, xp = bv[L0.perm], x[L0.perm].copy()
        for col in order:
            r = bp - Ap @ xp
            for c_, ids, inv in pats:
                if c_ == col:
                    xp[ids] += inv @ r[ids]
        out = np.empty_like(x); out[L0.perm] = xp
        return out
    NPS = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    def vc(l, bv):
        L = levs[l]
        if l == len(levs) - 1:
            return coarse_lu.solve(bv)
        x = np.zeros_like(bv)
        for _ in range(NPS if l == 0 else NUC):
            x = patch_gs(bv, x, (0, 1)) if l == 0 else L.gs(bv, x, (0, 1))
        r = bv - L.A @ x
        x = x + Ps[l] @ vcycle(l + 1, Ps[l].T @ r)
        for _ in range(NPS if l == 0 else NUC):
            x = patch_gs(bv, x, (1, 0)) if l == 0 else L.gs(bv, x, (1, 0))
        return x
    cnt = [0]
    def mv6(v):
        cnt[0] += 1
        return vc(0, v)
    x, info = spl.bicgstab(A, b, M=spl.LinearOperator((N, N), matvec=mv6), rtol=1e-8, maxiter=500)
    print("patch (2x2) smoother x%d: precond applications %d info %d" % (NPS, cnt[0], info))
