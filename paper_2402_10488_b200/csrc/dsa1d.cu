// dsa1d.cu -- K4: batched consistent-DSA solve for slab geometry.
//
// Replaces DsaOperator (dsa.cpp:154-277) for Slab1D: the coupled P1 moment
// system in (rho, J) that the reference assembles as a sparse matrix
// (dsa.cpp:197-215) and factors with Eigen::SparseLU (dsa.cpp:253).
//
// With the unknowns of cell i ordered [rho_0, rho_1, J_0, J_1] the matrix is
// block tridiagonal with 4x4 blocks
//   D_i = [[Ma_i - m1 DJ_ii,  3 m2 Dc_ii], [m2 Dc_ii,  3 m2 Mt_i - 3 m3 DJ_ii]]
//   L_i (to i-1) and U_i (to i+1) from the face couplings,
// where DJ = Dm - Dp (jump part), Dc = (Dp + Dm)/2 (central part) of the
// upwind/downwind streaming matrices (dsa.cpp:34-110) and m1, m2, m3 are
// quadrature moments (dsa.cpp:167-192).  After scaling the J rows by 3 the
// matrix is positive-real, so block elimination without
// inter-block pivoting is stable; each 4x4 pivot block is inverted with
// partial pivoting.  Setup factors once per sample (block Thomas: stores
// Dt_i^{-1}, G_i = L_i Dt_{i-1}^{-1}, U_i); each correction is one forward
// and one backward block substitution.  Samples run in parallel.
#include "rte_internal.cuh"

namespace rte {

namespace {

// 4x4 inverse by Gauss-Jordan with partial pivoting (row-major).
__device__ void inv4(const double* m, double* o) {
  double a[4][8];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      a[r][c] = m[4 * r + c];
      a[r][c + 4] = r == c ? 1.0 : 0.0;
    }
  for (int k = 0; k < 4; ++k) {
    int piv = k;
    double best = fabs(a[k][k]);
    for (int r = k + 1; r < 4; ++r)
      if (fabs(a[r][k]) > best) {
        best = fabs(a[r][k]);
        piv = r;
      }
    if (piv != k)
      for (int c = 0; c < 8; ++c) {
        const double t = a[k][c];
        a[k][c] = a[piv][c];
        a[piv][c] = t;
      }
    const double id = 1.0 / a[k][k];
    for (int c = 0; c < 8; ++c) a[k][c] *= id;
    for (int r = 0; r < 4; ++r)
      if (r != k) {
        const double f = a[r][k];
        for (int c = 0; c < 8; ++c) a[r][c] -= f * a[k][c];
      }
  }
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) o[4 * r + c] = a[r][c + 4];
}

__device__ void mm4(const double* x, const double* y, double* o) {
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      double t = 0;
      for (int k = 0; k < 4; ++k) t += x[4 * r + k] * y[4 * k + c];
      o[4 * r + c] = t;
    }
}

struct Dsa1DArgs {
  int S, N, block;
  const double* width;
  const double* mt;
  const double* ms;
  double m1, m2, m3;
  double* fac;
};

// Blocks of cell i (dsa.cpp:34-110, 197-215 with unknowns interleaved per cell).
__device__ void cell_blocks(const Dsa1DArgs& a, int s, int i, double* D, double* L, double* U) {
  const int N = a.N;
  const double h = a.width[i];
  const double er[4] = {1 / h, kSqrt3 / h, kSqrt3 / h, 3 / h};
  const double el[4] = {1 / h, -kSqrt3 / h, -kSqrt3 / h, 3 / h};
  const double sd[4] = {0, 0, 2.0 * kSqrt3 / h, 0};
  double dp[4], dm[4], dj[4], dc[4];
  for (int e = 0; e < 4; ++e) {
    dp[e] = er[e] - sd[e];
    dm[e] = -el[e] - sd[e];
    dj[e] = dm[e] - dp[e];
    dc[e] = 0.5 * dp[e] + 0.5 * dm[e];
  }
  double mt[4], ma[4];
  if (a.block == 4) {
    for (int e = 0; e < 4; ++e) {
      mt[e] = a.mt[((long)s * N + i) * 4 + e];
      ma[e] = mt[e] - a.ms[((long)s * N + i) * 4 + e];
    }
  } else {
    const double st = a.mt[(long)s * N + i], ss = a.ms[(long)s * N + i];
    mt[0] = st; mt[1] = 0; mt[2] = 0; mt[3] = st;
    ma[0] = st - ss; ma[1] = 0; ma[2] = 0; ma[3] = st - ss;
  }
  // D = [[Ma - m1 DJ, 3 m2 Dc], [m2 Dc, 3 m2 Mt - 3 m3 DJ]]
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      const int e = 2 * r + c;
      D[4 * r + c] = ma[e] - a.m1 * dj[e];
      D[4 * r + c + 2] = 3.0 * a.m2 * dc[e];
      D[4 * (r + 2) + c] = a.m2 * dc[e];
      D[4 * (r + 2) + c + 2] = 3.0 * a.m2 * mt[e] - 3.0 * a.m3 * dj[e];
    }
  for (int e = 0; e < 16; ++e) {
    L[e] = 0;
    U[e] = 0;
  }
  if (i > 0) {
    // Dp(i,i-1) = -cpl_p; DJ(i,i-1) = +cpl_p; Dc(i,i-1) = -cpl_p / 2
    const double si = 1.0 / sqrt(h), su = 1.0 / sqrt(a.width[i - 1]);
    const double cp[4] = {si * su, si * kSqrt3 * su, -kSqrt3 * si * su, -3 * si * su};
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) {
        const int e = 2 * r + c;
        const double djv = cp[e], dcv = 0.5 * (-cp[e]);
        L[4 * r + c] = -a.m1 * djv;
        L[4 * r + c + 2] = 3.0 * a.m2 * dcv;
        L[4 * (r + 2) + c] = a.m2 * dcv;
        L[4 * (r + 2) + c + 2] = -3.0 * a.m3 * djv;
      }
  }
  if (i < N - 1) {
    // Dm(i,i+1) = cpl_m; DJ(i,i+1) = cpl_m; Dc(i,i+1) = cpl_m / 2
    const double si = 1.0 / sqrt(h), su = 1.0 / sqrt(a.width[i + 1]);
    const double cm[4] = {si * su, -si * kSqrt3 * su, kSqrt3 * si * su, -3 * si * su};
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) {
        const int e = 2 * r + c;
        const double djv = cm[e], dcv = 0.5 * cm[e];
        U[4 * r + c] = -a.m1 * djv;
        U[4 * r + c + 2] = 3.0 * a.m2 * dcv;
        U[4 * (r + 2) + c] = a.m2 * dcv;
        U[4 * (r + 2) + c + 2] = -3.0 * a.m3 * djv;
      }
  }
}

// Block Thomas factorization, one thread per sample.
__global__ void dsa1d_factor(const Dsa1DArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  double D[16], L[16], U[16], Dt[16], inv[16], prev_inv[16], G[16], GU[16];
  for (int i = 0; i < a.N; ++i) {
    cell_blocks(a, s, i, D, L, U);
    double* f = a.fac + ((long)s * a.N + i) * 48;
    if (i == 0) {
      for (int e = 0; e < 16; ++e) Dt[e] = D[e];
      for (int e = 0; e < 16; ++e) G[e] = 0;
    } else {
      mm4(L, prev_inv, G);
      double Uprev[16];
      const double* fp = a.fac + ((long)s * a.N + i - 1) * 48;
      for (int e = 0; e < 16; ++e) Uprev[e] = fp[32 + e];
      mm4(G, Uprev, GU);
      for (int e = 0; e < 16; ++e) Dt[e] = D[e] - GU[e];
    }
    inv4(Dt, inv);
    for (int e = 0; e < 16; ++e) {
      f[e] = inv[e];
      f[16 + e] = G[e];
      f[32 + e] = U[e];
      prev_inv[e] = inv[e];
    }
  }
}

struct Dsa1DSolve {
  int S, N, block;
  const double* fac;
  const double* ms;      // to form Ms * delta when apply_ms
  const double* rhs;     // [S][2N]
  double* out;           // [S][2N]
  double* work;          // [S][N][4]
  const int* kind;       // optional mask: only samples with kind == KIND_DSA
  int apply_ms;
};

__global__ void dsa1d_solve(const Dsa1DSolve a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  if (a.kind && a.kind[s] != KIND_DSA) return;
  const long nd = 2L * a.N;
  const double* r = a.rhs + (long)s * nd;
  double* y = a.work + (long)s * a.N * 4;
  double yp[4] = {0, 0, 0, 0};
  for (int i = 0; i < a.N; ++i) {
    const double* f = a.fac + ((long)s * a.N + i) * 48;
    double r0 = r[2 * i], r1 = r[2 * i + 1];
    if (a.apply_ms) {
      if (a.block == 4) {
        const double* m = a.ms + ((long)s * a.N + i) * 4;
        const double t0 = m[0] * r0 + m[1] * r1, t1 = m[2] * r0 + m[3] * r1;
        r0 = t0;
        r1 = t1;
      } else {
        const double sg = a.ms[(long)s * a.N + i];
        r0 *= sg;
        r1 *= sg;
      }
    }
    double v[4] = {r0, r1, 0.0, 0.0};
    if (i > 0)
      for (int k = 0; k < 4; ++k)
        v[k] -= f[16 + 4 * k] * yp[0] + f[16 + 4 * k + 1] * yp[1] + f[16 + 4 * k + 2] * yp[2] +
                f[16 + 4 * k + 3] * yp[3];
    for (int k = 0; k < 4; ++k) {
      y[4 * i + k] = v[k];
      yp[k] = v[k];
    }
  }
  double xn[4] = {0, 0, 0, 0};
  for (int i = a.N - 1; i >= 0; --i) {
    const double* f = a.fac + ((long)s * a.N + i) * 48;
    double v[4];
    for (int k = 0; k < 4; ++k) v[k] = y[4 * i + k];
    if (i < a.N - 1)
      for (int k = 0; k < 4; ++k)
        v[k] -= f[32 + 4 * k] * xn[0] + f[32 + 4 * k + 1] * xn[1] + f[32 + 4 * k + 2] * xn[2] +
                f[32 + 4 * k + 3] * xn[3];
    double x[4];
    for (int k = 0; k < 4; ++k) x[k] = f[4 * k] * v[0] + f[4 * k + 1] * v[1] + f[4 * k + 2] * v[2] + f[4 * k + 3] * v[3];
    for (int k = 0; k < 4; ++k) xn[k] = x[k];
    a.out[(long)s * nd + 2 * i] = x[0];
    a.out[(long)s * nd + 2 * i + 1] = x[1];
  }
}

}  // namespace

void dsa2d_setup(rte_ctx* ctx, cudaStream_t st);
void dsa2d_solve(rte_ctx* ctx, const double* rhs, double* out, const int* kind, int apply_ms, cudaStream_t st);
void dsa2d_destroy(void* p);

// dsa.cpp:167-192: angular moments with the transport quadrature.
static void moments(const std::vector<double>& c, const std::vector<double>& w, double& m1, double& m2,
                    double& m3) {
  m1 = m2 = m3 = 0;
  for (size_t j = 0; j < c.size(); ++j) {
    if (c[j] > 0) m1 += w[j] * c[j];
    m2 += w[j] * c[j] * c[j];
    if (c[j] > 0) m3 += w[j] * c[j] * c[j] * c[j];
  }
}

void dsa_setup(rte_ctx* ctx, cudaStream_t st) {
  if (!ctx->dsa) ctx->dsa = new DsaState();
  DsaState* d = ctx->dsa;
  if (ctx->geom == RTE_XY2D) {
    d->nf = 3;
    d->dim = 3 * ctx->ndof;
    dsa2d_setup(ctx, st);
    return;
  }
  d->nf = 2;
  d->dim = 2 * ctx->ndof;
  moments(ctx->vx, ctx->w, d->m1, d->m2, d->m3);
  d->fac.alloc((size_t)ctx->S * ctx->ncells * 48);
  Dsa1DArgs a{ctx->S, ctx->ncells, ctx->block, ctx->width.p, ctx->mt.p, ctx->ms.p, d->m1, d->m2, d->m3, d->fac.p};
  dsa1d_factor<<<(ctx->S + 63) / 64, 64, 0, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

// out = C rhs (solve_density) or C Ms rhs (correct) depending on apply_ms;
// kind != null restricts to samples whose SI step chose DSA.
void dsa_apply(rte_ctx* ctx, const double* rhs, double* out, const int* kind, int apply_ms, cudaStream_t st) {
  RTE_REQUIRE(ctx->dsa, RTE_ERR_INVALID, "dsa: rte_dsa_setup was not called");
  if (ctx->geom == RTE_XY2D) {
    dsa2d_solve(ctx, rhs, out, kind, apply_ms, st);
    return;
  }
  ctx->ws_e.alloc((size_t)ctx->S * ctx->ncells * 4);
  Dsa1DSolve a{ctx->S, ctx->ncells, ctx->block, ctx->dsa->fac.p, ctx->ms.p, rhs, out, ctx->ws_e.p, kind, apply_ms};
  dsa1d_solve<<<(ctx->S + 31) / 32, 32, 0, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

void dsa_solve_density(rte_ctx* ctx, const double* rhs, double* out, const int* kind, cudaStream_t st) {
  dsa_apply(ctx, rhs, out, kind, 0, st);
}

void dsa_destroy(DsaState* d) {
  if (!d) return;
  if (d->impl2d) dsa2d_destroy(d->impl2d);
  delete d;
}

long dsa_coupled_dim(const rte_ctx* ctx) { return ctx->dsa ? ctx->dsa->dim : (ctx->geom == RTE_XY2D ? 3 : 2) * ctx->ndof; }

}  // namespace rte
