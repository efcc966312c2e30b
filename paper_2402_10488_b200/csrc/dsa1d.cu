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
// partial pivoting.  The system is solved by batched block cyclic reduction
// (one CTA per sample, ceil(log2 N) levels): setup eliminates the odd
// equations of every level once and stores, per level, D^{-1}, L, U of the
// eliminated equations and A = L D_{p-1}^{-1}, C = U D_{p+1}^{-1} of the kept
// ones; each correction is then log2 N forward rhs-reduction levels and log2 N
// back-substitution levels, every level parallel over its equations.
#include "rte_internal.cuh"
#include "slab_dev.cuh"

namespace rte {
using namespace slab;

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
  int tonly;  // 1: the current block T alone, padded with identity rho rows (apply_eliminated)
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
  if (a.tonly) {
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c)
        if (r < 2 || c < 2) {
          D[4 * r + c] = r == c ? 1.0 : 0.0;
          L[4 * r + c] = 0.0;
          U[4 * r + c] = 0.0;
        }
  }
}

// Block cyclic reduction setup, one CTA per sample.  work: [S][2][N][48]
// ping-pong of the current level's (D, L, U) per position; fac: per level l
// and position p (offset off_l + p): odd p -> (D^{-1}, L, U), even p ->
// (A, C, -); the last level's single entry holds D^{-1}.
__global__ void __launch_bounds__(kCrThreads) dsa1d_factor_cr(const Dsa1DArgs a, double* __restrict__ work) {
  const int s = blockIdx.x;
  const int N = a.N;
  double* cur = work + (long)s * 2 * N * 48;
  double* nxt = cur + (long)N * 48;
  double* fac = a.fac + (long)s * cr_entries(N) * 48;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double* e = cur + (long)i * 48;
    cell_blocks(a, s, i, e, e + 16, e + 32);
  }
  __syncthreads();
  long off = 0;
  for (int n = N; n > 1; n = (n + 1) / 2) {
    double* f = fac + off * 48;
    // eliminated (odd) equations: D^{-1}, L, U
    for (int p = 1 + 2 * threadIdx.x; p < n; p += 2 * blockDim.x) {
      const double* e = cur + (long)p * 48;
      double* o = f + (long)p * 48;
      inv4(e, o);
      for (int k = 0; k < 32; ++k) o[16 + k] = e[16 + k];
    }
    __syncthreads();
    // kept (even) equations: A = L D_{p-1}^{-1}, C = U D_{p+1}^{-1}; next-level blocks
    for (int p = 2 * threadIdx.x; p < n; p += 2 * blockDim.x) {
      const double* e = cur + (long)p * 48;
      double D[16], L[16], U[16], A[16], C[16], t[16];
      for (int k = 0; k < 16; ++k) {
        D[k] = e[k];
        L[k] = 0.0;
        U[k] = 0.0;
        A[k] = 0.0;
        C[k] = 0.0;
      }
      if (p >= 1) {
        const double* m = f + (long)(p - 1) * 48;  // D^{-1}, L, U of equation p-1
        mm4(e + 16, m, A);
        mm4(A, m + 32, t);  // A U_{p-1}
        for (int k = 0; k < 16; ++k) D[k] -= t[k];
        mm4(A, m + 16, t);  // A L_{p-1}
        for (int k = 0; k < 16; ++k) L[k] = -t[k];
      }
      if (p + 1 < n) {
        const double* m = f + (long)(p + 1) * 48;
        mm4(e + 32, m, C);
        mm4(C, m + 16, t);  // C L_{p+1}
        for (int k = 0; k < 16; ++k) D[k] -= t[k];
        mm4(C, m + 32, t);  // C U_{p+1}
        for (int k = 0; k < 16; ++k) U[k] = -t[k];
      }
      double* o = f + (long)p * 48;
      for (int k = 0; k < 16; ++k) {
        o[k] = A[k];
        o[16 + k] = C[k];
        o[32 + k] = 0.0;
      }
      double* q = nxt + (long)(p / 2) * 48;
      for (int k = 0; k < 16; ++k) {
        q[k] = D[k];
        q[16 + k] = L[k];
        q[32 + k] = U[k];
      }
    }
    __syncthreads();
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
    off += n;
  }
  if (threadIdx.x == 0) inv4(cur, fac + off * 48);
}

// Interleaved factor table -> compact component-major layout (slab_dev.cuh
// crc_*), one CTA per sample.
__global__ void dsa1d_repack_kernel(int N, const double* __restrict__ fac, double* __restrict__ fc) {
  const int s = blockIdx.x;
  const double* f = fac + (long)s * cr_entries(N) * 48;
  double* o = fc + (long)s * crc_doubles(N);
  long off = 0, co = 0;
  for (int n = N; n > 1; n = (n + 1) / 2) {
    const int ne = (n + 1) / 2, no = n / 2;
    for (int t = threadIdx.x; t < ne * 32; t += blockDim.x) {
      const int c = t / ne, m = t - c * ne;  // component c of kept equation p = 2m
      o[co + t] = f[(off + 2 * m) * 48 + c];
    }
    for (int t = threadIdx.x; t < no * 48; t += blockDim.x) {
      const int c = t / no, m = t - c * no;  // component c of eliminated equation p = 2m + 1
      o[co + (long)ne * 32 + t] = f[(off + 2 * m + 1) * 48 + c];
    }
    off += n;
    co += crc_level_size(n);
  }
  for (int t = threadIdx.x; t < 16; t += blockDim.x) o[co + t] = f[off * 48 + t];
}

struct Dsa1DSolve {
  int S, N, block;
  const double* fac;
  const double* ms;      // to form Ms * delta when apply_ms
  const double* rhs;     // [S][2N]
  double* out;           // [S][2N]
  double* work;          // [S][N][4]: reduced right-hand sides, then the solution
  const int* kind;       // optional mask: only samples with kind == KIND_DSA
  int apply_ms;
  int prepared;          // 1: work already holds the 4-vector rhs; the solution stays in work
};

// Block cyclic reduction solve, one CTA per sample.
__global__ void __launch_bounds__(kCrThreads) dsa1d_solve_cr(const Dsa1DSolve a) {
  const int s = blockIdx.x;
  if (a.kind && a.kind[s] != KIND_DSA) return;
  const int N = a.N;
  const long nd = 2L * N;
  const double* r = a.rhs + (long)s * nd;
  double* y = a.work + (long)s * N * 4;
  const double* fac = a.fac + (long)s * cr_entries(N) * 48;
  // rhs [(Ms) rho ; 0] per cell
  for (int i = threadIdx.x; i < N && !a.prepared; i += blockDim.x) {
    double r0 = r[2 * i], r1 = r[2 * i + 1];
    if (a.apply_ms) {
      if (a.block == 4) {
        const double* m = a.ms + ((long)s * N + i) * 4;
        const double t0 = m[0] * r0 + m[1] * r1, t1 = m[2] * r0 + m[3] * r1;
        r0 = t0;
        r1 = t1;
      } else {
        const double sg = a.ms[(long)s * N + i];
        r0 *= sg;
        r1 *= sg;
      }
    }
    y[4 * i] = r0;
    y[4 * i + 1] = r1;
    y[4 * i + 2] = 0.0;
    y[4 * i + 3] = 0.0;
  }
  __syncthreads();
  cr_solve_cta(N, fac, y);
  for (int i = threadIdx.x; i < N && !a.prepared; i += blockDim.x) {
    a.out[(long)s * nd + 2 * i] = y[4 * i];
    a.out[(long)s * nd + 2 * i + 1] = y[4 * i + 1];
  }
}

// Current-eliminated operator pieces (dsa.cpp:279-293) from the coupled
// blocks of cell i: phase 0 -> work_i = (0, 0, (A_Jr x)_i); phase 1 ->
// out_i = (A_rr x)_i - (A_rJ y)_i with y_i = work_i[2..3] = T^{-1} A_Jr x.
__global__ void k_elim1d(const Dsa1DArgs a, int phase, const double* __restrict__ x, double* __restrict__ work,
                         double* __restrict__ out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)a.S * a.N) return;
  const int s = (int)(t / a.N), i = (int)(t - (long)s * a.N);
  double B[3][16];
  cell_blocks(a, s, i, B[0], B[1], B[2]);
  const double* xs = x + (long)s * 2 * a.N;
  const double* ys = work + (long)s * a.N * 4;
  const int nb[3] = {i, i - 1, i + 1};
  double acc[2] = {0.0, 0.0};
  for (int k = 0; k < 3; ++k) {
    const int j = nb[k];
    if (j < 0 || j >= a.N) continue;
    const double* m = B[k];
    for (int r = 0; r < 2; ++r) {
      if (phase == 0) {
        acc[r] += m[4 * (r + 2)] * xs[2 * j] + m[4 * (r + 2) + 1] * xs[2 * j + 1];
      } else {
        acc[r] += m[4 * r] * xs[2 * j] + m[4 * r + 1] * xs[2 * j + 1];
        acc[r] -= m[4 * r + 2] * ys[4 * j + 2] + m[4 * r + 3] * ys[4 * j + 3];
      }
    }
  }
  if (phase == 0) {
    double* w = work + t * 4;
    w[0] = 0.0;
    w[1] = 0.0;
    w[2] = acc[0];
    w[3] = acc[1];
  } else {
    out[t * 2] = acc[0];
    out[t * 2 + 1] = acc[1];
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
  d->fac_t.release();
  moments(ctx->vx, ctx->w, d->m1, d->m2, d->m3);
  d->fac.alloc((size_t)ctx->S * cr_entries(ctx->ncells) * 48);
  Dsa1DArgs a{ctx->S, ctx->ncells, ctx->block, ctx->width.p, ctx->mt.p, ctx->ms.p, d->m1, d->m2, d->m3, d->fac.p};
  DBuf<double> work;
  work.alloc((size_t)ctx->S * 2 * ctx->ncells * 48);
  dsa1d_factor_cr<<<ctx->S, kCrThreads, 0, st>>>(a, work.p);
  RTE_CUDA(cudaGetLastError());
  d->fac_c.alloc((size_t)ctx->S * crc_doubles(ctx->ncells));
  dsa1d_repack_kernel<<<ctx->S, 256, 0, st>>>(ctx->ncells, d->fac.p, d->fac_c.p);
  RTE_CUDA(cudaGetLastError());
  RTE_CUDA(cudaStreamSynchronize(st));
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
  dsa1d_solve_cr<<<ctx->S, std::min(kCrThreads, std::max(32, (ctx->ncells + 1) / 2 / 32 * 32 + 32)), 0, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

void dsa2d_status_reset(rte_ctx* ctx, cudaStream_t st);
void dsa2d_status_read(rte_ctx* ctx, int* host, cudaStream_t st);
void dsa2d_history_reset(rte_ctx* ctx, cudaStream_t st);

// Per-sample rte_dsa_status of the solves since the last reset.  The slab
// solve is a direct block cyclic reduction (no iteration to fall short).
void dsa_status_reset(rte_ctx* ctx, cudaStream_t st) {
  if (ctx->dsa && ctx->dsa->impl2d) dsa2d_status_reset(ctx, st);
}
void dsa_status_read(rte_ctx* ctx, int* host, cudaStream_t st) {
  if (ctx->dsa && ctx->dsa->impl2d)
    dsa2d_status_read(ctx, host, st);
  else
    std::fill(host, host + ctx->S, 0);
}
const int* dsa2d_status_dev(rte_ctx* ctx);
const int* dsa_status_dev(rte_ctx* ctx) {
  return ctx->dsa && ctx->dsa->impl2d ? dsa2d_status_dev(ctx) : nullptr;
}
void dsa_history_reset(rte_ctx* ctx, cudaStream_t st) {
  if (ctx->dsa && ctx->dsa->impl2d) dsa2d_history_reset(ctx, st);
}
// throws RTE_ERR_RUNTIME naming the first sample whose solve fell short
void dsa_status_check(rte_ctx* ctx, cudaStream_t st, const char* what) {
  std::vector<int> f(ctx->S);
  dsa_status_read(ctx, f.data(), st);
  for (int s = 0; s < ctx->S; ++s)
    if (f[s] != RTE_DSA_OK) {
      static const char* why[] = {"ok", "iteration cap reached", "breakdown", "non-finite residual"};
      throw Error(RTE_ERR_RUNTIME, std::string(what) + ": coupled moment system solve failed at sample " +
                                       std::to_string(s) + " (" + why[f[s] & 3] + ")");
    }
}

void dsa_solve_density(rte_ctx* ctx, const double* rhs, double* out, const int* kind, cudaStream_t st) {
  dsa_apply(ctx, rhs, out, kind, 0, st);
}

void dsa2d_apply_eliminated(rte_ctx* ctx, const double* x, double* out, cudaStream_t st);

// DsaOperator::apply_eliminated (dsa.cpp:279-293): S x = A_rr x - A_rJ T^{-1} A_Jr x.
// Slab: T (the J-J block, block tridiagonal) is factored lazily on first use
// by the same block cyclic reduction, padded to 4x4 blocks with identity rho
// rows, like the reference's lazily built current-block SparseLU.
void dsa_apply_eliminated(rte_ctx* ctx, const double* x, double* out, cudaStream_t st) {
  RTE_REQUIRE(ctx->dsa, RTE_ERR_INVALID, "dsa: rte_dsa_setup was not called");
  if (ctx->geom == RTE_XY2D) {
    dsa2d_apply_eliminated(ctx, x, out, st);
    return;
  }
  DsaState* d = ctx->dsa;
  const int S = ctx->S, N = ctx->ncells;
  Dsa1DArgs a{S, N, ctx->block, ctx->width.p, ctx->mt.p, ctx->ms.p, d->m1, d->m2, d->m3, nullptr, 0};
  if (!d->fac_t.p) {
    d->fac_t.alloc((size_t)S * cr_entries(N) * 48);
    Dsa1DArgs at = a;
    at.fac = d->fac_t.p;
    at.tonly = 1;
    DBuf<double> work;
    work.alloc((size_t)S * 2 * N * 48);
    dsa1d_factor_cr<<<S, kCrThreads, 0, st>>>(at, work.p);
    RTE_CUDA(cudaGetLastError());
    RTE_CUDA(cudaStreamSynchronize(st));
  }
  ctx->ws_e.alloc((size_t)S * N * 4);
  const int nb = (int)(((long)S * N + 255) / 256);
  k_elim1d<<<nb, 256, 0, st>>>(a, 0, x, ctx->ws_e.p, nullptr);
  Dsa1DSolve sv{S, N, ctx->block, d->fac_t.p, nullptr, nullptr, nullptr, ctx->ws_e.p, nullptr, 0, 1};
  dsa1d_solve_cr<<<S, std::min(kCrThreads, std::max(32, (N + 1) / 2 / 32 * 32 + 32)), 0, st>>>(sv);
  k_elim1d<<<nb, 256, 0, st>>>(a, 1, x, ctx->ws_e.p, out);
  RTE_CUDA(cudaGetLastError());
}

void dsa_destroy(DsaState* d) {
  if (!d) return;
  if (d->impl2d) dsa2d_destroy(d->impl2d);
  delete d;
}

long dsa_coupled_dim(const rte_ctx* ctx) { return ctx->dsa ? ctx->dsa->dim : (ctx->geom == RTE_XY2D ? 3 : 2) * ctx->ndof; }

}  // namespace rte
