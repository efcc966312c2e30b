// rom.cu -- K6: online reduced-order stage on the device.
//
// Replaces ReducedModel::assemble (reduced_model.cpp:32-39), romig
// (strategies.cpp:8-28) and RomsaStrategy::setup/correct
// (strategies.cpp:34-53) for a batch of parameter samples.  Per sample the
// reduced operator A_r(mu) = sum_k psi_k(mu) a_r[k] is factored once with
// complete pivoting and the same rank test as Eigen::FullPivLU
// (|pivot| > eps * r * |max pivot|); each ROMSA correction is
//   rhs_r = U_iso^T (Ms delta),  c = A_r^{-1} rhs_r,  corr = U_rho c,
// done by one CTA per sample with fixed-order block reductions.
#include "rte_internal.cuh"
#include "slab_dev.cuh"

namespace rte {

struct RomState {
  int r = 0, K = 0;
  double eps_pod = 0, eps_train = 0;
  DBuf<double> u_rho, u_iso, a_r, b_r;  // column-major as in the reference
  DBuf<double> lu;                      // [S][r][r] row-major factors
  DBuf<int> rp, cp, sing;               // [S][r], [S][r], [S]
  DBuf<double> part, coef;              // batched correction: [chunks][S][r] partial projections, [S][r]
  bool factored = false;
};

namespace {
using namespace slab;

// Complete-pivoting LU of the r x r row-major matrix in place.
__device__ int fullpiv_lu(double* a, int r, int* rp, int* cp) {
  for (int i = 0; i < r; ++i) {
    rp[i] = i;
    cp[i] = i;
  }
  double maxpiv = 0.0;
  int nz = r;
  for (int k = 0; k < r; ++k) {
    double big = 0.0;
    int bi = k, bj = k;
    for (int j = k; j < r; ++j)  // column-major traversal, first maximum
      for (int i = k; i < r; ++i) {
        const double v = fabs(a[i * r + j]);
        if (v > big) {
          big = v;
          bi = i;
          bj = j;
        }
      }
    if (big == 0.0) {
      nz = k;
      break;
    }
    maxpiv = fmax(maxpiv, big);
    if (bi != k) {
      for (int j = 0; j < r; ++j) {
        const double t = a[k * r + j];
        a[k * r + j] = a[bi * r + j];
        a[bi * r + j] = t;
      }
      const int t = rp[k];
      rp[k] = rp[bi];
      rp[bi] = t;
    }
    if (bj != k) {
      for (int i = 0; i < r; ++i) {
        const double t = a[i * r + k];
        a[i * r + k] = a[i * r + bj];
        a[i * r + bj] = t;
      }
      const int t = cp[k];
      cp[k] = cp[bj];
      cp[bj] = t;
    }
    const double piv = a[k * r + k];
    for (int i = k + 1; i < r; ++i) {
      const double l = a[i * r + k] / piv;
      a[i * r + k] = l;
      for (int j = k + 1; j < r; ++j) a[i * r + j] -= l * a[k * r + j];
    }
  }
  const double thr = 2.220446049250313e-16 * r * maxpiv;
  int rank = 0;
  for (int i = 0; i < nz; ++i)
    if (fabs(a[i * r + i]) > thr) ++rank;
  return rank;
}

// A(mu_s) = sum_k psi_k a_r[k] (reduced_model.cpp:32-39), row-major.
__device__ void assemble(const double* a_r, const double* psi, int r, int K, double* out) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      double t = 0.0;
      for (int k = 0; k < K; ++k) t = t + psi[k] * a_r[(long)k * r * r + (long)j * r + i];
      out[i * r + j] = t;
    }
}

// One warp per sample (r <= 32; larger ranks: one thread per sample).
__global__ void rom_factor_kernel(int S, int r, int K, const double* a_r, const double* psi, double* lu, int* rp,
                                  int* cp, int* sing) {
  __shared__ double am[4][32 * 32];
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int s = blockIdx.x * 4 + w;
  if (s >= S) return;
  if (r > 32) {  // serial fallback
    if (ln) return;
    double* a = lu + (long)s * r * r;
    assemble(a_r, psi + (long)s * K, r, K, a);
    const int rank = fullpiv_lu(a, r, rp + (long)s * r, cp + (long)s * r);
    sing[s] = rank < r ? 1 : 0;
    return;
  }
  double* a = am[w];
  const double* ps = psi + (long)s * K;
  for (int e = ln; e < r * r; e += 32) {  // assemble (reduced_model.cpp:32-39), row-major
    const int i = e / r, j = e - i * r;
    double t = 0.0;
    for (int k = 0; k < K; ++k) t = t + ps[k] * a_r[(long)k * r * r + (long)j * r + i];
    a[e] = t;
  }
  __syncwarp();
  const int rank = warp_fullpiv_lu(a, r, rp + (long)s * r, cp + (long)s * r);
  for (int e = ln; e < r * r; e += 32) lu[(long)s * r * r + e] = a[e];
  if (ln == 0) sing[s] = rank < r ? 1 : 0;
}

struct RomCorrectArgs {
  int S, r, N, block;
  long nd;
  const double* u_rho;
  const double* u_iso;
  const double* lu;
  const int* rp;
  const int* cp;
  const double* ms;
  const double* delta;
  double* corr;
  const int* kind;
};

__global__ void rom_correct_kernel(const RomCorrectArgs a) {
  __shared__ double rhs[128], y[128], c[128], red[32 * 8];
  const int s = blockIdx.x;
  if (a.kind[s] != KIND_ROMSA) return;
  block_dots<8>(a.u_iso, a.nd, a.r, nullptr, a.ms, a.block, a.N, a.delta + (long)s * a.nd, s, rhs, red);
  if (a.r <= 32) {
    if (threadIdx.x < 32)
      warp_fullpiv_solve(a.lu + (long)s * a.r * a.r, a.r, a.rp + (long)s * a.r, a.cp + (long)s * a.r, rhs, c);
  } else if (threadIdx.x == 0) {
    fullpiv_solve(a.lu + (long)s * a.r * a.r, a.r, a.rp + (long)s * a.r, a.cp + (long)s * a.r, rhs, y, c);
  }
  __syncthreads();
  for (long i = threadIdx.x; i < a.nd; i += blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < a.r; ++k) t = fma(a.u_rho[(long)k * a.nd + i], c[k], t);
    a.corr[(long)s * a.nd + i] = t;
  }
}

// ---- batched ROMSA correction (the S per-sample GEMVs as two passes over the
// basis: U_iso^T [Ms delta]_S and U_rho C_S) -----------------
constexpr int kRomRows = 256;  // basis rows per CTA (staged in shared memory)

// partial projections of the chunk's rows: part[c][s][k] = sum_i U_iso[k][i] (Ms delta_s)_i
__global__ void __launch_bounds__(256) rom_proj_partial(int S, int r, int N, int block, long nd,
                                                         const double* __restrict__ u_iso,
                                                         const double* __restrict__ ms,
                                                         const double* __restrict__ delta, const int* __restrict__ kind,
                                                         double* __restrict__ part) {
  extern __shared__ double us[];  // [r][kRomRows]
  __shared__ double red[8][32];
  const long i0 = (long)blockIdx.x * kRomRows;
  const int rows = (int)min((long)kRomRows, nd - i0);
  for (int e = threadIdx.x; e < r * kRomRows; e += blockDim.x) {
    const int k = e / kRomRows, t = e - k * kRomRows;
    us[e] = t < rows ? u_iso[(long)k * nd + i0 + t] : 0.0;
  }
  __syncthreads();
  const int nl = (int)(nd / N);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int s = 0; s < S; ++s) {
    if (kind[s] != KIND_ROMSA) continue;  // uniform over the CTA
    const int t = threadIdx.x;
    double m = 0.0;
    if (t < rows) {  // (Ms delta)_i, as block_dots forms it
      const long i = i0 + t;
      const double* d = delta + (long)s * nd;
      if (block == nl * nl) {
        const long c = i / nl;
        const int rr = (int)(i - c * nl);
        const double* mm = ms + ((long)s * N + c) * block + nl * rr;
        for (int q = 0; q < nl; ++q) m = fma(mm[q], d[nl * c + q], m);
      } else {
        m = ms[(long)s * N + i / nl] * d[i];
      }
    }
    for (int k0 = 0; k0 < r; k0 += 32) {
      // lanes of a warp: the chunk's partial for 32 modes at a time
      double acc[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) acc[k] = (k0 + k < r) ? us[(k0 + k) * kRomRows + t] * m : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
      // lane k keeps mode k0 + k of this warp's sum
      double mine = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (ln == k) mine = acc[k];
      red[w][ln] = mine;
      __syncthreads();
      if (threadIdx.x < 32 && k0 + threadIdx.x < r) {
        double v = 0.0;
        for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) v += red[ww][threadIdx.x];
        part[((long)blockIdx.x * S + s) * r + k0 + threadIdx.x] = v;
      }
      __syncthreads();
    }
  }
}

// one warp per ROMSA sample: fixed-order sum of the chunk partials, then the
// reduced solve (r <= 32)
__global__ void rom_proj_finish(int S, int r, int nchunks, const double* __restrict__ part, const double* lu,
                                const int* rp, const int* cp, const int* __restrict__ kind, double* __restrict__ coef) {
  __shared__ double rhs[4][32], cc[4][32];
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int s = blockIdx.x * 4 + w;
  if (s >= S || kind[s] != KIND_ROMSA) return;
  double v = 0.0;
  if (ln < r)
    for (int c = 0; c < nchunks; ++c) v += part[((long)c * S + s) * r + ln];
  rhs[w][ln] = v;
  __syncwarp();
  warp_fullpiv_solve(lu + (long)s * r * r, r, rp + (long)s * r, cp + (long)s * r, rhs[w], cc[w]);
  __syncwarp();
  if (ln < r) coef[(long)s * r + ln] = cc[w][ln];
}

// corr_s = U_rho c_s for the ROMSA samples, the chunk of U_rho staged once
__global__ void __launch_bounds__(256) rom_lift(int S, int r, long nd, const double* __restrict__ u_rho,
                                                const double* __restrict__ coef, const int* __restrict__ kind,
                                                double* __restrict__ corr) {
  extern __shared__ double us[];  // [r][kRomRows]
  const long i0 = (long)blockIdx.x * kRomRows;
  const int rows = (int)min((long)kRomRows, nd - i0);
  for (int e = threadIdx.x; e < r * kRomRows; e += blockDim.x) {
    const int k = e / kRomRows, t = e - k * kRomRows;
    us[e] = t < rows ? u_rho[(long)k * nd + i0 + t] : 0.0;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= rows) return;
  for (int s = 0; s < S; ++s) {
    if (kind[s] != KIND_ROMSA) continue;
    const double* c = coef + (long)s * r;
    double v = 0.0;
    for (int k = 0; k < r; ++k) v = fma(us[k * kRomRows + t], c[k], v);
    corr[(long)s * nd + i0 + t] = v;
  }
}

struct RomigArgs {
  int S, r, K;
  long nd;
  const double* a_r;
  const double* b_r;
  const double* psi;
  const double* u_rho;
  double* work;  // [S][r*r]
  int* rp;
  int* cp;
  double* rho0;
  int* status;
};

__global__ void romig_kernel(const RomigArgs a) {
  __shared__ double c[128], y[128], b[128];
  __shared__ double am[32 * 32];
  __shared__ int ok;
  const int s = blockIdx.x;
  const int r = a.r;
  int* rp = a.rp + (long)s * r;
  int* cp = a.cp + (long)s * r;
  if (r <= 32) {
    // one warp: assemble, complete-pivoting LU, solve, Galerkin residual check
    if (threadIdx.x < 32) {
      const int ln = threadIdx.x;
      const double* ps = a.psi + (long)s * a.K;
      for (int e = ln; e < r * r; e += 32) {
        const int i = e / r, j = e - i * r;
        double t = 0.0;
        for (int k = 0; k < a.K; ++k) t = t + ps[k] * a.a_r[(long)k * r * r + (long)j * r + i];
        am[e] = t;
      }
      if (ln < r) b[ln] = a.b_r[ln];
      __syncwarp();
      const int rank = warp_fullpiv_lu(am, r, rp, cp);
      if (rank < r) {
        if (ln == 0) {
          a.status[s] = 1;
          ok = 0;
        }
      } else {
        warp_fullpiv_solve(am, r, rp, cp, b, c);
        __syncwarp();
        // Galerkin residual check (strategies.cpp:20-27), lane i = row i
        double resid = 0.0, rs = 0.0, cm = 0.0, bm = 0.0;
        if (ln < r) {
          double t = 0.0;
          for (int j = 0; j < r; ++j) {
            double aij = 0.0;
            for (int k = 0; k < a.K; ++k) aij = aij + ps[k] * a.a_r[(long)k * r * r + (long)j * r + ln];
            t += aij * c[j];
            rs += fabs(aij);
          }
          resid = fabs(b[ln] - t);
          cm = fabs(c[ln]);
          bm = fabs(b[ln]);
        }
        for (int o = 16; o > 0; o >>= 1) {
          resid = fmax(resid, __shfl_xor_sync(0xffffffffu, resid, o));
          rs = fmax(rs, __shfl_xor_sync(0xffffffffu, rs, o));
          cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
          bm = fmax(bm, __shfl_xor_sync(0xffffffffu, bm, o));
        }
        if (ln == 0) {
          const double scale = rs * cm + bm;
          const bool good = !(resid > 1e-10 * fmax(scale, 1e-300));
          a.status[s] = good ? 0 : 2;
          ok = good ? 1 : 0;
        }
      }
    }
  } else if (threadIdx.x == 0) {
    double* lu = a.work + (long)s * r * r;
    assemble(a.a_r, a.psi + (long)s * a.K, r, a.K, lu);
    for (int i = 0; i < r; ++i) b[i] = a.b_r[i];
    const int rank = fullpiv_lu(lu, r, rp, cp);
    ok = 1;
    if (rank < r) {
      a.status[s] = 1;
      ok = 0;
    } else {
      fullpiv_solve(lu, r, rp, cp, b, y, c);
      // Galerkin residual check (strategies.cpp:20-27)
      double resid = 0.0, rowmax = 0.0, cmax = 0.0, bmax = 0.0;
      for (int i = 0; i < r; ++i) {
        double t = 0.0, rs = 0.0;
        for (int j = 0; j < r; ++j) {
          double aij = 0.0;
          for (int k = 0; k < a.K; ++k) aij = aij + a.psi[(long)s * a.K + k] * a.a_r[(long)k * r * r + (long)j * r + i];
          t += aij * c[j];
          rs += fabs(aij);
        }
        resid = fmax(resid, fabs(b[i] - t));
        rowmax = fmax(rowmax, rs);
        cmax = fmax(cmax, fabs(c[i]));
        bmax = fmax(bmax, fabs(b[i]));
      }
      const double scale = rowmax * cmax + bmax;
      if (resid > 1e-10 * fmax(scale, 1e-300)) {
        a.status[s] = 2;
        ok = 0;
      } else {
        a.status[s] = 0;
      }
    }
  }
  __syncthreads();
  for (long i = threadIdx.x; i < a.nd; i += blockDim.x) {
    double t = 0.0;
    if (ok)
      for (int k = 0; k < r; ++k) t = fma(a.u_rho[(long)k * a.nd + i], c[k], t);
    a.rho0[(long)s * a.nd + i] = t;
  }
}

}  // namespace

void rom_load(rte_ctx* ctx, int which, const rte_rom* rom) {
  RTE_REQUIRE(which == 0 || which == 1, RTE_ERR_INVALID, "rom_load: which must be 0 or 1");
  RTE_REQUIRE(rom && rom->rank > 0 && rom->rank <= 128, RTE_ERR_INVALID, "rom_load: rank must be in [1,128]");
  RTE_REQUIRE(ctx->k_terms > 0, RTE_ERR_INVALID, "rom_load: call rte_set_affine first (psi per sample)");
  RTE_REQUIRE(rom->k_affine == ctx->k_terms, RTE_ERR_INVALID,
              "reduced model: affine term count does not match the system");
  if (!ctx->rom[which]) ctx->rom[which] = new RomState();
  RomState* m = ctx->rom[which];
  m->r = rom->rank;
  m->K = rom->k_affine;
  m->eps_pod = rom->eps_pod;
  m->eps_train = rom->eps_train;
  const size_t nd = (size_t)ctx->ndof, r = (size_t)m->r;
  m->u_rho.upload(rom->u_rho, nd * r);
  m->u_iso.upload(rom->u_iso, nd * r);
  m->a_r.upload(rom->a_r, (size_t)m->K * r * r);
  m->b_r.upload(rom->b_r, r);
  m->lu.alloc((size_t)ctx->S * r * r);
  m->rp.alloc((size_t)ctx->S * r);
  m->cp.alloc((size_t)ctx->S * r);
  m->sing.alloc((size_t)ctx->S);
  m->factored = false;
}

void rom_setup(rte_ctx* ctx, int which, int* singular_dev, cudaStream_t st) {
  RomState* m = ctx->rom[which];
  RTE_REQUIRE(m, RTE_ERR_INVALID, "rom: model not loaded");
  rom_factor_kernel<<<(ctx->S + 3) / 4, 128, 0, st>>>(ctx->S, m->r, m->K, m->a_r.p, ctx->psi.p, m->lu.p, m->rp.p,
                                                       m->cp.p, m->sing.p);
  RTE_CUDA(cudaGetLastError());
  if (singular_dev) RTE_CUDA(cudaMemcpyAsync(singular_dev, m->sing.p, sizeof(int) * ctx->S, cudaMemcpyDeviceToDevice, st));
  m->factored = true;
}

void rom_correct(rte_ctx* ctx, const double* delta, double* corr, const int* kind, cudaStream_t st) {
  RomState* m = ctx->rom[1];
  RTE_REQUIRE(m && m->factored, RTE_ERR_INVALID, "rom: correction model not set up");
  const int S = ctx->S, r = m->r;
  const long nd = ctx->ndof;
  if (r <= 32) {  // batched: the basis is read once per correction, not once per sample
    const int nchunks = (int)((nd + kRomRows - 1) / kRomRows);
    m->part.ensure((size_t)nchunks * S * r);
    m->coef.ensure((size_t)S * r);
    const size_t smem = sizeof(double) * r * kRomRows;
    rom_proj_partial<<<nchunks, 256, smem, st>>>(S, r, ctx->ncells, ctx->block, nd, m->u_iso.p, ctx->ms.p, delta,
                                                 kind, m->part.p);
    rom_proj_finish<<<(S + 3) / 4, 128, 0, st>>>(S, r, nchunks, m->part.p, m->lu.p, m->rp.p, m->cp.p, kind,
                                                 m->coef.p);
    rom_lift<<<nchunks, 256, smem, st>>>(S, r, nd, m->u_rho.p, m->coef.p, kind, corr);
    RTE_CUDA(cudaGetLastError());
    return;
  }
  RomCorrectArgs a{S, r, ctx->ncells, ctx->block, nd, m->u_rho.p, m->u_iso.p, m->lu.p, m->rp.p,
                   m->cp.p, ctx->ms.p, delta, corr, kind};
  rom_correct_kernel<<<S, 256, 0, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

void rom_fill_si1d(rte_ctx* ctx, Si1DArgs& a) {
  RomState* m = ctx->rom[1];
  RTE_REQUIRE(m && m->factored, RTE_ERR_INVALID, "rom: correction model not set up");
  a.r = m->r;
  a.u_rho = m->u_rho.p;
  a.u_iso = m->u_iso.p;
  a.lu = m->lu.p;
  a.rp = m->rp.p;
  a.cp = m->cp.p;
}

void romig(rte_ctx* ctx, double* rho0, int* status_dev, cudaStream_t st) {
  RomState* m = ctx->rom[0];
  RTE_REQUIRE(m, RTE_ERR_INVALID, "romig: primary model not loaded");
  DBuf<double> work;
  work.alloc((size_t)ctx->S * m->r * m->r);
  RomigArgs a{ctx->S, m->r, m->K, ctx->ndof, m->a_r.p, m->b_r.p, ctx->psi.p, m->u_rho.p, work.p, m->rp.p, m->cp.p,
              rho0, status_dev};
  romig_kernel<<<ctx->S, 256, 0, st>>>(a);
  RTE_CUDA(cudaGetLastError());
  RTE_CUDA(cudaStreamSynchronize(st));
}

void rom_destroy(RomState* r) { delete r; }

}  // namespace rte
