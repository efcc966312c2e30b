// kinetic.cu -- K8: kinetic-space term operators and batched snapshot
// collection (the offline training path).
//
// apply_term_kinetic (transport_system.cpp:560-596):
//   term 0: out_j = D_j u_j + Mt_0 u_j - Ms_0 avg      (D_j = upwind streaming)
//   term k: out_j =           Mt_k u_j - Ms_k avg      (k >= 1)
// with avg = sum_j w_j u_j (density_of), for a batch of kinetic columns.
// collect_snapshots (snapshots.cpp:118-194): training SI-DSA in kinetic form
// for every sample of the context, storing f^(l) (l <= window), drho^(l) and
// the converged f.
#include <cmath>

#include "rte_internal.cuh"

namespace rte {

void dsa_apply(rte_ctx* ctx, const double* rhs, double* out, const int* kind, int apply_ms, cudaStream_t st);

namespace {

struct TermArgs {
  int geom, nx, ny, nl, nv, block, k, ncols;
  long ndof;
  const double* width;   // slab widths
  double hx, hy;
  const double* vx;
  const double* vy;
  const double* tmt;     // [cells][block] of term k
  const double* tms;
  const double* avg;     // [ncols][ndof]
  const double* u;       // [ncols][nv][ndof]
  double* out;
};

// 1D upwind streaming D_j f for cell i (transport_system.cpp:446-478).
__device__ void dj_1d(const TermArgs& a, double v, const double* f, int i, double* o) {
  const int n = a.nx;
  const double h = a.width[i];
  const double s = 1.0 / sqrt(h);
  const double trL0 = s, trL1 = -kSqrt3 * s, trR0 = s, trR1 = kSqrt3 * s;
  if (v > 0) {
    const double fr = f[2 * i] * trR0 + f[2 * i + 1] * trR1;
    o[0] = v * fr * trR0;
    o[1] = v * (fr * trR1 - 2.0 * kSqrt3 / h * f[2 * i]);
    if (i > 0) {
      const double su = 1.0 / sqrt(a.width[i - 1]);
      const double u = f[2 * i - 2] * su + f[2 * i - 1] * kSqrt3 * su;
      o[0] -= v * u * trL0;
      o[1] -= v * u * trL1;
    }
  } else {
    const double fl = f[2 * i] * trL0 + f[2 * i + 1] * trL1;
    o[0] = -v * fl * trL0;
    o[1] = -v * (fl * trL1 + 2.0 * kSqrt3 / h * f[2 * i]);
    if (i < n - 1) {
      const double su = 1.0 / sqrt(a.width[i + 1]);
      const double u = f[2 * i + 2] * su + f[2 * i + 3] * (-kSqrt3 * su);
      o[0] += v * u * trR0;
      o[1] += v * u * trR1;
    }
  }
}

// 2D upwind streaming (apply_streaming_collision without the collision term,
// transport_system.cpp:490-551).
__device__ void dj_2d(const TermArgs& a, double ux, double uy, const double* f, int ix, int iy, double* oc) {
  const int nx = a.nx, ny = a.ny;
  const double hx = a.hx, hy = a.hy;
  const double rx = 1.0 / sqrt(hx), ry = 1.0 / sqrt(hy);
  const double bxL0 = rx, bxL1 = -kSqrt3 * rx, bxR0 = rx, bxR1 = kSqrt3 * rx;
  const double byL0 = ry, byL1 = -kSqrt3 * ry, byR0 = ry, byR1 = kSqrt3 * ry;
  const int cell = ix + nx * iy;
  const double* fc = f + 4 * cell;
  for (int k = 0; k < 4; ++k) oc[k] = 0.0;
  for (int b = 0; b < 2; ++b) {
    const double c0 = fc[2 * b], c1 = fc[2 * b + 1];
    if (ux > 0) {
      const double fr = c0 * bxR0 + c1 * bxR1;
      oc[2 * b] += ux * fr * bxR0;
      oc[2 * b + 1] += ux * (fr * bxR1 - 2.0 * kSqrt3 / hx * c0);
      if (ix > 0) {
        const double* cu = f + 4 * (cell - 1);
        const double u = cu[2 * b] * bxR0 + cu[2 * b + 1] * bxR1;
        oc[2 * b] -= ux * u * bxL0;
        oc[2 * b + 1] -= ux * u * bxL1;
      }
    } else {
      const double fl = c0 * bxL0 + c1 * bxL1;
      oc[2 * b] += -ux * fl * bxL0;
      oc[2 * b + 1] += -ux * (fl * bxL1 + 2.0 * kSqrt3 / hx * c0);
      if (ix < nx - 1) {
        const double* cu = f + 4 * (cell + 1);
        const double u = cu[2 * b] * bxL0 + cu[2 * b + 1] * bxL1;
        oc[2 * b] += ux * u * bxR0;
        oc[2 * b + 1] += ux * u * bxR1;
      }
    }
  }
  for (int aa = 0; aa < 2; ++aa) {
    const double c0 = fc[aa], c1 = fc[aa + 2];
    if (uy > 0) {
      const double fr = c0 * byR0 + c1 * byR1;
      oc[aa] += uy * fr * byR0;
      oc[aa + 2] += uy * (fr * byR1 - 2.0 * kSqrt3 / hy * c0);
      if (iy > 0) {
        const double* cu = f + 4 * (cell - nx);
        const double u = cu[aa] * byR0 + cu[aa + 2] * byR1;
        oc[aa] -= uy * u * byL0;
        oc[aa + 2] -= uy * u * byL1;
      }
    } else {
      const double fl = c0 * byL0 + c1 * byL1;
      oc[aa] += -uy * fl * byL0;
      oc[aa + 2] += -uy * (fl * byL1 + 2.0 * kSqrt3 / hy * c0);
      if (iy < ny - 1) {
        const double* cu = f + 4 * (cell + nx);
        const double u = cu[aa] * byL0 + cu[aa + 2] * byL1;
        oc[aa] += uy * u * byR0;
        oc[aa + 2] += uy * u * byR1;
      }
    }
  }
}

__global__ void k_term_apply(const TermArgs a) {
  const long ncell = a.geom == RTE_SLAB1D ? a.nx : (long)a.nx * a.ny;
  const long per_col = (long)a.nv * ncell;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)a.ncols * per_col) return;
  const long col = t / per_col;
  const long rem = t - col * per_col;
  const int j = (int)(rem / ncell);
  const int cell = (int)(rem - (long)j * ncell);
  const int nl = a.nl;
  const double* uj = a.u + (col * a.nv + j) * a.ndof;
  const double* av = a.avg + col * a.ndof;
  double o[4] = {0, 0, 0, 0};
  if (a.k == 0) {
    if (a.geom == RTE_SLAB1D)
      dj_1d(a, a.vx[j], uj, cell, o);
    else
      dj_2d(a, a.vx[j], a.vy[j], uj, cell % a.nx, cell / a.nx, o);
  }
  // + Mt_k u_j - Ms_k avg (per-cell blocks, transport_system.cpp:589-594)
  for (int r = 0; r < nl; ++r) {
    double s1 = 0, s2 = 0;
    for (int q = 0; q < nl; ++q) {
      double mtk, msk;
      if (a.block == 1) {
        mtk = r == q ? a.tmt[cell] : 0.0;
        msk = r == q ? a.tms[cell] : 0.0;
      } else {
        mtk = a.tmt[(long)cell * a.block + nl * r + q];
        msk = a.tms[(long)cell * a.block + nl * r + q];
      }
      s1 += mtk * uj[(long)nl * cell + q];
      s2 += msk * av[(long)nl * cell + q];
    }
    o[r] += s1;
    o[r] -= s2;
  }
  double* oj = a.out + (col * a.nv + j) * a.ndof + (long)nl * cell;
  for (int r = 0; r < nl; ++r) oj[r] = o[r];
}

__global__ void k_density_cols(int ncols, int nv, long nd, const double* __restrict__ w, const double* __restrict__ u,
                               double* __restrict__ avg) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)ncols * nd) return;
  const long col = t / nd, i = t - col * nd;
  double v = 0.0;
  for (int j = 0; j < nv; ++j) v = v + w[j] * u[(col * nv + j) * nd + i];
  avg[t] = v;
}

// training bookkeeping: store f / drho for l <= window, convergence test
__global__ void k_snap_step(int S, long kdim, long nd, int l, int window, double eps, const double* __restrict__ f,
                            const double* __restrict__ drho, double* __restrict__ f_iter,
                            double* __restrict__ drho_iter, double* __restrict__ f_conv, int* __restrict__ active,
                            int* __restrict__ conv, int* __restrict__ n_iter, const unsigned long long* bits) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < kdim; i += (long)gridDim.x * blockDim.x) {
    const double v = f[(long)s * kdim + i];
    if (l <= window) f_iter[((long)s * window + (l - 1)) * kdim + i] = v;
    f_conv[(long)s * kdim + i] = v;  // last f is the converged snapshot (snapshots.cpp:167)
    if (l <= window && i < nd) drho_iter[((long)s * window + (l - 1)) * nd + i] = drho[(long)s * nd + i];
  }
}

__global__ void k_snap_decide(int S, int l, double eps, const unsigned long long* bits, int* active, int* conv,
                              int* n_iter, int* kind, int* n_active, int max_iters) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  if (!active[s]) {
    kind[s] = KIND_IDLE;
    return;
  }
  const double ch = __longlong_as_double((long long)bits[2 * s]);
  n_iter[s] = l;
  if (ch < eps) {
    conv[s] = 1;
    active[s] = 0;
    kind[s] = KIND_ACCEPT;
    return;
  }
  kind[s] = KIND_DSA;
  if (l >= max_iters)
    active[s] = 0;
  else
    atomicAdd(n_active, 1);
}

__global__ void k_snap_update(int S, long nd, const int* kind, const double* rstar, const double* corr, double* rho) {
  const int s = blockIdx.y;
  if (kind[s] != KIND_DSA) return;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += (long)gridDim.x * blockDim.x)
    rho[(long)s * nd + i] = rstar[(long)s * nd + i] + corr[(long)s * nd + i];
}

// (D_j + Sigma_t) f for one direction and every sample (transport_system.cpp:
// 482-558): upwind streaming with zero inflow plus the sample's Mt blocks.
__global__ void k_stream_coll(const TermArgs a, int S, int j, const double* __restrict__ mt) {
  const long ncell = a.geom == RTE_SLAB1D ? a.nx : (long)a.nx * a.ny;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)S * ncell) return;
  const int s = (int)(t / ncell);
  const int cell = (int)(t - (long)s * ncell);
  const int nl = a.nl;
  const double* fs = a.u + (long)s * a.ndof;
  double o[4] = {0, 0, 0, 0};
  if (a.geom == RTE_SLAB1D)
    dj_1d(a, a.vx[j], fs, cell, o);
  else
    dj_2d(a, a.vx[j], a.vy[j], fs, cell % a.nx, cell / a.nx, o);
  for (int r = 0; r < nl; ++r) {
    double v = 0.0;
    if (a.block == 1) {
      v = mt[(long)s * ncell + cell] * fs[(long)nl * cell + r];
    } else {
      const double* m = mt + ((long)s * ncell + cell) * a.block + (long)nl * r;
      for (int q = 0; q < nl; ++q) v += m[q] * fs[(long)nl * cell + q];
    }
    a.out[(long)s * a.ndof + (long)nl * cell + r] = o[r] + v;
  }
}

// out[s] += psi[s][k] * t[s] over the kinetic vectors of every sample
__global__ void k_psi_axpy(int S, long kdim, int K, int k, const double* __restrict__ psi,
                           const double* __restrict__ t, double* __restrict__ out, int first) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)S * kdim) return;
  const int s = (int)(i / kdim);
  const double v = psi[(long)s * K + k] * t[i];
  out[i] = first ? v : out[i] + v;
}

}  // namespace

void apply_streaming_collision(rte_ctx* ctx, int j, const double* f, double* out, cudaStream_t st) {
  DBuf<double> dvx, dvy;
  dvx.upload(ctx->vx.data(), ctx->nv);
  dvy.upload(ctx->vy.data(), ctx->nv);
  TermArgs a{};
  a.geom = ctx->geom;
  a.nx = ctx->nx;
  a.ny = ctx->ny;
  a.nl = ctx->nl;
  a.nv = ctx->nv;
  a.block = ctx->block;
  a.ndof = ctx->ndof;
  a.width = ctx->width.p;
  a.hx = ctx->hx;
  a.hy = ctx->hy;
  a.vx = dvx.p;
  a.vy = dvy.p;
  a.u = f;
  a.out = out;
  const long n = (long)ctx->S * ctx->ncells;
  k_stream_coll<<<(int)((n + 127) / 128), 128, 0, st>>>(a, ctx->S, j, ctx->mt.p);
  RTE_CUDA(cudaGetLastError());
  RTE_CUDA(cudaStreamSynchronize(st));
}

// A_mu u = sum_k psi_k(mu_s) A_k u_s for every sample (transport_system.cpp:598-613)
void apply_kinetic(rte_ctx* ctx, const double* u, double* out, cudaStream_t st) {
  RTE_REQUIRE(ctx->k_terms > 0 && ctx->psi.p, RTE_ERR_INVALID,
              "apply_kinetic: call rte_set_affine with per-term mass blocks first");
  const long kdim = (long)ctx->nv * ctx->ndof;
  DBuf<double> t;
  t.alloc((size_t)ctx->S * kdim);
  const long n = (long)ctx->S * kdim;
  for (int k = 0; k < ctx->k_terms; ++k) {
    apply_term_kinetic(ctx, k, ctx->S, u, t.p, st);
    k_psi_axpy<<<(int)((n + 255) / 256), 256, 0, st>>>(ctx->S, kdim, ctx->k_terms, k, ctx->psi.p, t.p, out,
                                                         k == 0 ? 1 : 0);
    RTE_CUDA(cudaGetLastError());
  }
  RTE_CUDA(cudaStreamSynchronize(st));
}

void apply_term_kinetic(rte_ctx* ctx, int k, int ncols, const double* u, double* out, cudaStream_t st) {
  RTE_REQUIRE(ctx->k_terms > 0 && ctx->term_mt.p, RTE_ERR_INVALID,
              "apply_term_kinetic: call rte_set_affine with per-term mass blocks first");
  RTE_REQUIRE(k >= 0 && k < ctx->k_terms, RTE_ERR_INVALID, "apply_term_kinetic: bad term index");
  DBuf<double> avg, dvx, dvy, dw;
  avg.alloc((size_t)ncols * ctx->ndof);
  dvx.upload(ctx->vx.data(), ctx->nv);
  dvy.upload(ctx->vy.data(), ctx->nv);
  dw.upload(ctx->w.data(), ctx->nv);
  const long n1 = (long)ncols * ctx->ndof;
  k_density_cols<<<(int)((n1 + 255) / 256), 256, 0, st>>>(ncols, ctx->nv, ctx->ndof, dw.p, u, avg.p);
  TermArgs a{};
  a.geom = ctx->geom;
  a.nx = ctx->nx;
  a.ny = ctx->ny;
  a.nl = ctx->nl;
  a.nv = ctx->nv;
  a.block = ctx->block;
  a.k = k;
  a.ncols = ncols;
  a.ndof = ctx->ndof;
  a.width = ctx->width.p;
  a.hx = ctx->hx;
  a.hy = ctx->hy;
  a.vx = dvx.p;
  a.vy = dvy.p;
  a.tmt = ctx->term_mt.p + (size_t)k * ctx->ncells * ctx->block;
  a.tms = ctx->term_ms.p + (size_t)k * ctx->ncells * ctx->block;
  a.avg = avg.p;
  a.u = u;
  a.out = out;
  const long n = (long)ncols * ctx->nv * ctx->ncells;
  k_term_apply<<<(int)((n + 127) / 128), 128, 0, st>>>(a);
  RTE_CUDA(cudaGetLastError());
  RTE_CUDA(cudaStreamSynchronize(st));
}

void kinetic_fixed_point(rte_ctx* ctx, const double* rho, double* rstar, double* f, const int* active,
                         double* delta, unsigned long long* bits, cudaStream_t st);

void collect_snapshots(rte_ctx* ctx, int window, double eps, int max_iters, double* f_iter, double* f_conv,
                       double* drho_iter, int* conv_h, int* n_iter_h, cudaStream_t st) {
  const int S = ctx->S;
  const long nd = ctx->ndof, kdim = (long)ctx->nv * nd;
  if (!ctx->dsa) dsa_setup(ctx, st);
  dsa_history_reset(ctx, st);
  dsa_status_reset(ctx, st);
  DBuf<double> rho, rstar, delta, corr, f;
  rho.alloc((size_t)S * nd);
  rstar.alloc((size_t)S * nd);
  delta.alloc((size_t)S * nd);
  corr.alloc((size_t)S * nd);
  f.alloc((size_t)S * kdim);
  rho.zero(st);
  DBuf<int> ib;
  ib.alloc((size_t)4 * S + 1);
  RTE_CUDA(cudaMemsetAsync(ib.p, 0, sizeof(int) * (4 * S + 1), st));
  int* active = ib.p;
  int* conv = ib.p + S;
  int* n_iter = ib.p + 2 * S;
  int* kind = ib.p + 3 * S;
  int* n_act = ib.p + 4 * S;
  {
    std::vector<int> ones(S, 1);
    RTE_CUDA(cudaMemcpyAsync(active, ones.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
    RTE_CUDA(cudaStreamSynchronize(st));
  }
  DBuf<unsigned long long> bits;
  bits.alloc((size_t)2 * S);
  int h_act = S;
  for (int l = 1; l <= max_iters && h_act > 0; ++l) {
    bits.zero(st);
    kinetic_fixed_point(ctx, rho.p, rstar.p, f.p, active, delta.p, bits.p, st);
    const int bx = (int)std::min<long>((kdim + 255) / 256, 1024);
    k_snap_step<<<dim3(bx, S), 256, 0, st>>>(S, kdim, nd, l, window, eps, f.p, delta.p, f_iter, drho_iter, f_conv,
                                             active, conv, n_iter, bits.p);
    RTE_CUDA(cudaMemsetAsync(n_act, 0, sizeof(int), st));
    k_snap_decide<<<(S + 127) / 128, 128, 0, st>>>(S, l, eps, bits.p, active, conv, n_iter, kind, n_act, max_iters);
    dsa_apply(ctx, delta.p, corr.p, kind, 1, st);
    const int bx2 = (int)std::min<long>((nd + 255) / 256, 1024);
    k_snap_update<<<dim3(bx2, S), 256, 0, st>>>(S, nd, kind, rstar.p, corr.p, rho.p);
    RTE_CUDA(cudaGetLastError());
    RTE_CUDA(cudaMemcpyAsync(&h_act, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
    RTE_CUDA(cudaStreamSynchronize(st));
  }
  RTE_CUDA(cudaMemcpy(conv_h, conv, sizeof(int) * S, cudaMemcpyDeviceToHost));
  RTE_CUDA(cudaMemcpy(n_iter_h, n_iter, sizeof(int) * S, cudaMemcpyDeviceToHost));
  dsa_status_check(ctx, st, "collect_snapshots: DSA correction");
}

}  // namespace rte
