// sweep1d.cu -- K1: batched 1D upwind-DG transport sweep with fused
// scalar-flux reduction, source assembly and SI epilogue.
//
// Replaces TransportSystem::sweep_into 1D branch (transport_system.cpp:
// 279-310) and the direction loops of apply_L / assemble_rhs / kinetic_sweep
// (transport_system.cpp:393-431).
//
// Algorithm.  For one direction the reference visits cells in upwind order,
//   f_i = B_i^{-1} (rhs_i + |v| u_{i-1} t_in,i),   u_i = t_out,i . f_i,
// with B_i = streaming(v, h_i) + Mt_i (transport_system.cpp:74-78, 214-227)
// and t_in / t_out the basis traces on the inflow / outflow face.  The only
// quantity carried between cells is the scalar outflow trace u, which obeys
// the first-order affine recurrence u_i = alpha_i + beta_i u_{i-1}
// (alpha_i = t_out.B_i^{-1} rhs_i, beta_i = |v| t_out.B_i^{-1} t_in).  One
// warp owns one (sample, direction) chain: each lane composes the affine maps
// of its CPL consecutive cells, a 5-step shuffle scan composes the lanes, and
// a second pass rebuilds f with the exact incoming trace.  B_i^{-1} is formed
// on the fly (the reference caches it per direction slot and cell).
//
// One CTA per sample; warps take directions in rounds; the sum
// rho = sum_j w_j f_j is accumulated in shared memory in the fixed order
// j = 0..n-1 (deterministic, like transport_system.cpp:398-401).
#include <cstdlib>

#include "rte_internal.cuh"
#include "slab_dev.cuh"

namespace rte {
namespace {
using namespace slab;

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

template <int CPL, bool CACHED>
__global__ void __launch_bounds__(256) sweep1d_kernel(const Sweep1DArgs a) {
  extern __shared__ double sm[];
  const int s = blockIdx.x;
  if (a.active && !a.active[s]) return;
  const long nd = a.ndof;
  constexpr int NV = 2 * 32 * CPL;  // lane-major vector length (slab_dev.cuh)
  double* q = sm;
  double* acc = sm + NV;
  double* stage = sm + 2 * NV;
  const int lane = threadIdx.x & 31;
  sweep_cta<CPL, CACHED>(a, s, a.rho ? a.rho + (long)s * nd : nullptr, false, q, acc, stage);

  if (a.out) {
    double mx_d = 0.0, mx_r = 0.0;
    for (long i = threadIdx.x; i < nd; i += blockDim.x) {
      const double o = acc[lane_major_dof<CPL>(i)];
      a.out[(long)s * nd + i] = o;
      if (a.delta) {
        const double dd = o - a.rho_prev[(long)s * nd + i];
        a.delta[(long)s * nd + i] = dd;
        mx_d = fmax(mx_d, fabs(dd));
        mx_r = fmax(mx_r, fabs(o));
        if (dd != dd) mx_d = dd;  // propagate NaN
      }
    }
    if (a.change_bits) {
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        mx_d = fmax(mx_d, __shfl_xor_sync(0xffffffffu, mx_d, d));
        mx_r = fmax(mx_r, __shfl_xor_sync(0xffffffffu, mx_r, d));
      }
      if (lane == 0) {
        atomicMax(a.change_bits + 2 * s, dbits(fabs(mx_d)));
        atomicMax(a.change_bits + 2 * s + 1, dbits(mx_r));
      }
    }
  }
}

template <int CPL>
void launch_cpl(const Sweep1DArgs& a, cudaStream_t st) {
  const long nv = 2 * 32 * CPL;  // lane-major vector length
  const int jn = a.j_single >= 0 ? 1 : a.nv;
  int nw = 8;  // 256 threads: at 512 ptxas caps the kernel at 64 registers and spills
  const long budget = 200 * 1024;
  while (nw > 1 && (long)(2 + nw) * nv * 8 > budget) nw >>= 1;
  nw = std::min(nw, std::max(1, jn));
  const size_t smem = (size_t)(2 + nw) * nv * 8;
  RTE_REQUIRE(smem <= (size_t)(227 * 1024), RTE_ERR_UNSUPPORTED, "sweep1d: slab too large for one CTA");
  static bool configured = false;
  if (!configured) {
    RTE_CUDA(cudaFuncSetAttribute(sweep1d_kernel<CPL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    RTE_CUDA(cudaFuncSetAttribute(sweep1d_kernel<CPL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    configured = true;
  }
  if (a.cache)
    sweep1d_kernel<CPL, true><<<a.S, nw * 32, smem, st>>>(a);
  else
    sweep1d_kernel<CPL, false><<<a.S, nw * 32, smem, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

// One thread per (sample, direction, sweep position): the cell block inverse
// and trace gain exactly as the on-the-fly path computes them.
__global__ void slab_cache_kernel(Sweep1DArgs a, int cpl, double* cache, double* sc_out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int N = a.N;
  if (t >= (long)a.S * a.nv * N) return;
  const int p = (int)(t % N);
  const long sj = t / N;
  const int j = (int)(sj % a.nv), s = (int)(sj / a.nv);
  const double v = a.vx[j];
  const bool fwd = v > 0;
  const int i = fwd ? p : N - 1 - p;
  double bi[4];
  cell_block(a, s, i, v, bi);
  const double sc = 1.0 / sqrt(a.width[i]);
  const double be = trace_gain(bi, sc, fabs(v), fwd);
  const long stride = 32L * cpl;
  double* e = cache + sj * 5 * stride + (long)(p % cpl) * 32 + p / cpl;
  e[0] = bi[0];
  e[stride] = bi[1];
  e[2 * stride] = bi[2];
  e[3 * stride] = bi[3];
  e[4 * stride] = be;
  if (sj == 0) sc_out[i] = sc;
}

}  // namespace

int sweep1d_cpl(int N) {
  for (int c = 1; c <= 128; c *= 2)
    if (N <= 32 * c) return c;
  return 0;
}

void slab_cache_ensure(rte_ctx* ctx, cudaStream_t st) {
  if (ctx->slab_cache_tried) return;
  ctx->slab_cache_tried = true;
  static const bool off = [] {  // RTE_SLAB_CACHE=0: cell blocks on the fly (tests of that path)
    const char* e = std::getenv("RTE_SLAB_CACHE");
    return e && std::atoi(e) == 0;
  }();
  if (off) return;
  const int cpl = sweep1d_cpl(ctx->ncells);
  if (!cpl) return;
  const size_t n = (size_t)ctx->S * ctx->nv * 5 * 32 * cpl;
  const size_t fr = device_free_bytes();
  if (n * sizeof(double) > std::min<size_t>(fr / 4, (size_t)4 << 30)) return;  // on the fly instead
  ctx->slab_cache.alloc(n);
  ctx->slab_sc.alloc(ctx->ncells);
  Sweep1DArgs a{};
  a.S = ctx->S;
  a.N = ctx->ncells;
  a.nv = ctx->nv;
  a.width = ctx->width.p;
  a.vx = ctx->dvx.p;
  a.block = ctx->block;
  a.mt = ctx->mt.p;
  const long total = (long)ctx->S * ctx->nv * ctx->ncells;
  slab_cache_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a, cpl, ctx->slab_cache.p, ctx->slab_sc.p);
  RTE_CUDA(cudaGetLastError());
}

void launch_sweep1d(const Sweep1DArgs& a, cudaStream_t st) {
  const int N = a.N;
  if (N <= 32) return launch_cpl<1>(a, st);
  if (N <= 64) return launch_cpl<2>(a, st);
  if (N <= 128) return launch_cpl<4>(a, st);
  if (N <= 256) return launch_cpl<8>(a, st);
  if (N <= 512) return launch_cpl<16>(a, st);
  if (N <= 1024) return launch_cpl<32>(a, st);
  if (N <= 2048) return launch_cpl<64>(a, st);
  if (N <= 4096) return launch_cpl<128>(a, st);
  throw Error(RTE_ERR_UNSUPPORTED, "sweep1d: more than 4096 cells");
}

}  // namespace rte
