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
#include "rte_internal.cuh"

namespace rte {
namespace {

__device__ __forceinline__ void cell_block(const Sweep1DArgs& a, int s, int i, double v, double* binv) {
  const double h = a.width[i];
  double b0, b1, b2, b3;
  // streaming_block_1d (transport_system.cpp:74-78): v>0: v(E_R - S), else v(-E_L - S)
  if (v > 0) {
    b0 = v * (1.0 / h);
    b1 = v * (kSqrt3 / h);
    b2 = v * (kSqrt3 / h - 2.0 * kSqrt3 / h);
    b3 = v * (3.0 / h);
  } else {
    b0 = v * (-(1.0 / h));
    b1 = v * (kSqrt3 / h);
    b2 = v * (kSqrt3 / h - 2.0 * kSqrt3 / h);
    b3 = v * (-(3.0 / h));
  }
  if (a.block == 4) {
    const double* m = a.mt + ((long)s * a.N + i) * 4;
    b0 += m[0];
    b1 += m[1];
    b2 += m[2];
    b3 += m[3];
  } else {
    const double sg = a.mt[(long)s * a.N + i];
    b0 += sg;
    b3 += sg;
  }
  const double id = 1.0 / (b0 * b3 - b2 * b1);
  binv[0] = b3 * id;
  binv[1] = -b1 * id;
  binv[2] = -b2 * id;
  binv[3] = b0 * id;
}

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

template <int CPL>
__global__ void __launch_bounds__(512) sweep1d_kernel(const Sweep1DArgs a) {
  extern __shared__ double sm[];
  const int s = blockIdx.x;
  if (a.active && !a.active[s]) return;
  const int N = a.N;
  const long nd = a.ndof;
  double* q = sm;
  double* acc = sm + nd;
  double* stage = sm + 2 * nd;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- source q (apply_Ms + G, or the raw rhs) ----
  for (long i = threadIdx.x; i < nd; i += blockDim.x) {
    double v = 0.0;
    const long si = (long)s * nd + i;
    if (a.mode & SRC_RAW) {
      v = a.rho[si];
    } else {
      if (a.mode & SRC_MS_RHO) {
        const long c = i >> 1;
        const int r = (int)(i & 1);
        if (a.block == 4) {
          const double* m = a.ms + ((long)s * N + c) * 4 + 2 * r;
          v = m[0] * a.rho[(long)s * nd + 2 * c] + m[1] * a.rho[(long)s * nd + 2 * c + 1];
        } else {
          v = a.ms[(long)s * N + c] * a.rho[si];
        }
      }
      if (a.mode & SRC_G) v += a.g[(a.g_shared ? 0 : (long)s * nd) + i];
    }
    q[i] = v;
    acc[i] = 0.0;
  }
  __syncthreads();

  const int jlo = a.j_single >= 0 ? a.j_single : 0;
  const int jn = a.j_single >= 0 ? 1 : a.nv;
  for (int r0 = 0; r0 < jn; r0 += nw) {
    const int jj = r0 + warp;
    if (jj < jn) {
      const int j = jlo + jj;
      const double v = a.vx[j];
      const double c = fabs(v);
      const bool fwd = v > 0;
      double u0 = 0.0;
      if (a.mode & SRC_BC) u0 = fwd ? a.inflow_l : a.inflow_r;
      // pass 1: compose the lane's affine maps u -> A + B u
      double A = 0.0, B = 1.0;
      for (int k = 0; k < CPL; ++k) {
        const int p = lane * CPL + k;
        if (p < N) {
          const int i = fwd ? p : N - 1 - p;
          double bi[4];
          cell_block(a, s, i, v, bi);
          const double sc = 1.0 / sqrt(a.width[i]);
          const double tin0 = sc, tin1 = fwd ? -kSqrt3 * sc : kSqrt3 * sc;
          const double tout0 = sc, tout1 = fwd ? kSqrt3 * sc : -kSqrt3 * sc;
          const double r0v = q[2 * i], r1v = q[2 * i + 1];
          const double y0 = bi[0] * r0v + bi[1] * r1v, y1 = bi[2] * r0v + bi[3] * r1v;
          const double z0 = bi[0] * tin0 + bi[1] * tin1, z1 = bi[2] * tin0 + bi[3] * tin1;
          const double al = tout0 * y0 + tout1 * y1;
          const double be = c * (tout0 * z0 + tout1 * z1);
          A = al + be * A;
          B = be * B;
        }
      }
      // inclusive warp scan of the affine maps
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double Ap = __shfl_up_sync(0xffffffffu, A, d);
        const double Bp = __shfl_up_sync(0xffffffffu, B, d);
        if (lane >= d) {
          A = A + B * Ap;
          B = B * Bp;
        }
      }
      const double Ae = __shfl_up_sync(0xffffffffu, A, 1);
      const double Be = __shfl_up_sync(0xffffffffu, B, 1);
      double u = lane == 0 ? u0 : Ae + Be * u0;
      // pass 2: cell solves with the exact incoming trace
      double* st = stage + (long)warp * nd;
      double* fo = nullptr;
      if (a.fout) fo = a.fout + (a.j_single >= 0 ? (long)s * nd : ((long)s * a.nv + j) * nd);
      for (int k = 0; k < CPL; ++k) {
        const int p = lane * CPL + k;
        if (p < N) {
          const int i = fwd ? p : N - 1 - p;
          double bi[4];
          cell_block(a, s, i, v, bi);
          const double sc = 1.0 / sqrt(a.width[i]);
          const double tin0 = sc, tin1 = fwd ? -kSqrt3 * sc : kSqrt3 * sc;
          const double tout0 = sc, tout1 = fwd ? kSqrt3 * sc : -kSqrt3 * sc;
          const double cu = c * u;
          const double r0v = q[2 * i] + cu * tin0, r1v = q[2 * i + 1] + cu * tin1;
          const double f0 = bi[0] * r0v + bi[1] * r1v, f1 = bi[2] * r0v + bi[3] * r1v;
          u = tout0 * f0 + tout1 * f1;
          st[2 * i] = f0;
          st[2 * i + 1] = f1;
          if (fo) {
            fo[2 * i] = f0;
            fo[2 * i + 1] = f1;
          }
        }
      }
    }
    __syncthreads();
    const int cnt = min(nw, jn - r0);
    for (long i = threadIdx.x; i < nd; i += blockDim.x) {
      double t = acc[i];
      for (int k = 0; k < cnt; ++k) {
        const double wj = a.j_single >= 0 ? 1.0 : a.w[r0 + k];
        t = t + wj * stage[(long)k * nd + i];
      }
      acc[i] = t;
    }
    __syncthreads();
  }

  if (a.out) {
    double mx_d = 0.0, mx_r = 0.0;
    for (long i = threadIdx.x; i < nd; i += blockDim.x) {
      const double o = acc[i];
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
  const long nd = a.ndof;
  const int jn = a.j_single >= 0 ? 1 : a.nv;
  int nw = 16;
  const long budget = 200 * 1024;
  while (nw > 1 && (long)(2 + nw) * nd * 8 > budget) nw >>= 1;
  nw = std::min(nw, std::max(1, jn));
  const size_t smem = (size_t)(2 + nw) * nd * 8;
  RTE_REQUIRE(smem <= (size_t)(227 * 1024), RTE_ERR_UNSUPPORTED, "sweep1d: slab too large for one CTA");
  static bool configured = false;
  if (!configured) {
    RTE_CUDA(cudaFuncSetAttribute(sweep1d_kernel<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    configured = true;
  }
  sweep1d_kernel<CPL><<<a.S, nw * 32, smem, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

}  // namespace

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
