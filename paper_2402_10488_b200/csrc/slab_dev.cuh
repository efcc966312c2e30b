// slab_dev.cuh -- device building blocks shared by the per-kernel slab path
// (sweep1d.cu, dsa1d.cu, rom.cu) and the fused slab SI kernel (si1d.cu):
// the slab cell block, the CTA-wide sweep of one sample, the block
// cyclic-reduction solve of one sample, and the reduced-model projection /
// complete-pivoting solve.  Everything here is per sample and CTA-wide, so the
// separate kernels and the fused loop run identical arithmetic.
#pragma once

#include "rte_internal.cuh"

namespace rte {
namespace slab {

#ifdef RTE_SWEEP_TRACE  // development: per-phase SM clocks of CTA 0 / thread 0 (build variant)
__device__ long long g_sweep_trace[8];
#define SW_T0() long long _tt = (blockIdx.x == 0 && threadIdx.x == 0) ? clock64() : 0
#define SW_T(k)                                                            \
  do {                                                                     \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                             \
      const long long _n = clock64();                                      \
      g_sweep_trace[k] += _n - _tt;                                        \
      _tt = _n;                                                            \
    }                                                                      \
  } while (0)
#else
#define SW_T0()
#define SW_T(k)
#endif

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

// Outflow-trace gain of a cell for the scan: beta = |v| t_out . B^-1 t_in.
__device__ __forceinline__ double trace_gain(const double* bi, double sc, double c, bool fwd) {
  const double tin0 = sc, tin1 = fwd ? -kSqrt3 * sc : kSqrt3 * sc;
  const double tout0 = sc, tout1 = fwd ? kSqrt3 * sc : -kSqrt3 * sc;
  const double z0 = bi[0] * tin0 + bi[1] * tin1, z1 = bi[2] * tin0 + bi[3] * tin1;
  return c * (tout0 * z0 + tout1 * z1);
}

// Cached cell data of sweep position p = lane * CPL + k (Sweep1DArgs::cache).
__device__ __forceinline__ double ld_na(const double* p) {  // read-only, not allocated in L1
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <int CPL>
__device__ __forceinline__ void load_cached_t(const double* cc, int k, int lane, double* bi, double& be) {
  const double* e = cc + k * 32 + lane;
  bi[0] = ld_na(e);
  bi[1] = ld_na(e + 32 * CPL);
  bi[2] = ld_na(e + 2 * 32 * CPL);
  bi[3] = ld_na(e + 3 * 32 * CPL);
  be = ld_na(e + 4 * 32 * CPL);
}
#define load_cached(cc, k, lane, bi, be) load_cached_t<CPL>(cc, k, lane, bi, be)

// Shared-memory layout of the slab sweep's per-sample vectors ("lane-major"):
// DOF e = 2 c + comp of cell c lives at comp * 32 CPL + (c % CPL) * 32 + c / CPL,
// so the 32 lanes of a warp, which own cells lane * CPL + k (forward) or their
// mirror images (backward), touch 32 consecutive doubles: no bank conflicts in
// the sweep's inner loops.  Vectors hold 2 * 32 * CPL doubles (>= n_dof).
template <int CPL>
__device__ __forceinline__ int lane_major(int c, int comp) {
  return comp * (32 * CPL) + (c % CPL) * 32 + c / CPL;
}
template <int CPL>
__device__ __forceinline__ int lane_major_dof(long e) {
  return lane_major<CPL>((int)(e >> 1), (int)(e & 1));
}

// Source assembly and the direction sweeps of one sample by the whole CTA
// (blockDim.x / 32 warps): q = source moments, acc = sum_j w_j f_j in the
// fixed order j = 0..n-1, both in the lane-major layout (stage: nw such
// vectors).  rho_s is the sample's rho: natural layout in global memory, or
// lane-major in shared memory (rho_lane_major).  Ends with a __syncthreads.
// Shared by sweep1d_kernel and the fused slab SI kernel (si1d.cu).
template <int CPL, bool CACHED>
__device__ __forceinline__ void sweep_cta(const Sweep1DArgs& a, int s, const double* rho_s, bool rho_lane_major,
                                          double* q, double* acc, double* stage) {
  constexpr int NP = 32 * CPL;
  const int N = a.N;
  const long nd = a.ndof;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SW_T0();
  // ---- source q (apply_Ms + G, or the raw rhs) ----
  for (long e = threadIdx.x; e < nd; e += blockDim.x) {
    const long c = e >> 1;
    const int r = (int)(e & 1);
    const int le = lane_major<CPL>((int)c, r);
    double v = 0.0;
    if (a.mode & SRC_RAW) {
      v = rho_lane_major ? rho_s[le] : rho_s[e];
    } else {
      if (a.mode & SRC_MS_RHO) {
        const double x0 = rho_lane_major ? rho_s[lane_major<CPL>((int)c, 0)] : rho_s[2 * c];
        const double x1 = rho_lane_major ? rho_s[lane_major<CPL>((int)c, 1)] : rho_s[2 * c + 1];
        if (a.block == 4) {
          const double* m = a.ms + ((long)s * N + c) * 4 + 2 * r;
          v = m[0] * x0 + m[1] * x1;
        } else {
          v = a.ms[(long)s * N + c] * (r ? x1 : x0);
        }
      }
      if (a.mode & SRC_G) v += a.g[(a.g_shared ? 0 : (long)s * nd) + e];
    }
    q[le] = v;
    acc[le] = 0.0;
  }
  __syncthreads();
  SW_T(0);

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
      const double* cc = CACHED ? a.cache + ((long)s * a.nv + j) * 5 * NP : nullptr;
      // pass 1: compose the lane's affine maps u -> A + B u (cell data of a
      // block of KB cells loaded up front, off the dependency chain)
      constexpr int KB = CPL < 8 ? CPL : 8;
      double A = 0.0, B = 1.0;
      for (int k0 = 0; k0 < CPL; k0 += KB) {
        double bi[KB][4], sc[KB], be[KB];
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const int p = lane * CPL + k0 + kk;
          if (p < N) {
            const int i = fwd ? p : N - 1 - p;
            if (CACHED) {
              load_cached(cc, k0 + kk, lane, bi[kk], be[kk]);
              sc[kk] = a.cache_sc[i];
            } else {
              cell_block(a, s, i, v, bi[kk]);
              sc[kk] = 1.0 / sqrt(a.width[i]);
              be[kk] = trace_gain(bi[kk], sc[kk], c, fwd);
            }
          }
        }
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const int p = lane * CPL + k0 + kk;
          if (p < N) {
            const int i = fwd ? p : N - 1 - p;
            const int li = lane_major<CPL>(i, 0);
            const double tout0 = sc[kk], tout1 = fwd ? kSqrt3 * sc[kk] : -kSqrt3 * sc[kk];
            const double r0v = q[li], r1v = q[li + NP];
            const double y0 = bi[kk][0] * r0v + bi[kk][1] * r1v, y1 = bi[kk][2] * r0v + bi[kk][3] * r1v;
            const double al = tout0 * y0 + tout1 * y1;
            A = al + be[kk] * A;
            B = be[kk] * B;
          }
        }
      }
      SW_T(1);
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
      SW_T(2);
      // pass 2: cell solves with the exact incoming trace
      double* st = stage + (long)warp * 2 * NP;
      double* fo = nullptr;
      if (a.fout) fo = a.fout + (a.j_single >= 0 ? (long)s * nd : ((long)s * a.nv + j) * nd);
      for (int k0 = 0; k0 < CPL; k0 += KB) {
        double bi[KB][4], sc[KB];
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const int p = lane * CPL + k0 + kk;
          if (p < N) {
            const int i = fwd ? p : N - 1 - p;
            if (CACHED) {
              double be;
              load_cached(cc, k0 + kk, lane, bi[kk], be);
              sc[kk] = a.cache_sc[i];
            } else {
              cell_block(a, s, i, v, bi[kk]);
              sc[kk] = 1.0 / sqrt(a.width[i]);
            }
          }
        }
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const int p = lane * CPL + k0 + kk;
          if (p < N) {
            const int i = fwd ? p : N - 1 - p;
            const int li = lane_major<CPL>(i, 0);
            const double tin0 = sc[kk], tin1 = fwd ? -kSqrt3 * sc[kk] : kSqrt3 * sc[kk];
            const double tout0 = sc[kk], tout1 = fwd ? kSqrt3 * sc[kk] : -kSqrt3 * sc[kk];
            const double cu = c * u;
            const double r0v = q[li] + cu * tin0, r1v = q[li + NP] + cu * tin1;
            const double f0 = bi[kk][0] * r0v + bi[kk][1] * r1v, f1 = bi[kk][2] * r0v + bi[kk][3] * r1v;
            u = tout0 * f0 + tout1 * f1;
            st[li] = f0;
            st[li + NP] = f1;
            if (fo) {
              fo[2 * i] = f0;
              fo[2 * i + 1] = f1;
            }
          }
        }
      }
    }
    SW_T(3);
    __syncthreads();
    SW_T(4);
    // fixed-order accumulation over the round's directions (lane-major index t
    // belongs to cell (t % 32) * CPL + (t % NP) / 32)
    const int cnt = min(nw, jn - r0);
    for (int t = threadIdx.x; t < 2 * NP; t += blockDim.x) {
      const int tt = t % NP;
      if ((tt & 31) * CPL + (tt >> 5) >= N) continue;
      double x = acc[t];
      for (int k = 0; k < cnt; ++k) {
        const double wj = a.j_single >= 0 ? 1.0 : a.w[r0 + k];
        x = x + wj * stage[(long)k * 2 * NP + t];
      }
      acc[t] = x;
    }
    __syncthreads();
    SW_T(5);
  }
}

constexpr int kCrThreads = 256;

// level sizes of the reduction: n_0 = N, n_{l+1} = ceil(n_l / 2) until 1
__host__ __device__ inline int cr_levels(int N) {
  int l = 0;
  for (int n = N; n > 1; n = (n + 1) / 2) ++l;
  return l;
}
__host__ __device__ inline long cr_entries(int N) {  // sum of n_l over all levels incl. the last (1)
  long t = 0;
  int n = N;
  for (;;) {
    t += n;
    if (n == 1) break;
    n = (n + 1) / 2;
  }
  return t;
}

__device__ inline void mv4(const double* m, const double* x, double* y) {
  for (int r = 0; r < 4; ++r) y[r] = m[4 * r] * x[0] + m[4 * r + 1] * x[1] + m[4 * r + 2] * x[2] + m[4 * r + 3] * x[3];
}

// Block cyclic reduction solve of one sample by the whole CTA: y [N][4]
// holds the right-hand side on entry and the solution on exit; fac is the
// sample's factor table (dsa1d_factor_cr).  Starts after and ends with a
// __syncthreads.
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Issues L1 prefetches of the factor entries (lines of 128 B) this thread
// reads at a level: forward levels read (A, C) of even positions (2 lines),
// backward levels (D^-1, L, U) of odd positions (3 lines).
__device__ __forceinline__ void cr_prefetch(const double* f, int n, bool fwd) {
  for (int p = (fwd ? 0 : 1) + 2 * threadIdx.x; p < n; p += 2 * blockDim.x) {
    const char* e = reinterpret_cast<const char*>(f + (long)p * 48);
    prefetch_l1(e);
    prefetch_l1(e + 128);
    if (!fwd) prefetch_l1(e + 256);
  }
}

__device__ __forceinline__ void cr_solve_cta(int N, const double* fac, double* y) {
  // level sizes and offsets of the reduction
  int ns[32];
  long offs[32];
  int L = 0;
  {
    long o = 0;
    for (int n = N; n > 1; n = (n + 1) / 2) {
      ns[L] = n;
      offs[L++] = o;
      o += n;
    }
    offs[L] = o;  // the last level's single entry
  }
  // forward: at level l (stride st) kept equation p (index p*st) absorbs its odd neighbours
  if (L > 0) cr_prefetch(fac, ns[0], true);
  for (int l = 0, st = 1; l < L; ++l, st *= 2) {
    const int n = ns[l];
    if (l + 1 < L) cr_prefetch(fac + offs[l + 1] * 48, ns[l + 1], true);
    const double* f = fac + offs[l] * 48;
    for (int p = 2 * threadIdx.x; p < n; p += 2 * blockDim.x) {
      const double* e = f + (long)p * 48;
      double v[4], t[4];
      for (int k = 0; k < 4; ++k) v[k] = y[4L * p * st + k];
      if (p >= 1) {
        mv4(e, y + 4L * (p - 1) * st, t);
        for (int k = 0; k < 4; ++k) v[k] -= t[k];
      }
      if (p + 1 < n) {
        mv4(e + 16, y + 4L * (p + 1) * st, t);
        for (int k = 0; k < 4; ++k) v[k] -= t[k];
      }
      for (int k = 0; k < 4; ++k) y[4L * p * st + k] = v[k];
    }
    __syncthreads();
  }
  if (L > 0) cr_prefetch(fac + offs[L - 1] * 48, ns[L - 1], false);
  if (threadIdx.x == 0) {
    double t[4];
    mv4(fac + offs[L] * 48, y, t);
    for (int k = 0; k < 4; ++k) y[k] = t[k];
  }
  __syncthreads();
  // backward: odd equations of each level from the top, x = D^{-1} (y - L x_{p-1} - U x_{p+1})
  for (int l = L - 1; l >= 0; --l) {
    const int n = ns[l];
    const int stl = 1 << l;
    if (l > 0) cr_prefetch(fac + offs[l - 1] * 48, ns[l - 1], false);
    const double* f = fac + offs[l] * 48;
    for (int p = 1 + 2 * threadIdx.x; p < n; p += 2 * blockDim.x) {
      const double* e = f + (long)p * 48;
      double v[4], t[4];
      for (int k = 0; k < 4; ++k) v[k] = y[4L * p * stl + k];
      mv4(e + 16, y + 4L * (p - 1) * stl, t);
      for (int k = 0; k < 4; ++k) v[k] -= t[k];
      if (p + 1 < n) {
        mv4(e + 32, y + 4L * (p + 1) * stl, t);
        for (int k = 0; k < 4; ++k) v[k] -= t[k];
      }
      mv4(e, v, t);
      for (int k = 0; k < 4; ++k) y[4L * p * stl + k] = t[k];
    }
    __syncthreads();
  }
}

// Compact factor layout of the cyclic reduction for the fused SI kernel
// (dsa1d.cu repacks the factor table into it): per level l with n_l
// equations, ne = ceil(n_l / 2) kept (even) and no = floor(n_l / 2)
// eliminated (odd) ones, first the forward data A, C (32 components) of the
// kept equations, component-major [32][ne], then the backward data D^-1, L, U
// (48 components) of the eliminated ones, [48][no]; after the last level the
// final D^-1 (16 doubles).  Component-major so that consecutive threads read
// consecutive doubles (no shared-memory bank conflicts, coalesced in global
// memory).  163 KB per sample at N = 256: it can live in shared memory for a
// whole solve.
__host__ __device__ inline long crc_level_size(int n) { return (long)((n + 1) / 2) * 32 + (long)(n / 2) * 48; }
__host__ __device__ inline long crc_doubles(int N) {
  long t = 16;
  for (int n = N; n > 1; n = (n + 1) / 2) t += crc_level_size(n);
  return t;
}

// y = m x for a 4x4 block stored with component stride ms and a 4-vector
// with component stride xs (same accumulation order as mv4).
__device__ __forceinline__ void mv4s(const double* m, int ms, const double* x, int xs, double* y) {
  for (int r = 0; r < 4; ++r)
    y[r] = m[(4 * r) * ms] * x[0] + m[(4 * r + 1) * ms] * x[xs] + m[(4 * r + 2) * ms] * x[2 * xs] +
           m[(4 * r + 3) * ms] * x[3 * xs];
}

// Block cyclic reduction on the compact layout with per-level reduced
// systems: Y holds, level after level, the right-hand sides of the n_l
// equations of level l component-major [4][n_l] (8 N doubles in all); on
// entry Y[0..4N) is level 0's right-hand side [4][N], on exit the solution.
// Same formulas and accumulation order as cr_solve_cta.  Starts after and
// ends with a __syncthreads.
__device__ __forceinline__ void cr_solve_compact(int N, const double* fc, double* Y) {
  int ns[24];
  int offs[25], yo[25];
  int L = 0;
  {
    int o = 0, q = 0;
    for (int n = N; n > 1; n = (n + 1) / 2) {
      ns[L] = n;
      offs[L] = o;
      yo[L++] = q;
      o += (int)crc_level_size(n);
      q += 4 * n;
    }
    offs[L] = o;
    yo[L] = q;
    ns[L] = 1;
  }
  // forward: kept equation m = p / 2 of level l becomes equation m of level l+1
  for (int l = 0; l < L; ++l) {
    const int n = ns[l], ne = (n + 1) / 2;
    const double* f = fc + offs[l];
    const double* y = Y + yo[l];
    double* yn = Y + yo[l + 1];
    for (int m = threadIdx.x; m < ne; m += blockDim.x) {
      const int p = 2 * m;
      double v[4], t[4];
      for (int k = 0; k < 4; ++k) v[k] = y[k * n + p];
      if (p >= 1) {
        mv4s(f + m, ne, y + p - 1, n, t);
        for (int k = 0; k < 4; ++k) v[k] -= t[k];
      }
      if (p + 1 < n) {
        mv4s(f + 16 * ne + m, ne, y + p + 1, n, t);
        for (int k = 0; k < 4; ++k) v[k] -= t[k];
      }
      for (int k = 0; k < 4; ++k) yn[k * ne + m] = v[k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double t[4];
    double* y = Y + yo[L];
    mv4s(fc + offs[L], 1, y, 1, t);
    for (int k = 0; k < 4; ++k) y[k] = t[k];
  }
  __syncthreads();
  // backward: level l's kept equations take level l+1's solution, the
  // eliminated ones x = D^-1 (y - L x_{p-1} - U x_{p+1})
  for (int l = L - 1; l >= 0; --l) {
    const int n = ns[l], ne = (n + 1) / 2, no = n / 2;
    const double* f = fc + offs[l] + (long)ne * 32;
    double* y = Y + yo[l];
    const double* xn = Y + yo[l + 1];
    for (int m = threadIdx.x; m < ne; m += blockDim.x)
      for (int k = 0; k < 4; ++k) y[k * n + 2 * m] = xn[k * ne + m];
    __syncthreads();
    for (int m = threadIdx.x; m < no; m += blockDim.x) {
      const int p = 2 * m + 1;
      double v[4], t[4];
      for (int k = 0; k < 4; ++k) v[k] = y[k * n + p];
      mv4s(f + 16 * no + m, no, y + p - 1, n, t);
      for (int k = 0; k < 4; ++k) v[k] -= t[k];
      if (p + 1 < n) {
        mv4s(f + 32 * no + m, no, y + p + 1, n, t);
        for (int k = 0; k < 4; ++k) v[k] -= t[k];
      }
      mv4s(f + m, no, v, 1, t);
      for (int k = 0; k < 4; ++k) y[k * n + p] = t[k];
    }
    __syncthreads();
  }
}

__device__ inline void fullpiv_solve(const double* a, int r, const int* rp, const int* cp, const double* b, double* y,
                              double* x) {
  for (int i = 0; i < r; ++i) {
    double t = b[rp[i]];
    for (int k = 0; k < i; ++k) t -= a[i * r + k] * y[k];
    y[i] = t;
  }
  for (int i = r - 1; i >= 0; --i) {
    double t = y[i];
    for (int k = i + 1; k < r; ++k) t -= a[i * r + k] * y[k];
    y[i] = t / a[i * r + i];
  }
  for (int i = 0; i < r; ++i) x[cp[i]] = y[i];
}

// Complete-pivoting LU (FullPivLU semantics, rom.cu fullpiv_lu) of the
// r x r row-major matrix a in shared memory by one warp, r <= 32, lane i owns
// row i: the same pivot choices (first maximum in column-major order) and the
// same per-element arithmetic as the serial version, so the factors are
// bitwise equal.  Returns the rank (|pivot| > eps r max|pivot|) on all lanes.
__device__ __forceinline__ int warp_fullpiv_lu(double* a, int r, int* rp, int* cp) {
  const int ln = threadIdx.x & 31;
  if (ln < r) {
    rp[ln] = ln;
    cp[ln] = ln;
  }
  __syncwarp();
  double maxpiv = 0.0;
  int nz = r;
  for (int k = 0; k < r; ++k) {
    // this lane's row: first maximum over columns k..r-1
    double big = 0.0;
    int bj = k;
    if (ln >= k && ln < r)
      for (int j = k; j < r; ++j) {
        const double v = fabs(a[ln * r + j]);
        if (v > big) {
          big = v;
          bj = j;
        }
      }
    int bi = ln;
    // warp arg-max: larger value, then smaller column, then smaller row
    for (int o = 16; o > 0; o >>= 1) {
      const double b2 = __shfl_xor_sync(0xffffffffu, big, o);
      const int j2 = __shfl_xor_sync(0xffffffffu, bj, o), i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (b2 > big || (b2 == big && (j2 < bj || (j2 == bj && i2 < bi)))) {
        big = b2;
        bj = j2;
        bi = i2;
      }
    }
    if (big == 0.0) {
      nz = k;
      break;
    }
    maxpiv = fmax(maxpiv, big);
    if (bi != k) {  // row swap (lane = column)
      if (ln < r) {
        const double t = a[k * r + ln];
        a[k * r + ln] = a[bi * r + ln];
        a[bi * r + ln] = t;
      }
      if (ln == 0) {
        const int t = rp[k];
        rp[k] = rp[bi];
        rp[bi] = t;
      }
    }
    __syncwarp();
    if (bj != k) {  // column swap (lane = row)
      if (ln < r) {
        const double t = a[ln * r + k];
        a[ln * r + k] = a[ln * r + bj];
        a[ln * r + bj] = t;
      }
      if (ln == 0) {
        const int t = cp[k];
        cp[k] = cp[bj];
        cp[bj] = t;
      }
    }
    __syncwarp();
    const double piv = a[k * r + k];
    if (ln > k && ln < r) {
      const double l = a[ln * r + k] / piv;
      a[ln * r + k] = l;
      for (int j = k + 1; j < r; ++j) a[ln * r + j] -= l * a[k * r + j];
    }
    __syncwarp();
  }
  const double thr = 2.220446049250313e-16 * r * maxpiv;
  const bool ok = ln < nz && fabs(a[ln * r + ln]) > thr;
  return __popc(__ballot_sync(0xffffffffu, ok));
}

// fullpiv_solve by one warp (r <= 32; lane j owns row / unknown j), LU in
// shared memory: forward substitution subtracts in the same (ascending)
// order as the serial version, backward in descending order.
__device__ __forceinline__ void warp_fullpiv_solve(const double* a, int r, const int* rp, const int* cp,
                                                   const double* b, double* x) {
  const int j = threadIdx.x & 31;
  double t = j < r ? b[rp[j]] : 0.0;
  for (int i = 0; i < r; ++i) {  // L y = P b (unit lower)
    const double yi = __shfl_sync(0xffffffffu, t, i);
    if (j > i && j < r) t -= a[j * r + i] * yi;
  }
  for (int i = r - 1; i >= 0; --i) {  // U z = y
    if (j == i) t = t / a[i * r + i];
    const double zi = __shfl_sync(0xffffffffu, t, i);
    if (j < i) t -= a[j * r + i] * zi;
  }
  if (j < r) x[cp[j]] = t;
}

template <int CH>
__device__ inline void block_dots(const double* u, long nd, int r, const double* v_smem_or_null, const double* ms,
                           int block, int N, const double* d, int s, double* out_smem, double* red) {
  // out[k] = sum_i u[k*nd + i] * (Ms delta)_i, fixed-order reduction
  for (int k0 = 0; k0 < r; k0 += CH) {
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = 0.0;
    for (long i = threadIdx.x; i < nd; i += blockDim.x) {
      double m;
      const int nl = (int)(nd / N);
      if (block == nl * nl) {  // full per-cell block (1D block 4, XY block 16)
        const long c = i / nl;
        const int rr = (int)(i - c * nl);
        const double* mm = ms + ((long)s * N + c) * block + nl * rr;
        m = 0.0;
        for (int q = 0; q < nl; ++q) m = fma(mm[q], d[nl * c + q], m);
      } else {
        m = ms[(long)s * N + i / nl] * d[i];
      }
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (k0 + c < r) acc[c] = fma(u[(long)(k0 + c) * nd + i], m, acc[c]);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double v = acc[c];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) red[(threadIdx.x >> 5) * CH + c] = v;
    }
    __syncthreads();
    if (threadIdx.x < CH && k0 + (int)threadIdx.x < r) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w * CH + threadIdx.x];
      out_smem[k0 + threadIdx.x] = t;
    }
    __syncthreads();
  }
}


}  // namespace slab
}  // namespace rte
