// si1d.cu -- fused slab source iteration: the whole sisa_solve loop
// (sisa.cpp:14-54) of one parameter sample in one CTA, all samples of the
// batch in one launch.
//
// Per iteration the CTA runs, with no kernel boundary and no host round trip:
//   rho* = L rho + bbar     the source assembly and direction sweeps
//                           (slab::sweep_cta, transport_system.cpp:279-310,
//                           393-418; fixed-order w_j f_j sum)
//   delta = rho* - rho, ||delta||_inf, ||rho*||_inf   (block max reduction)
//   the stop test / strategy choice (si_decide semantics: sisa.cpp:123-127,
//                           strategies.cpp:55-76 monotone ROMSAD switch)
//   the correction          DSA: block cyclic reduction of [Ms delta; 0]
//                           (slab::cr_solve_compact, dsa.cpp:264-277), the
//                           sample's factors held in shared memory when they
//                           fit; ROMSA: U_rho A_r^{-1} U_iso^T Ms delta
//                           (strategies.cpp:37-53), warp-parallel solve
//   rho = rho* + correction
// rho, rho*, delta (lane-major layout, slab_dev.cuh) and the cyclic-reduction
// levels live in shared memory; the
// per-sample report state (iterations, history, log, switch iteration,
// convergence) is written to the same SiState arrays the per-kernel loop
// fills, so rte_si_solve's reporting is shared.  Samples finish
// independently (a converged sample's CTA exits).  The per-kernel loop
// (capi.cu) remains for slabs too large for one CTA's shared memory and for
// caller strategies (RTE_CUSTOM).
#include "rte_internal.cuh"
#include "slab_dev.cuh"

namespace rte {
using namespace slab;

namespace {

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
  return m;
}

template <int CPL, bool CACHED, bool FAC_SMEM>
__global__ void __launch_bounds__(256) si1d_kernel(const Si1DArgs a) {
  extern __shared__ double sm[];
  __shared__ double red[32], rom_rhs[32], rom_c[32], rom_red[32 * 8];
  __shared__ int kind_sh, done_sh;
  constexpr int NP = 32 * CPL, NV = 2 * NP;  // lane-major vectors (slab_dev.cuh)
  const int s = blockIdx.x;
  const int N = a.sw.N;
  const long nd = a.sw.ndof;
  const int nw = blockDim.x >> 5;
  double* q = sm;                 // source moments, then delta (lane-major)
  double* acc = q + NV;           // rho* (lane-major)
  double* stage = acc + NV;       // [nw][NV] direction fluxes of one round
  double* rho = stage + nw * NV;  // current iterate (lane-major)
  double* y = rho + NV;           // cyclic-reduction levels (8 N doubles) / natural-layout delta for ROMSA
  double* fsm = y + 4 * NV;       // FAC_SMEM: the sample's compact CR factors for the whole solve
  const SiState& st = a.st;
  const rte_si_config& cfg = a.cfg;
  if (!st.active[s]) return;
  const double* fac = a.fac ? a.fac + (long)s * crc_doubles(N) : nullptr;
  if (FAC_SMEM && fac) {
    const long nf = crc_doubles(N);
    for (long t = threadIdx.x; t < nf; t += blockDim.x) fsm[t] = __ldg(fac + t);
    fac = fsm;
  }
  for (long e = threadIdx.x; e < nd; e += blockDim.x) rho[lane_major_dof<CPL>(e)] = a.rho[(long)s * nd + e];
  __syncthreads();
  const int limit = cfg.fixed_iters > 0 ? cfg.fixed_iters : cfg.max_iters;
  const bool clk = a.phase_clk && s == 0 && threadIdx.x == 0;
  long long c0 = clk ? clock64() : 0, c1 = 0, c2 = 0;
  for (int l = 1;; ++l) {
    const long long ci = clk ? clock64() : 0;
    sweep_cta<CPL, CACHED>(a.sw, s, rho, true, q, acc, stage);
    if (clk) c1 += clock64() - ci;
    // SI epilogue: delta = rho* - rho and the two inf-norms
    double mx_d = 0.0, mx_r = 0.0;
    for (int t = threadIdx.x; t < NV; t += blockDim.x) {
      const int tt = t % NP;
      if ((tt & 31) * CPL + (tt >> 5) >= N) continue;
      const double o = acc[t];
      const double dd = o - rho[t];
      q[t] = dd;
      mx_d = fmax(mx_d, fabs(dd));
      mx_r = fmax(mx_r, fabs(o));
      if (dd != dd) mx_d = dd;  // propagate NaN
    }
    const double ch = fabs(block_max(mx_d, red));
    const double rm = block_max(mx_r, red);
    // stop test and strategy choice for this sample (si_decide_kernel)
    if (threadIdx.x == 0) {
      double chn = ch;
      if (cfg.norm == RTE_NORM_REL && rm > 0) chn = ch / rm;
      st.history[(long)s * cfg.max_iters + l - 1] = chn;
      st.iters[s] = l;
      st.last_change[s] = chn;
      int kind = KIND_ACCEPT, done = 0;
      char lg = 0;
      if (cfg.fixed_iters <= 0 && chn < cfg.eps) {  // sisa.cpp:123-127
        st.converged[s] = 1;
        st.active[s] = 0;
        done = 1;
      } else {
        switch (cfg.method) {
          case RTE_DSA:
          case RTE_ROMIG:
            kind = KIND_DSA;
            lg = 'D';
            break;
          case RTE_ROMSA:
            kind = st.singular[s] ? KIND_SINGULAR : KIND_ROMSA;
            lg = st.singular[s] ? 'S' : 'R';
            break;
          case RTE_ROMSAD:  // strategies.cpp:67-76 (monotone switch)
            if (!st.switched[s] && l <= cfg.theta && ch >= cfg.eps_romsad) {
              kind = KIND_ROMSA;
              lg = 'R';
            } else {
              st.switched[s] = 1;
              kind = KIND_DSA;
              lg = 'D';
            }
            break;
          default:  // RTE_SI
            break;
        }
        if (kind == KIND_DSA && st.switch_iter[s] < 0) st.switch_iter[s] = l;
        if (lg) st.log[(long)s * cfg.max_iters + l - 1] = lg;
        if (l >= limit) {
          st.active[s] = 0;
          done = 1;
        }
      }
      st.kind[s] = kind;
      kind_sh = kind;
      done_sh = done;
    }
    __syncthreads();
    const long long cd = clk ? clock64() : 0;
    const int kind = kind_sh;
    if (kind == KIND_DSA) {
      // rhs [Ms delta; 0] per cell (dsa1d_solve_cr with apply_ms)
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int li = lane_major<CPL>(i, 0);
        double r0 = q[li], r1 = q[li + NP];
        if (a.sw.block == 4) {
          const double* m = a.sw.ms + ((long)s * N + i) * 4;
          const double t0 = m[0] * r0 + m[1] * r1, t1 = m[2] * r0 + m[3] * r1;
          r0 = t0;
          r1 = t1;
        } else {
          const double sg = a.sw.ms[(long)s * N + i];
          r0 *= sg;
          r1 *= sg;
        }
        y[i] = r0;  // level-0 right-hand side, component-major [4][N]
        y[N + i] = r1;
        y[2 * N + i] = 0.0;
        y[3 * N + i] = 0.0;
      }
      __syncthreads();
      cr_solve_compact(N, fac, y);
      for (long e = threadIdx.x; e < nd; e += blockDim.x) {
        const int le = lane_major_dof<CPL>(e);
        rho[le] = acc[le] + y[(e & 1) * N + (e >> 1)];
      }
    } else if (kind == KIND_ROMSA) {
      // natural-layout delta and the sample's LU factors (r <= 32) in the CR region
      double* lu = y + nd;
      for (long e = threadIdx.x; e < nd; e += blockDim.x) y[e] = q[lane_major_dof<CPL>(e)];
      for (int e = threadIdx.x; e < a.r * a.r; e += blockDim.x) lu[e] = __ldg(a.lu + (long)s * a.r * a.r + e);
      __syncthreads();
      block_dots<8>(a.u_iso, nd, a.r, nullptr, a.sw.ms, a.sw.block, N, y, s, rom_rhs, rom_red);
      if (threadIdx.x < 32) warp_fullpiv_solve(lu, a.r, a.rp + (long)s * a.r, a.cp + (long)s * a.r, rom_rhs, rom_c);
      __syncthreads();
      for (long e = threadIdx.x; e < nd; e += blockDim.x) {
        double t = 0.0;
        for (int k = 0; k < a.r; ++k) t = fma(a.u_rho[(long)k * nd + e], rom_c[k], t);
        const int le = lane_major_dof<CPL>(e);
        rho[le] = acc[le] + t;
      }
    } else {  // accepted (converged / plain SI) or singular ROMSA ('S': zero correction)
      for (int t = threadIdx.x; t < NV; t += blockDim.x) rho[t] = acc[t];
    }
    __syncthreads();
    if (clk) c2 += clock64() - cd;
    if (done_sh) break;
  }
  if (clk) {
    const long long tot = clock64() - c0;
    a.phase_clk[0] = c1;
    a.phase_clk[2] = c2;
    a.phase_clk[1] = tot - c1 - c2;
    a.phase_clk[3] = tot;
  }
  for (long e = threadIdx.x; e < nd; e += blockDim.x) a.rho[(long)s * nd + e] = rho[lane_major_dof<CPL>(e)];
}

template <int CPL, bool CACHED, bool FAC_SMEM>
void launch_one(const Si1DArgs& a, int nw, size_t smem, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    RTE_CUDA(cudaFuncSetAttribute(si1d_kernel<CPL, CACHED, FAC_SMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    configured = true;
  }
  si1d_kernel<CPL, CACHED, FAC_SMEM><<<a.sw.S, nw * 32, smem, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

template <int CPL>
bool launch_cpl(const Si1DArgs& a, cudaStream_t st) {
  const long nv = 2 * 32 * CPL;  // lane-major vector length
  const long budget = 220 * 1024;  // dynamic; + static (ROM scratch)
  if ((long)a.r * a.r > 3 * nv) return false;  // the ROMSA LU copy shares the CR region with delta
  int nw = 8;  // 256 threads: at 512 ptxas caps the kernel at 64 registers and spills
  while (nw > 1 && (long)(7 + nw) * nv * 8 > budget) nw >>= 1;
  nw = std::min(nw, std::max(1, a.sw.nv));
  if ((long)(7 + nw) * nv * 8 > budget) return false;
  // the DSA factors stay in shared memory for the whole solve when they fit
  // next to at least 4 direction warps (fewer warps, more sweep rounds)
  const size_t fbytes = a.fac ? (size_t)crc_doubles(a.sw.N) * 8 : 0;
  bool fac_smem = false;
  if (a.fac)
    for (int w = nw; w >= std::min(nw, 4) && !fac_smem; --w)
      if ((long)((7 + w) * nv * 8 + fbytes) <= budget) {
        nw = w;
        fac_smem = true;
      }
  const size_t smem = (size_t)(7 + nw) * nv * 8 + (fac_smem ? fbytes : 0);
  const bool cached = a.sw.cache != nullptr;
  if (fac_smem) {
    if (cached)
      launch_one<CPL, true, true>(a, nw, smem, st);
    else
      launch_one<CPL, false, true>(a, nw, smem, st);
  } else {
    if (cached)
      launch_one<CPL, true, false>(a, nw, smem, st);
    else
      launch_one<CPL, false, false>(a, nw, smem, st);
  }
  return true;
}

}  // namespace

// Runs the whole SI loop if the slab fits one CTA's shared memory; false:
// the caller uses the per-kernel loop.
bool si1d_fused(const Si1DArgs& a, cudaStream_t st) {
  const int N = a.sw.N;
  if (a.r > 32) return false;  // warp_fullpiv_solve; LU in the CR region
  if (N <= 32) return launch_cpl<1>(a, st);
  if (N <= 64) return launch_cpl<2>(a, st);
  if (N <= 128) return launch_cpl<4>(a, st);
  if (N <= 256) return launch_cpl<8>(a, st);
  if (N <= 512) return launch_cpl<16>(a, st);
  if (N <= 1024) return launch_cpl<32>(a, st);
  if (N <= 2048) return launch_cpl<64>(a, st);
  return false;
}

}  // namespace rte

#ifdef RTE_SWEEP_TRACE
extern "C" int rte_dev_sweep_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, rte::slab::g_sweep_trace, sizeof(long long) * 8) == cudaSuccess ? 0 : 1;
}
#endif
