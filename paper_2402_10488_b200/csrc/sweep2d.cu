// sweep2d.cu -- K2: batched 2D upwind-DG transport sweep (KBA-style band
// wavefront) with the source assembly and quadrature-weighted scalar-flux
// reduction fused in.
//
// Replaces TransportSystem::sweep_into 2D branch (transport_system.cpp:
// 312-363) with its per-slot cached inverses (build_sweep_cache, :189-261)
// and the direction loops of apply_L / assemble_rhs (:393-418).
//
// Decomposition.  Directions are folded to unique (vx, vy) slots (the +/-vz
// pairs of the product quadrature share one transport equation; weights are
// summed) and grouped by quadrant.  A work item is (band of 32 rows, sample,
// quadrant, direction group).  Inside an item each warp owns D directions and
// each lane one row; the warp marches the band along x as a diagonal
// wavefront: at step k lane t solves cell (x = k - t, row t) for its D
// directions, receives the incoming y-face traces of lane t-1 by warp
// shuffle and keeps its x-face traces in registers.  The D directions of a
// lane are independent chains (ILP) and share one load of (rho, sigma, G)
// per cell.  The NW warps of a CTA cover NW*D directions of the same
// quadrant; their w-weighted partial fluxes are reduced through shared memory
// in a fixed order and written once per item, so the scalar flux of a sweep
// is deterministic.  Band b+1 consumes band b's top traces through a global
// buffer guarded by per-item progress counters; items are taken from an
// atomic ticket in dependency order, so every producer an item waits on is
// already resident (no deadlock).
//
// Per-cell solve.  Per-cell coefficients are constant, so the cell block is
// B = sigma I + I (x) (a K) + (b K) (x) I with K = [[1, s3], [-s3, 3]] in the
// quadrant-reflected basis (a = |vx|/hx, b = |vy|/hy).  All blocks are
// polynomials in K, so B^{-1} has the closed form used in solve_cell() (one
// reciprocal, ~66 FP64 instructions per cell-direction).  It replaces the
// 16-double cached inverse per slot and cell of the reference.
#include "rte_internal.cuh"

namespace rte {
namespace {

constexpr int kNW = 8;  // warps per CTA
constexpr int kC = 8;   // steps per synchronisation chunk

struct DirConst {
  double a, b, w, e1, e2, tb, be, bcx, bcy, pad;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Canonical cell solve.  In: q (reflected source moments), X (incoming x-face
// traces per y-mode, pre-scaled by a), Y (incoming y-face traces per x-mode,
// pre-scaled by b).  Out: f and the outgoing traces.
__device__ __forceinline__ void solve_cell(const DirConst& dc, double sig, const double q[4], double X0,
                                           double X1, double Y0, double Y1, double f[4], double& Xo0,
                                           double& Xo1, double& Yo0, double& Yo1) {
  const double s3 = kSqrt3;
  const double r00 = q[0] + X0 + Y0;
  const double r01 = fma(-s3, X0, q[1] + Y1);
  const double r10 = fma(-s3, Y0, q[2] + X1);
  const double r11 = fma(-s3, X1, fma(-s3, Y1, q[3]));
  const double p = sig + dc.b;
  const double tt = p + dc.tb;
  const double del = fma(p, tt, dc.e1);
  const double al = fma(2.0 * dc.a, p, dc.e2);
  const double u4 = fma(4.0, al, del);
  const double det = fma(del, u4, 6.0 * al * al);
  const double inv = 1.0 / det;
  const double c1 = u4 * inv, c2 = -al * inv;
  // K r
  const double k00 = fma(s3, r01, r00), k01 = fma(3.0, r01, -s3 * r00);
  const double k10 = fma(s3, r11, r10), k11 = fma(3.0, r11, -s3 * r10);
  // g0 = tt r0 + a K r0 - be r1 ; g1 = p r1 + a K r1 + be r0
  const double g00 = fma(tt, r00, fma(dc.a, k00, -dc.be * r10));
  const double g01 = fma(tt, r01, fma(dc.a, k01, -dc.be * r11));
  const double g10 = fma(p, r10, fma(dc.a, k10, dc.be * r00));
  const double g11 = fma(p, r11, fma(dc.a, k11, dc.be * r01));
  // f = c1 g + c2 K g
  const double h00 = fma(s3, g01, g00), h01 = fma(3.0, g01, -s3 * g00);
  const double h10 = fma(s3, g11, g10), h11 = fma(3.0, g11, -s3 * g10);
  f[0] = fma(c1, g00, c2 * h00);
  f[1] = fma(c1, g01, c2 * h01);
  f[2] = fma(c1, g10, c2 * h10);
  f[3] = fma(c1, g11, c2 * h11);
  Xo0 = dc.a * fma(s3, f[1], f[0]);
  Xo1 = dc.a * fma(s3, f[3], f[2]);
  Yo0 = dc.b * fma(s3, f[2], f[0]);
  Yo1 = dc.b * fma(s3, f[3], f[1]);
}

template <int D>
__global__ void __launch_bounds__(kNW * 32, 2) sweep2d_kernel(const Sweep2DArgs a) {
  extern __shared__ double sm[];
  double* red = sm;  // [kC][kNW][32][4]
  DirConst* tab = reinterpret_cast<DirConst*>(sm + kC * kNW * 32 * 4);  // [kNW*D]
  __shared__ int item_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nx = a.nx, ny = a.ny;
  const long ncell = (long)nx * ny, nd = 4 * ncell;
  const int nbands = (ny + 31) / 32;
  const int per_band = a.S * 4 * a.groups;
  const int total = nbands * per_band;
  const int ndir = kNW * D;
  unsigned* ticket = a.sync;
  unsigned* progress = a.sync + 1;

  for (;;) {
    if (threadIdx.x == 0) item_sh = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int item = item_sh;
    if (item >= total) break;
    const int band = item / per_band;
    const int rem = item - band * per_band;
    const int s = rem / (4 * a.groups);
    const int qg = rem - s * 4 * a.groups;
    const int qd = qg / a.groups;
    const int grp = qg - qd * a.groups;
    const int ibase = (s * 4 + qd) * a.groups + grp;
    if (a.active && !a.active[s]) {
      __syncthreads();
      continue;
    }
    const int qx = qd & 1, qy = qd >> 1;
    const double sx = qx ? -1.0 : 1.0, sy = qy ? -1.0 : 1.0;

    // direction table of this item
    for (int i = threadIdx.x; i < ndir; i += blockDim.x) {
      const Slot2D sl = a.slots[qd * a.nq_pad + grp * ndir + i];
      DirConst d;
      d.a = sl.a;
      d.b = sl.b;
      d.w = sl.w;
      d.e1 = 3.0 * sl.b * sl.b - 6.0 * sl.a * sl.a;
      d.e2 = 2.0 * sl.a * sl.b + 4.0 * sl.a * sl.a;
      d.tb = 2.0 * sl.b;
      d.be = kSqrt3 * sl.b;
      d.bcx = (a.mode & SRC_BC) ? sl.bcx : 0.0;
      d.bcy = (a.mode & SRC_BC) ? sl.bcy : 0.0;
      tab[i] = d;
    }
    __syncthreads();

    const int yr = band * 32 + lane;  // canonical row
    const bool row_ok = yr < ny;
    const int iy = qy ? ny - 1 - yr : yr;
    double X[D][2], Y[D][2];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      X[d][0] = tab[warp * D + d].bcx;
      X[d][1] = 0.0;
      Y[d][0] = 0.0;
      Y[d][1] = 0.0;
    }
    const double2* ybelow =
        reinterpret_cast<const double2*>(a.ybuf) + ((long)(ibase * nbands + band - 1) * nx) * ndir;
    double2* yabove = reinterpret_cast<double2*>(a.ybuf) + ((long)(ibase * nbands + band) * nx) * ndir;
    const double* gsrc = a.g + (a.g_shared ? 0 : (long)s * nd);
    const double* rho = a.rho + (long)s * nd;
    const double* sgt = a.sig_t + (long)s * ncell;
    const double* sgs = a.sig_s + (long)s * ncell;
    double* part = a.part + ((long)(qd * a.groups + grp) * a.S + s) * nd;

    const int nsteps = nx + 31;
    for (int k0 = 0; k0 < nsteps; k0 += kC) {
      if (band > 0) {
        if (threadIdx.x == 0) {
          const unsigned need = (unsigned)min(nx, k0 + kC);
          const unsigned* pc = progress + ibase * nbands + band - 1;
          while (ld_acquire(pc) < need) __nanosleep(100);
        }
        __syncthreads();
      }
#pragma unroll 1
      for (int kk = 0; kk < kC; ++kk) {
        const int x = k0 + kk - lane;
        const bool ok = row_ok && x >= 0 && x < nx;
        double q[4] = {0.0, 0.0, 0.0, 0.0};
        double sig = 1.0;
        long cell = 0;
        if (ok) {
          const int ix = qx ? nx - 1 - x : x;
          cell = (long)iy * nx + ix;
          sig = sgt[cell];
          if (a.mode & SRC_RAW) {
            const double2 r01 = *reinterpret_cast<const double2*>(rho + 4 * cell);
            const double2 r23 = *reinterpret_cast<const double2*>(rho + 4 * cell + 2);
            q[0] = r01.x; q[1] = r01.y; q[2] = r23.x; q[3] = r23.y;
          } else {
            if (a.mode & SRC_MS_RHO) {
              const double ss = sgs[cell];
              const double2 r01 = *reinterpret_cast<const double2*>(rho + 4 * cell);
              const double2 r23 = *reinterpret_cast<const double2*>(rho + 4 * cell + 2);
              q[0] = ss * r01.x; q[1] = ss * r01.y; q[2] = ss * r23.x; q[3] = ss * r23.y;
            }
            if (a.mode & SRC_G) {
              const double2 g01 = *reinterpret_cast<const double2*>(gsrc + 4 * cell);
              const double2 g23 = *reinterpret_cast<const double2*>(gsrc + 4 * cell + 2);
              q[0] += g01.x; q[1] += g01.y; q[2] += g23.x; q[3] += g23.y;
            }
          }
          q[1] *= sx;
          q[2] *= sy;
          q[3] *= sx * sy;
        }
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const DirConst& dc = tab[warp * D + d];
          double Y0 = __shfl_up_sync(0xffffffffu, Y[d][0], 1);
          double Y1 = __shfl_up_sync(0xffffffffu, Y[d][1], 1);
          if (lane == 0) {
            if (band == 0) {
              Y0 = dc.bcy;
              Y1 = 0.0;
            } else if (x >= 0 && x < nx) {
              const double2 yb = __ldcg(ybelow + (long)x * ndir + warp * D + d);
              Y0 = yb.x;
              Y1 = yb.y;
            }
          }
          double f[4], xo0, xo1, yo0, yo1;
          solve_cell(dc, sig, q, X[d][0], X[d][1], Y0, Y1, f, xo0, xo1, yo0, yo1);
          Y[d][0] = yo0;
          Y[d][1] = yo1;
          if (ok) {
            X[d][0] = xo0;
            X[d][1] = xo1;
            acc0 = fma(dc.w, f[0], acc0);
            acc1 = fma(dc.w, f[1], acc1);
            acc2 = fma(dc.w, f[2], acc2);
            acc3 = fma(dc.w, f[3], acc3);
            if (lane == 31 && band + 1 < nbands) __stcg(yabove + (long)x * ndir + warp * D + d, make_double2(yo0, yo1));
          }
        }
        double* rr = red + ((kk * kNW + warp) * 32 + lane) * 4;
        rr[0] = acc0;
        rr[1] = acc1;
        rr[2] = acc2;
        rr[3] = acc3;
      }
      __syncthreads();
      // fixed-order reduction over the warps (direction subgroups) of the chunk
      for (int t = threadIdx.x; t < kC * 32; t += blockDim.x) {
        const int kk = t >> 5, ln = t & 31;
        const int x = k0 + kk - ln;
        const int yy = band * 32 + ln;
        if (x >= 0 && x < nx && yy < ny) {
          double v0 = 0, v1 = 0, v2 = 0, v3 = 0;
          for (int w = 0; w < kNW; ++w) {
            const double* rr = red + ((kk * kNW + w) * 32 + ln) * 4;
            v0 += rr[0];
            v1 += rr[1];
            v2 += rr[2];
            v3 += rr[3];
          }
          const int ix = qx ? nx - 1 - x : x;
          const int iyy = qy ? ny - 1 - yy : yy;
          double* o = part + 4 * ((long)iyy * nx + ix);
          *reinterpret_cast<double2*>(o) = make_double2(v0, sx * v1);
          *reinterpret_cast<double2*>(o + 2) = make_double2(sy * v2, sx * sy * v3);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && band + 1 < nbands) {
        __threadfence();
        const int avail = min(nx, max(0, k0 + kC - 31));
        st_release(progress + ibase * nbands + band, (unsigned)avail);
      }
    }
  }
}

template <int D>
void launch_d(const Sweep2DArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)kC * kNW * 32 * 4 * 8 + (size_t)kNW * D * sizeof(DirConst);
  static int max_ctas = -1;
  if (max_ctas < 0) {
    RTE_CUDA(cudaFuncSetAttribute(sweep2d_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, dev = 0, sms = 0;
    RTE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep2d_kernel<D>, kNW * 32, smem));
    RTE_CUDA(cudaGetDevice(&dev));
    RTE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    max_ctas = std::max(1, per_sm) * sms;
  }
  const int nbands = (a.ny + 31) / 32;
  const long total = (long)nbands * a.S * 4 * a.groups;
  const int grid = (int)std::min<long>(total, max_ctas);
  sweep2d_kernel<D><<<grid, kNW * 32, smem, st>>>(a);
  RTE_CUDA(cudaGetLastError());
}

__global__ void reduce_partials_kernel(int S, long nd, int nparts, const double* __restrict__ part,
                                       double* __restrict__ out, const double* __restrict__ rho_prev,
                                       double* __restrict__ delta, unsigned long long* change_bits,
                                       const int* active) {
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  double mx_d = 0.0, mx_r = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += stride) {
    double v = 0.0;
    for (int p = 0; p < nparts; ++p) v += __ldcs(part + ((long)p * S + s) * nd + i);
    out[(long)s * nd + i] = v;
    if (delta) {
      const double d = v - rho_prev[(long)s * nd + i];
      delta[(long)s * nd + i] = d;
      mx_d = fmax(mx_d, fabs(d));
      if (d != d) mx_d = d;
      mx_r = fmax(mx_r, fabs(v));
    }
  }
  if (change_bits) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      mx_d = fmax(mx_d, __shfl_xor_sync(0xffffffffu, mx_d, d));
      mx_r = fmax(mx_r, __shfl_xor_sync(0xffffffffu, mx_r, d));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMax(change_bits + 2 * s, (unsigned long long)__double_as_longlong(fabs(mx_d)));
      atomicMax(change_bits + 2 * s + 1, (unsigned long long)__double_as_longlong(mx_r));
    }
  }
}

}  // namespace

void launch_sweep2d(const Sweep2DArgs& a, cudaStream_t st) {
  const int dpc = a.nq_pad / a.groups / kNW;  // directions per lane
  switch (dpc) {
    case 1: return launch_d<1>(a, st);
    case 2: return launch_d<2>(a, st);
    case 4: return launch_d<4>(a, st);
    case 8: return launch_d<8>(a, st);
    default: throw Error(RTE_ERR_UNSUPPORTED, "sweep2d: unsupported direction grouping");
  }
}

void launch_reduce_partials(int S, long nd, int nparts, const double* part, double* out, const double* rho_prev,
                            double* delta, unsigned long long* change_bits, const int* active, cudaStream_t st) {
  const int threads = 256;
  const long blocks_x = std::min<long>((nd + threads - 1) / threads, std::max<long>(1, 4096 / S));
  dim3 grid((unsigned)blocks_x, (unsigned)S);
  reduce_partials_kernel<<<grid, threads, 0, st>>>(S, nd, nparts, part, out, rho_prev, delta, change_bits, active);
  RTE_CUDA(cudaGetLastError());
}

int sweep2d_dirs_per_cta() { return kNW; }

}  // namespace rte
