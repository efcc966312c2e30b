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
#include <cstdint>
#include <type_traits>

namespace rte {
namespace {

#ifndef RTE_SWEEP_NW
#define RTE_SWEEP_NW 8
#endif
#ifndef RTE_SWEEP_MINB
#define RTE_SWEEP_MINB 2
#endif
#ifndef RTE_SWEEP_KK_UNROLL
#define RTE_SWEEP_KK_UNROLL 1
#endif
#ifndef RTE_SWEEP_LEAD
#define RTE_SWEEP_LEAD 4
#endif
#ifndef RTE_SWEEP_PUB
#define RTE_SWEEP_PUB 1
#endif
// Columns the band below must have finished before an item starts (at least
// one chunk).  Measured at C5 (RTE_SWEEP_DEBUG_WAIT): items spend ~1% of their
// cycles in this start wait and ~12% in later chunk waits; a lead of 64
// columns changes neither (2.4% / 12%), 256 moves the wait to the start (26% /
// 4%) -- consecutive bands of a (sample, quadrant) chain are co-resident (296
// CTA slots for 64 chains) and a consumer whose SM-mate idles catches up with
// its producer whatever head start the producer had.
constexpr int kLead = RTE_SWEEP_LEAD;
constexpr int kPub = RTE_SWEEP_PUB;  // progress is published every kPub chunks (and at the end)
constexpr int kKU = RTE_SWEEP_KK_UNROLL;  // unroll of the step loop inside a chunk
constexpr int kNW = RTE_SWEEP_NW;  // warps per CTA (direction subgroups)
constexpr int kC = 4;    // steps per synchronisation chunk
constexpr int kRC = 40;  // ring slots (columns): >= 31 + 2 * kC
constexpr int kRP = 162; // ring slot pitch in doubles (5 comps x 32 rows, padded to even)

// Bulk staging (TMA bulk copies, used when nx is a multiple of kC so every row
// segment is 16-byte aligned): each band row's kC cells of rho / G / sigma_t /
// sigma_s and the chunk's band-below traces are contiguous in global memory
// and arrive by cp.async.bulk into row-major stage arrays (padded pitches
// against bank conflicts), completion counted on an mbarrier.
constexpr int kSP4 = 4 * kC + 2;  // row pitch (doubles) of the staged rho / G rows
constexpr int kSP1 = kC + 2;      // row pitch of the staged sigma_t / sigma_s rows
constexpr int kStageDoubles = 2 * 32 * kSP4 + 2 * 32 * kSP1;  // >= kC * 32 * 10 of the cp.async layout

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned addr = smem_u32(bar);
  unsigned done = 0;
  for (unsigned spins = 0; !done; ++spins) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (!done && spins > (1u << 24)) __trap();  // a lost bulk copy must not hang the device
  }
}
// global -> shared bulk copy (bytes and both addresses multiples of 16), completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Per-direction constants of the canonical cell solve, 16-byte aligned so the
// pairs below load as one 128-bit shared-memory access each.
struct __align__(16) DirConst {
  double a, b;      // |vx|/hx, |vy|/hy
  double sa, sb;    // sqrt3 a, sqrt3 b
  double c4b, k1;   // del = sig (sig + 4b) + 6 (b^2 - a^2)
  double a2, k2;    // al = 2a sig + 4ab + 4a^2
  double cA, cB;    // diagonal shifts of G = (sig I + C) r: 3b + a, 3b + 3a
  double cC, cD;    //                                          b + a,  b + 3a
  double w, bcx;    // folded weight; unscaled x-face inflow trace (y-mode 0)
  double bcy, pad0; // unscaled y-face inflow trace (x-mode 0)
  int dir0, dir1, pad1, pad2;
};

// The constants solve_cell reads, as 128-bit shared-memory loads.
struct DirK {
  double a, b, sa, sb, c4b, k1, a2, k2, cA, cB, cC, cD, w;
};
__device__ __forceinline__ DirK load_dirk(const DirConst* p) {
  const double2* v = reinterpret_cast<const double2*>(p);
  const double2 v0 = v[0], v1 = v[1], v2 = v[2], v3 = v[3], v4 = v[4], v5 = v[5], v6 = v[6];
  return DirK{v0.x, v0.y, v1.x, v1.y, v2.x, v2.y, v3.x, v3.y, v4.x, v4.y, v5.x, v5.y, v6.x};
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 1/x for x > 0 (normal): hardware approximation + two Newton steps (~1 ulp).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Canonical cell solve (see file header).  q: reflected source moments;
// x0, x1: incoming x-face traces per y-mode; y0, y1: incoming y-face traces
// per x-mode (unscaled).  With r = q + face terms, the block is
// B = sig I + I (x) aK + bK (x) I and B^-1 = E (sig I + C) with C a constant
// per direction and E = [[e1, -e2], [e2, e3]] on each mode pair, where
// del = sig (sig + 4b) + 6 (b^2 - a^2), al = 2a sig + 4ab + 4a^2,
// n1 = del + 3 al, n3 = del + al, det = n1 n3 + 3 al^2,
// e1 = n1 / det, e3 = n3 / det, e2 = sqrt3 al / det
// (the closed form of (del I + al K)^-1 applied after (sig I + C); 56 FP64
// instructions per cell-direction including the weighted accumulation).
__device__ __forceinline__ void solve_cell(const DirK& dc, double sig, const double q[4], double x0, double x1,
                                           double y0, double y1, double f[4], double& xo0, double& xo1,
                                           double& yo0, double& yo1) {
  const double s3 = kSqrt3;
  const double r00 = fma(dc.a, x0, fma(dc.b, y0, q[0]));
  const double r01 = fma(-dc.sa, x0, fma(dc.b, y1, q[1]));
  const double r10 = fma(-dc.sb, y0, fma(dc.a, x1, q[2]));
  const double r11 = fma(-dc.sa, x1, fma(-dc.sb, y1, q[3]));
  const double del = fma(sig, sig + dc.c4b, dc.k1);
  const double al = fma(dc.a2, sig, dc.k2);
  const double n1 = fma(3.0, al, del);
  const double n3 = del + al;
  const double inv = fast_rcp(fma(n1, n3, (3.0 * al) * al));
  const double e1 = n1 * inv, e3 = n3 * inv, e2 = (s3 * al) * inv;
  const double g00 = fma(sig + dc.cA, r00, fma(dc.sa, r01, -dc.sb * r10));
  const double g01 = fma(sig + dc.cB, r01, fma(-dc.sa, r00, -dc.sb * r11));
  const double g10 = fma(sig + dc.cC, r10, fma(dc.sa, r11, dc.sb * r00));
  const double g11 = fma(sig + dc.cD, r11, fma(-dc.sa, r10, dc.sb * r01));
  f[0] = fma(e1, g00, -e2 * g01);
  f[1] = fma(e3, g01, e2 * g00);
  f[2] = fma(e1, g10, -e2 * g11);
  f[3] = fma(e3, g11, e2 * g10);
  xo0 = fma(s3, f[1], f[0]);
  xo1 = fma(s3, f[3], f[2]);
  yo0 = fma(s3, f[2], f[0]);
  yo1 = fma(s3, f[3], f[1]);
}

// General cell solve for full per-cell mass blocks (intra-cell-varying
// coefficients): B = M + I (x) (a K) + (b K) (x) I with M the reflected 4x4
// total-interaction block; LU without pivoting (the symmetric part of B is
// positive definite), same face-trace algebra as solve_cell.
__device__ __forceinline__ void solve_cell_full(const DirK& dc, const double M[16], const double q[4], double x0,
                                                double x1, double y0, double y1, double f[4], double& xo0,
                                                double& xo1, double& yo0, double& yo1) {
  const double s3 = kSqrt3;
  double r[4];
  r[0] = fma(dc.a, x0, fma(dc.b, y0, q[0]));
  r[1] = fma(-dc.sa, x0, fma(dc.b, y1, q[1]));
  r[2] = fma(-dc.sb, y0, fma(dc.a, x1, q[2]));
  r[3] = fma(-dc.sa, x1, fma(-dc.sb, y1, q[3]));
  double B[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) B[e] = M[e];
  const double a = dc.a, b = dc.b;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int o = 2 * k;  // (I (x) aK): x-mode pair (o, o+1) of y-mode k
    B[o * 4 + o] += a;
    B[o * 4 + o + 1] += s3 * a;
    B[(o + 1) * 4 + o] -= s3 * a;
    B[(o + 1) * 4 + o + 1] += 3.0 * a;
    // (bK (x) I): y-mode pair (k, k+2) of x-mode k
    B[k * 4 + k] += b;
    B[k * 4 + k + 2] += s3 * b;
    B[(k + 2) * 4 + k] -= s3 * b;
    B[(k + 2) * 4 + k + 2] += 3.0 * b;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double piv = fast_rcp(B[k * 4 + k]);
#pragma unroll
    for (int i = k + 1; i < 4; ++i) {
      const double l = B[i * 4 + k] * piv;
#pragma unroll
      for (int j = k + 1; j < 4; ++j) B[i * 4 + j] = fma(-l, B[k * 4 + j], B[i * 4 + j]);
      r[i] = fma(-l, r[k], r[i]);
    }
    B[k * 4 + k] = piv;
  }
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    double v = r[i];
#pragma unroll
    for (int j = i + 1; j < 4; ++j) v = fma(-B[i * 4 + j], f[j], v);
    f[i] = v * B[i * 4 + i];
  }
  xo0 = fma(s3, f[1], f[0]);
  xo1 = fma(s3, f[3], f[2]);
  yo0 = fma(s3, f[2], f[0]);
  yo1 = fma(s3, f[3], f[1]);
}

#ifdef RTE_SWEEP_DEBUG_WAIT
__device__ unsigned long long g_dbg[8];  // [0] prologue wait, [1] chunk waits, [2] item cycles, [3] items, [4] polls
#define DBG_T0() const long long dbg_t0 = clock64()
#define DBG_ADD(i) atomicAdd(&g_dbg[i], (unsigned long long)(clock64() - dbg_t0))
#else
#define DBG_T0()
#define DBG_ADD(i)
#endif

struct Smem {
  double* red;    // [kC][kNW][4][32]
  double* ring;   // [kRC][kRP]: comps 0..3 = reflected q, 4 = sigma_t; row fastest
  double* stage;  // cp.async path: [kC*32][10] raw rho(4), G(4), sigma_t, sigma_s of the next columns;
                  // bulk path: rho rows [32][kSP4], G rows [32][kSP4], sigma_t rows [32][kSP1], sigma_s rows [32][kSP1]
  unsigned long long* bar;  // mbarrier of the bulk staging
  double* ystg;   // [2][kC][ndir][2]
  DirConst* tab;  // [ndir]
};

template <int D>
__device__ __forceinline__ void issue_chunk_loads(const Sweep2DArgs& a, const Smem& sm, int c0, int band,
                                                  int qx, int qy, int s, const double2* ybelow, int ybuf_slot) {
  const int nx = a.nx, ny = a.ny;
  const long ncell = (long)nx * ny, nd = 4 * ncell;
  const int t = threadIdx.x;
  // raw cell data: 128 cells, two threads per cell
  {
    const int cell = t & (kC * 32 - 1);
    const int part = t / (kC * 32);
    const int col = c0 + (cell >> 5), row = band * 32 + (cell & 31);
    if (part < 2 && col < nx && row < ny) {
      const int ix = qx ? nx - 1 - col : col;
      const int iy = qy ? ny - 1 - row : row;
      const long pc = (long)iy * nx + ix;
      double* dst = sm.stage + cell * 10;
      // rho / G are only staged when the mode reads them (the rhs assembly
      // passes no per-sample rho; apply_L skips the G stream)
      if (part == 0) {
        if (a.mode & (SRC_MS_RHO | SRC_RAW)) {
          const double* src = a.rho + (long)s * nd + 4 * pc;
          cp_async16(dst, src);
          cp_async16(dst + 2, src + 2);
        }
        cp_async8(dst + 8, a.sig_t + (long)s * ncell + pc);
      } else {
        if (a.mode & SRC_G) {
          const double* src = a.g + (a.g_shared ? 0 : (long)s * nd) + 4 * pc;
          cp_async16(dst + 4, src);
          cp_async16(dst + 6, src + 2);
        }
        cp_async8(dst + 9, a.sig_s + (long)s * ncell + pc);
      }
    }
  }
  // band-boundary traces from the band below; the bottom band reads the
  // inflow traces (y-face, x-mode 0) of its directions instead
  {
    constexpr int ndir = kNW * D;
    for (int i = t; i < kC * ndir; i += blockDim.x) {
      const int kk = i / ndir, dd = i - kk * ndir;
      const int col = c0 + kk;
      double* dst = sm.ystg + (((ybuf_slot * kC + kk) * ndir + dd) << 1);
      if (band > 0) {
        if (col < nx) cp_async16(dst, ybelow + (long)col * ndir + dd);
      } else {
        dst[0] = sm.tab[dd].bcy;
        dst[1] = 0.0;
      }
    }
  }
  cp_async_commit();
}

// Bulk-copy version of issue_chunk_loads (nx % kC == 0): one copy per band row
// and array (threads 0..127: row = t % 32, array = t / 32), one for the chunk's
// band-below traces; thread 0 posts the expected byte count first.
template <int D>
__device__ __forceinline__ void issue_chunk_bulk(const Sweep2DArgs& a, const Smem& sm, int c0, int band, int qx,
                                                 int qy, int s, const double2* ybelow, int ybuf_slot) {
  constexpr int ndir = kNW * D;
  const int nx = a.nx, ny = a.ny;
  const long ncell = (long)nx * ny, nd = 4 * ncell;
  const int t = threadIdx.x;
  const bool want_rho = (a.mode & (SRC_MS_RHO | SRC_RAW)) != 0, want_g = (a.mode & SRC_G) != 0;
  if (t == 0) {
    const int rows = min(32, ny - band * 32);
    unsigned bytes = (unsigned)rows * (2u * kC * 8u + (want_rho ? 4u * kC * 8u : 0u) + (want_g ? 4u * kC * 8u : 0u));
    if (band > 0) bytes += (unsigned)(kC * ndir * sizeof(double2));
    mbar_arrive_expect_tx(sm.bar, bytes);
  }
  __syncwarp();
  if (t < 128) {
    const int row = t & 31, arr = t >> 5;
    const int yrow = band * 32 + row;
    if (yrow < ny) {
      const int ix0 = qx ? nx - c0 - kC : c0;  // the chunk's kC cells are contiguous along x (reversed when reflected)
      const long pc = (long)(qy ? ny - 1 - yrow : yrow) * nx + ix0;
      if (arr == 0) {
        if (want_rho) bulk_g2s(sm.stage + row * kSP4, a.rho + (long)s * nd + 4 * pc, 4 * kC * 8, sm.bar);
      } else if (arr == 1) {
        if (want_g)
          bulk_g2s(sm.stage + 32 * kSP4 + row * kSP4, a.g + (a.g_shared ? 0 : (long)s * nd) + 4 * pc, 4 * kC * 8,
                   sm.bar);
      } else if (arr == 2) {
        bulk_g2s(sm.stage + 64 * kSP4 + row * kSP1, a.sig_t + (long)s * ncell + pc, kC * 8, sm.bar);
      } else {
        bulk_g2s(sm.stage + 64 * kSP4 + 32 * kSP1 + row * kSP1, a.sig_s + (long)s * ncell + pc, kC * 8, sm.bar);
      }
    }
  } else if (t == 128 && band > 0) {
    bulk_g2s(sm.ystg + (size_t)ybuf_slot * kC * ndir * 2, ybelow + (long)c0 * ndir, kC * ndir * sizeof(double2),
             sm.bar);
  }
  if (band == 0) {
    // the bottom band reads the inflow traces (y-face, x-mode 0) of its directions
    for (int i = t; i < kC * ndir; i += blockDim.x) {
      const int dd = i % ndir;
      double* dst = sm.ystg + (((size_t)ybuf_slot * kC * ndir + i) << 1);
      dst[0] = sm.tab[dd].bcy;
      dst[1] = 0.0;
    }
  }
}

// stage -> ring (reflected source moments + sigma_t) for columns c0..c0+kC-1
template <bool FULL, bool BULK>
__device__ __forceinline__ void convert_chunk(const Sweep2DArgs& a, const Smem& sm, int c0, int band, double sx,
                                              double sy, int s, int qx, int qy) {
  const int t = threadIdx.x;
  if (t >= kC * 32) return;
  const int col = c0 + (t >> 5), row = t & 31;
  const bool ok = col < a.nx && band * 32 + row < a.ny;
  double r[10];
  if (BULK) {
    // row-major staged rows; the cells of a reflected chunk arrive in reverse order
    const int j = qx ? kC - 1 - (t >> 5) : (t >> 5);
    const double* pr = sm.stage + row * kSP4 + 4 * j;
    const double* pg = pr + 32 * kSP4;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      r[e] = pr[e];
      r[4 + e] = pg[e];
    }
    r[8] = sm.stage[64 * kSP4 + row * kSP1 + j];
    r[9] = sm.stage[64 * kSP4 + 32 * kSP1 + row * kSP1 + j];
  } else {
    const double* pr = sm.stage + t * 10;
#pragma unroll
    for (int e = 0; e < 10; ++e) r[e] = pr[e];
  }
  double q0 = 0, q1 = 0, q2 = 0, q3 = 0, sg = 1.0;
  if (ok) {
    sg = r[8];
    if (a.mode & SRC_RAW) {
      q0 = r[0]; q1 = r[1]; q2 = r[2]; q3 = r[3];
    } else {
      if (a.mode & SRC_MS_RHO) {
        if (FULL) {
          // full per-cell scattering block (physical orientation; reflected below)
          const int ix = qx ? a.nx - 1 - col : col;
          const int iy = qy ? a.ny - 1 - (band * 32 + row) : band * 32 + row;
          const double* m = a.ms_blk + ((long)s * a.nx * a.ny + (long)iy * a.nx + ix) * 16;
          q0 = m[0] * r[0] + m[1] * r[1] + m[2] * r[2] + m[3] * r[3];
          q1 = m[4] * r[0] + m[5] * r[1] + m[6] * r[2] + m[7] * r[3];
          q2 = m[8] * r[0] + m[9] * r[1] + m[10] * r[2] + m[11] * r[3];
          q3 = m[12] * r[0] + m[13] * r[1] + m[14] * r[2] + m[15] * r[3];
        } else {
          const double ss = r[9];
          q0 = ss * r[0]; q1 = ss * r[1]; q2 = ss * r[2]; q3 = ss * r[3];
        }
      }
      if (a.mode & SRC_G) {
        q0 += r[4]; q1 += r[5]; q2 += r[6]; q3 += r[7];
      }
    }
  }
  double* dst = sm.ring + (col % kRC) * kRP + row;
  dst[0] = q0;
  dst[32] = sx * q1;
  dst[64] = sy * q2;
  dst[96] = sx * sy * q3;
  dst[128] = sg;
}

template <int D, bool KIN, bool FULL>
__global__ void __launch_bounds__(kNW * 32, RTE_SWEEP_MINB) sweep2d_kernel(const Sweep2DArgs a) {
  extern __shared__ double smraw[];
  constexpr int ndir = kNW * D;
  Smem sm;
  sm.red = smraw;
  sm.ring = sm.red + kC * kNW * 4 * 32;
  sm.stage = sm.ring + kRC * kRP;
  sm.ystg = sm.stage + kStageDoubles;
  __shared__ __align__(8) unsigned long long stage_bar;
  sm.bar = &stage_bar;
#ifdef RTE_SWEEP_NOBULK
  const bool bulk = false;
#else
  const bool bulk = a.nx % kC == 0;
#endif
  sm.tab = reinterpret_cast<DirConst*>(sm.ystg + 2 * kC * ndir * 2);
  __shared__ int item_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nx = a.nx, ny = a.ny;
  const long ncell = (long)nx * ny, nd = 4 * ncell;
  const int nbands = (ny + 31) / 32;
  const int per_band = a.S * 4 * a.groups;
  const int total = nbands * per_band;
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
    // every item starts the staging barrier at phase 0 (one arrival: thread 0's expect_tx)
    if (bulk && threadIdx.x == 0) mbar_init(sm.bar, 1);
    for (int i = threadIdx.x; i < ndir; i += blockDim.x) {
      const Slot2D sl = a.slots[qd * a.nq_pad + grp * ndir + i];
      DirConst d;
      d.a = sl.a;
      d.b = sl.b;
      d.sa = kSqrt3 * sl.a;
      d.sb = kSqrt3 * sl.b;
      d.w = sl.w;
      d.c4b = 4.0 * sl.b;
      d.k1 = 6.0 * (sl.b * sl.b - sl.a * sl.a);
      d.a2 = 2.0 * sl.a;
      d.k2 = 4.0 * sl.a * sl.b + 4.0 * sl.a * sl.a;
      d.cA = 3.0 * sl.b + sl.a;
      d.cB = 3.0 * sl.b + 3.0 * sl.a;
      d.cC = sl.b + sl.a;
      d.cD = sl.b + 3.0 * sl.a;
      // Slot2D carries the inflow ghost traces scaled by a (x) / b (y)
      d.bcx = (a.mode & SRC_BC) && sl.a > 0.0 ? sl.bcx / sl.a : 0.0;
      d.bcy = (a.mode & SRC_BC) && sl.b > 0.0 ? sl.bcy / sl.b : 0.0;
      d.pad0 = 0.0;
      d.dir0 = sl.dir0;
      d.dir1 = sl.dir1;
      sm.tab[i] = d;
    }
    const double2* ybelow =
        reinterpret_cast<const double2*>(a.ybuf) + ((long)(ibase * nbands + band - 1) * nx) * ndir;
    double2* yabove = reinterpret_cast<double2*>(a.ybuf) + ((long)(ibase * nbands + band) * nx) * ndir;
    double* part = a.part + ((long)(qd * a.groups + grp) * a.S + s) * nd;
    const unsigned* prod = progress + ibase * nbands + band - 1;

    // prologue: columns [0, kC).  Thread 0 keeps the last progress value it
    // observed (`seen`): once the band below runs ahead, most chunks need no
    // poll at all.
    unsigned seen = 0;
#ifndef RTE_SWEEP_NOWAIT  // development bound only: drops the band hand-off (wrong answers)
#ifdef RTE_SWEEP_DEBUG_WAIT
    const long long dbg_item0 = clock64();
#endif
    if (band > 0 && threadIdx.x == 0) {
      DBG_T0();
      const unsigned need = (unsigned)min(nx, max(kC, kLead));
      while ((seen = ld_acquire(prod)) < need) __nanosleep(64);
      DBG_ADD(0);
    }
#endif
    __syncthreads();
    if (bulk) {
      issue_chunk_bulk<D>(a, sm, 0, band, qx, qy, s, ybelow, 0);
      mbar_wait(sm.bar, 0);
    } else {
      issue_chunk_loads<D>(a, sm, 0, band, qx, qy, s, ybelow, 0);
      cp_async_wait_all();
    }
    __syncthreads();
    if (bulk)
      convert_chunk<FULL, true>(a, sm, 0, band, sx, sy, s, qx, qy);
    else
      convert_chunk<FULL, false>(a, sm, 0, band, sx, sy, s, qx, qy);

    const int yr = band * 32 + lane;
    const bool row_ok = yr < ny;
    const bool band_full = band * 32 + 31 < ny;
    double X[D][2], Y[D][2];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      X[d][0] = sm.tab[warp * D + d].bcx;
      X[d][1] = 0.0;
      Y[d][0] = 0.0;
      Y[d][1] = 0.0;
    }
    const int nsteps = nx + 31;
    int ys = 0;  // ystg slot holding the current chunk
    for (int k0 = 0; k0 < nsteps; k0 += kC) {
#ifndef RTE_SWEEP_NOWAIT
      if (band > 0 && threadIdx.x == 0) {
        const unsigned need = (unsigned)min(nx, k0 + 2 * kC);
        if (seen < need) {
          DBG_T0();
          while ((seen = ld_acquire(prod)) < need) __nanosleep(64);
          DBG_ADD(1);
#ifdef RTE_SWEEP_DEBUG_WAIT
          atomicAdd(&g_dbg[4], 1ull);
#endif
        }
      }
#endif
      __syncthreads();
      if (k0 + kC < nx) {
        if (bulk)
          issue_chunk_bulk<D>(a, sm, k0 + kC, band, qx, qy, s, ybelow, ys ^ 1);
        else
          issue_chunk_loads<D>(a, sm, k0 + kC, band, qx, qy, s, ybelow, ys ^ 1);
      }
      // One step of the wavefront for this lane's D directions.  EDGE = false
      // is the interior version (every lane of the chunk solves a real cell:
      // no validity selects); EDGE = true handles the fill / drain chunks and
      // partial bands.  Lane 0's incoming y-traces (the band below's top
      // traces, or the inflow values) are loaded into lane 31's Y registers,
      // whose own traces went to `yabove` at the end of the previous step, so a
      // rotating shuffle delivers every lane's incoming trace without a select.
      auto step = [&](auto edge_tag, int kk) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        const int x = k0 + kk - lane;
        const bool ok = !EDGE || (row_ok && x >= 0 && x < nx);
        const double* rg = sm.ring + (EDGE ? ((x % kRC) + kRC) % kRC : x % kRC) * kRP + lane;
        double q[4];
        q[0] = rg[0];
        q[1] = rg[32];
        q[2] = rg[64];
        q[3] = rg[96];
        const double sig = ok ? rg[128] : 1.0;
        if (!ok) q[0] = q[1] = q[2] = q[3] = 0.0;
        double M[FULL ? 16 : 1];
        if (FULL) {
          // reflected full block of this lane's cell: M'_ij = s_i s_j M_ij, s = (1, sx, sy, sx sy)
          const int ix = qx ? nx - 1 - x : x;
          const int iyy = qy ? ny - 1 - yr : yr;
          const double* m = a.mt_blk + ((long)s * ncell + (long)iyy * nx + (ok ? ix : 0)) * 16;
          const double sg[4] = {1.0, sx, sy, sx * sy};
#pragma unroll
          for (int e = 0; e < 16; ++e) M[e] = ok ? __ldg(m + e) * sg[e >> 2] * sg[e & 3] : (e % 5 == 0 ? 1.0 : 0.0);
        }
        const double* yst = sm.ystg + ((ys * kC + kk) * ndir + warp * D) * 2;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        // Branch-free direction loop: the D chains are independent and the
        // compiler interleaves them (no reconvergence points inside).
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const DirK dc = load_dirk(sm.tab + warp * D + d);
          if (lane == 31) {
            const double2 ysv = *reinterpret_cast<const double2*>(yst + 2 * d);
            Y[d][0] = ysv.x;
            Y[d][1] = ysv.y;
          }
          const double Y0 = __shfl_sync(0xffffffffu, Y[d][0], lane + 31);
          const double Y1 = __shfl_sync(0xffffffffu, Y[d][1], lane + 31);
          double f[4], xo0, xo1, yo0, yo1;
          if (FULL)
            solve_cell_full(dc, M, q, X[d][0], X[d][1], Y0, Y1, f, xo0, xo1, yo0, yo1);
          else
            solve_cell(dc, sig, q, X[d][0], X[d][1], Y0, Y1, f, xo0, xo1, yo0, yo1);
          Y[d][0] = yo0;
          Y[d][1] = yo1;
          X[d][0] = ok ? xo0 : X[d][0];
          X[d][1] = ok ? xo1 : X[d][1];
          const double wv = ok ? dc.w : 0.0;
          acc0 = fma(wv, f[0], acc0);
          acc1 = fma(wv, f[1], acc1);
          acc2 = fma(wv, f[2], acc2);
          acc3 = fma(wv, f[3], acc3);
          if (KIN && ok) {
            // kinetic store: f of every original direction of this slot
            const int ix = qx ? nx - 1 - x : x;
            const long pc = (long)(qy ? ny - 1 - yr : yr) * nx + ix;
            const double2 v01 = make_double2(f[0], sx * f[1]), v23 = make_double2(sy * f[2], sx * sy * f[3]);
            const DirConst& dcf = sm.tab[warp * D + d];
            if (dcf.dir0 >= 0) {
              double* o = a.fout + ((long)s * a.nv + dcf.dir0) * nd + 4 * pc;
              *reinterpret_cast<double2*>(o) = v01;
              *reinterpret_cast<double2*>(o + 2) = v23;
            }
            if (dcf.dir1 >= 0) {
              double* o = a.fout + ((long)s * a.nv + dcf.dir1) * nd + 4 * pc;
              *reinterpret_cast<double2*>(o) = v01;
              *reinterpret_cast<double2*>(o + 2) = v23;
            }
          }
        }
        if (lane == 31 && ok && band + 1 < nbands) {
#pragma unroll
          for (int d = 0; d < D; ++d) __stcg(yabove + (long)x * ndir + warp * D + d, make_double2(Y[d][0], Y[d][1]));
        }
        double* rr = sm.red + ((kk * kNW + warp) * 4) * 32 + lane;
        rr[0] = acc0;
        rr[32] = acc1;
        rr[64] = acc2;
        rr[96] = acc3;
      };
      if (band_full && k0 >= 31 && k0 + kC <= nx) {
#pragma unroll kKU
        for (int kk = 0; kk < kC; ++kk) step(std::false_type{}, kk);
      } else {
#pragma unroll 1
        for (int kk = 0; kk < kC; ++kk) step(std::true_type{}, kk);
      }
      // the next chunk's staged data: bulk copies complete on the mbarrier
      // (phase parity = chunk index), cp.async copies on the thread's group
      if (bulk) {
        if (k0 + kC < nx) {
          mbar_wait(sm.bar, ((k0 + kC) / kC) & 1);
#ifndef RTE_SWEEP_NODISCARD
          // The band-below traces of the chunk just staged are dead in global
          // memory (one producer, one consumer per sweep): drop their L2 lines
          // instead of letting them be written back to DRAM (sweep DRAM traffic
          // 8.8 -> 7.6 GB at C5; about half of the trace lines are still
          // written back before the band above gets to them).
          if (band > 0 && warp == kNW - 1) {
            const char* base = reinterpret_cast<const char*>(ybelow + (long)(k0 + kC) * ndir);
            for (int o = lane * 128; o < (int)(kC * ndir * sizeof(double2)); o += 32 * 128)
              asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + o) : "memory");
          }
#endif
        }
      } else {
        cp_async_wait_all();
      }
      __syncthreads();
      // fixed-order reduction over the warps (direction subgroups) of the chunk
      {
        const int t = threadIdx.x;
        if (t < kC * 32) {
          const int kk = t >> 5, ln = t & 31;
          const int x = k0 + kk - ln;
          const int yy = band * 32 + ln;
          if (x >= 0 && x < nx && yy < ny) {
            double v0 = 0, v1 = 0, v2 = 0, v3 = 0;
            for (int w = 0; w < kNW; ++w) {
              const double* rr = sm.red + ((kk * kNW + w) * 4) * 32 + ln;
              v0 += rr[0];
              v1 += rr[32];
              v2 += rr[64];
              v3 += rr[96];
            }
            const int ix = qx ? nx - 1 - x : x;
            const int iyy = qy ? ny - 1 - yy : yy;
            double* o = part + 4 * ((long)iyy * nx + ix);
            __stcs(reinterpret_cast<double2*>(o), make_double2(v0, sx * v1));
            __stcs(reinterpret_cast<double2*>(o + 2), make_double2(sy * v2, sx * sy * v3));
          }
        }
      }
      if (k0 + kC < nx) {
        if (bulk)
          convert_chunk<FULL, true>(a, sm, k0 + kC, band, sx, sy, s, qx, qy);
        else
          convert_chunk<FULL, false>(a, sm, k0 + kC, band, sx, sy, s, qx, qy);
      }
      ys ^= 1;
      if (threadIdx.x == 0 && band + 1 < nbands &&
          (kPub == 1 || (k0 / kC) % kPub == kPub - 1 || k0 + kC >= nsteps)) {
        DBG_T0();
        // the release store orders the CTA's top traces (stored before the
        // chunk barrier above) before the new progress value
#ifdef RTE_SWEEP_DOUBLE_FENCE
        __threadfence();
#endif
        const int avail = min(nx, max(0, k0 + kC - 31));
        st_release(progress + ibase * nbands + band, (unsigned)avail);
        DBG_ADD(5);
      }
    }
#ifdef RTE_SWEEP_DEBUG_WAIT
    if (threadIdx.x == 0) {
      atomicAdd(&g_dbg[2], (unsigned long long)(clock64() - dbg_item0));
      atomicAdd(&g_dbg[3], 1ull);
    }
#endif
    if (bulk && threadIdx.x == 0) mbar_inval(sm.bar);  // every phase was waited for before the last chunk barrier
    __syncthreads();
  }
}

template <int D>
size_t smem_bytes() {  // NOLINT
  return sizeof(double) * ((size_t)kC * kNW * 4 * 32 + (size_t)kRC * kRP + (size_t)kStageDoubles +
                           (size_t)2 * kC * kNW * D * 2) +
         sizeof(DirConst) * kNW * D;
}

template <int D, bool KIN, bool FULL>
void launch_d(const Sweep2DArgs& a, cudaStream_t st) {
  const size_t smem = smem_bytes<D>();
  static int max_ctas = -1;
  if (max_ctas < 0) {
    RTE_CUDA(cudaFuncSetAttribute(sweep2d_kernel<D, KIN, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    int per_sm = 0, dev = 0, sms = 0;
    RTE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep2d_kernel<D, KIN, FULL>, kNW * 32, smem));
    RTE_CUDA(cudaGetDevice(&dev));
    RTE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    max_ctas = std::max(1, per_sm) * sms;
  }
  const int nbands = (a.ny + 31) / 32;
  const long total = (long)nbands * a.S * 4 * a.groups;
  const int grid = (int)std::min<long>(total, max_ctas);
  sweep2d_kernel<D, KIN, FULL><<<grid, kNW * 32, smem, st>>>(a);
  RTE_CUDA(cudaGetLastError());
#ifdef RTE_SWEEP_DEBUG_WAIT
  {
    unsigned long long h[8];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_dbg, sizeof(h));
    fprintf(stderr, "sweep dbg: items %llu item-cycles %.3e prologue-wait %.3e (%.1f%%) chunk-wait %.3e (%.1f%%) polls/item %.1f publish %.3e (%.1f%%)\n",
            h[3], (double)h[2], (double)h[0], 100.0 * h[0] / h[2], (double)h[1], 100.0 * h[1] / h[2], (double)h[4] / h[3],
            (double)h[5], 100.0 * h[5] / h[2]);
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
  }
#endif
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

template <bool FULL>
void launch_full(const Sweep2DArgs& a, cudaStream_t st, int dpc) {
  if (a.fout) {
    switch (dpc) {
      case 1: return launch_d<1, true, FULL>(a, st);
      case 2: return launch_d<2, true, FULL>(a, st);
      case 4: return launch_d<4, true, FULL>(a, st);
      case 8: return launch_d<8, true, FULL>(a, st);
      default: throw Error(RTE_ERR_UNSUPPORTED, "sweep2d: unsupported direction grouping");
    }
  }
  switch (dpc) {
    case 1: return launch_d<1, false, FULL>(a, st);
    case 2: return launch_d<2, false, FULL>(a, st);
    case 4: return launch_d<4, false, FULL>(a, st);
    case 8: return launch_d<8, false, FULL>(a, st);
    default: throw Error(RTE_ERR_UNSUPPORTED, "sweep2d: unsupported direction grouping");
  }
}

void launch_sweep2d(const Sweep2DArgs& a, cudaStream_t st) {
  // the staging copies (cp.async.bulk / 16-byte cp.async) need 16-byte aligned vectors
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  RTE_REQUIRE(aligned(a.rho) && aligned(a.g) && aligned(a.sig_t) && aligned(a.sig_s), RTE_ERR_INVALID,
              "sweep2d: device vectors must be 16-byte aligned");
  const int dpc = a.nq_pad / a.groups / kNW;  // directions per lane
  if (a.mt_blk)
    launch_full<true>(a, st, dpc);
  else
    launch_full<false>(a, st, dpc);
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
