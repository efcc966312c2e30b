// pod.cu -- K7: offline POD and Galerkin projections on the device.
//
// Replaces pod_truncate (pod.cpp:141-304: dgesdd in-core or out-of-core TSQR)
// and build_reduced_model (reduced_model.cpp:106-199).
//
// POD: repeated (shifted) CholeskyQR (Fukaya, Kannan, Nakatsukasa, Yamamoto,
// Yanagisawa 2020): shifted passes until the basis is well conditioned, then
// CholeskyQR2, so small singular values keep the accuracy the reference's
// Householder/SVD path gives, also past 1/u (a plain Gram eigen-decomposition
// would square the condition number).  The only O(m) work -- the Gram products
// F^T F and the right-multiplications F R^{-1}, Q W -- runs on the device
// with deterministic two-stage reductions; the n x n factors (n <= 128)
// are handled on the host: Cholesky and a one-sided Jacobi SVD of R (high
// relative accuracy).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "rte_internal.cuh"
#include <cstdlib>

namespace rte {
namespace {

constexpr int TT = 32;        // output tile
constexpr int RCH = 32;       // rows per smem stage
constexpr int kRowChunk = 8192;

// partial[chunk][tile] of C = A^T B (A: m x p, B: m x q, column-major, ld = m)
__global__ void k_gram_partial(long m, int p, int q, const double* __restrict__ A, const double* __restrict__ B,
                               double* __restrict__ part) {
  __shared__ double sa[RCH][TT + 1], sb[RCH][TT + 1];
  const int tiles_q = (q + TT - 1) / TT;
  const int ti = blockIdx.y / tiles_q, tj = blockIdx.y % tiles_q;
  const long r0 = (long)blockIdx.x * kRowChunk;
  const long r1 = min(m, r0 + kRowChunk);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads, 4 outputs each
  double acc[4] = {0, 0, 0, 0};
  for (long rb = r0; rb < r1; rb += RCH) {
    for (int e = threadIdx.x; e < RCH * TT; e += blockDim.x) {
      const int rr = e % RCH, cc = e / RCH;
      const long row = rb + rr;
      const int ca = ti * TT + cc, cb = tj * TT + cc;
      sa[rr][cc] = (row < r1 && ca < p) ? A[(long)ca * m + row] : 0.0;
      sb[rr][cc] = (row < r1 && cb < q) ? B[(long)cb * m + row] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < RCH; ++rr) {
      const double bv = sb[rr][tx];
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = fma(sa[rr][ty * 4 + k], bv, acc[k]);
    }
    __syncthreads();
  }
  double* o = part + ((long)blockIdx.x * gridDim.y + blockIdx.y) * TT * TT;
#pragma unroll
  for (int k = 0; k < 4; ++k) o[(ty * 4 + k) * TT + tx] = acc[k];
}

__global__ void k_gram_reduce(int nchunks, int p, int q, const double* __restrict__ part, double* __restrict__ C) {
  const int tiles_q = (q + TT - 1) / TT;
  const int ntiles = gridDim.x;
  const int tile = blockIdx.x;
  const int ti = tile / tiles_q, tj = tile % tiles_q;
  for (int e = threadIdx.x; e < TT * TT; e += blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < nchunks; ++c) v += part[((long)c * ntiles + tile) * TT * TT + e];
    const int i = ti * TT + e / TT, j = tj * TT + e % TT;
    if (i < p && j < q) C[(long)j * p + i] = v;  // column-major p x q
  }
}

// Y (m x k) = A (m x n) M (n x k), column-major; M in shared memory
__global__ void k_rmul(long m, int n, int k, const double* __restrict__ A, const double* __restrict__ M,
                       double* __restrict__ Y) {
  extern __shared__ double sm[];
  for (int e = threadIdx.x; e < n * k; e += blockDim.x) sm[e] = M[e];
  __syncthreads();
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  for (int c0 = 0; c0 < k; c0 += 16) {
    double acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.0;
    for (int l = 0; l < n; ++l) {
      const double a = A[(long)l * m + row];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c0 + c < k) acc[c] = fma(a, sm[(long)(c0 + c) * n + l], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c0 + c < k) Y[(long)(c0 + c) * m + row] = acc[c];
  }
}

// ---- blocked kernels for p, q, n, k <= 128 (all POD shapes of the configs) ----
// One CTA reads each row chunk of A and B once and accumulates the whole
// p x q product (16 x 16 threads, 8 x 8 outputs each, columns strided by 16
// so shared-memory reads are conflict-free).  CUDA-core FP64 version, kept as
// the RTE_POD_DMMA=0 comparison: 21.5 ms for the C4 correction matrix
// (8.4M x 120) against 9.0 ms for the tensor-core kernel k_gram_dmma below.
constexpr int kW = 128;         // max columns
constexpr int kGR = 16;         // rows per shared-memory stage
constexpr int kGChunk = 16384;  // rows per CTA

__global__ void __launch_bounds__(512) k_gram_wide(long m, int p, int q, const double* __restrict__ A,
                                                   const double* __restrict__ B, double* __restrict__ part) {
  // 32 x 16 threads, 4 x 8 outputs each (rows ty + 32 a, columns tx + 16 b);
  // the next stage's rows are prefetched into registers while this one computes
  extern __shared__ double gsm[];
  auto sa = reinterpret_cast<double (*)[kGR][kW]>(gsm);                // [2][kGR][kW]
  auto sb = reinterpret_cast<double (*)[kGR][kW]>(gsm + 2 * kGR * kW);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long r0 = (long)blockIdx.x * kGChunk;
  const long r1 = min(m, r0 + kGChunk);
  double acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  constexpr int kPer = kGR * kW / 512;  // elements per thread per matrix and stage
  double ra[kPer], rb_[kPer];
  auto load = [&](long rb) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + t * 512;
      const int rr = e % kGR, cc = e / kGR;
      const long row = rb + rr;
      ra[t] = (row < r1 && cc < p) ? __ldg(A + (long)cc * m + row) : 0.0;
      rb_[t] = (row < r1 && cc < q) ? __ldg(B + (long)cc * m + row) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + t * 512;
      sa[buf][e % kGR][e / kGR] = ra[t];
      sb[buf][e % kGR][e / kGR] = rb_[t];
    }
  };
  int buf = 0;
  load(r0);
  store(0);
  __syncthreads();
  for (long rb = r0; rb < r1; rb += kGR) {
    const bool more = rb + kGR < r1;
    if (more) load(rb + kGR);
#pragma unroll 4
    for (int rr = 0; rr < kGR; ++rr) {
      double va[4], vb[8];
#pragma unroll
      for (int a = 0; a < 4; ++a) va[a] = sa[buf][rr][ty + 32 * a];
#pragma unroll
      for (int b = 0; b < 8; ++b) vb[b] = sb[buf][rr][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fma(va[a], vb[b], acc[a][b]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  double* o = part + (long)blockIdx.x * kW * kW;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) o[(ty + 32 * a) * kW + tx + 16 * b] = acc[a][b];
}

// ---- FP64 tensor-core Gram (DMMA: mma.sync m8n8k4 f64) --------------------
// C = A^T B for p, q <= 128: a CTA of 16 warps (4 x 4) accumulates the whole
// 128 x 128 product of its row range; each warp owns a 32 x 32 block as 4 x 4
// m8n8 accumulator tiles (32 doubles per lane) and per 4 rows issues 16 DMMAs
// from 8 fragment loads (the CUDA-core version needs 12 shared-memory loads
// per 32 DFMAs and reached a third of the FP64 peak).  Rows are staged column
// by column (the matrices are column-major, rows contiguous) with a pitch of
// kDR + 4 doubles, which makes the (row, column) fragment reads of every
// half-warp hit 16 distinct banks.  Partial products per CTA, summed by
// k_gram_wide_reduce in a fixed order (deterministic).
constexpr int kDR = 32;       // rows per shared-memory stage
constexpr int kDP = kDR + 4;  // staged column pitch in doubles

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(512, 1) k_gram_dmma(long m, long rows_per_cta, int p, int q,
                                                      const double* __restrict__ A, const double* __restrict__ B,
                                                      double* __restrict__ part) {
  extern __shared__ double gsm[];
  double* sa = gsm;                  // [2][kW][kDP]
  double* sb = gsm + 2 * kW * kDP;   // [2][kW][kDP]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wi = warp >> 2, wj = warp & 3, g = lane >> 2, t4 = lane & 3;
  const long r0 = (long)blockIdx.x * rows_per_cta;
  const long r1 = min(m, r0 + rows_per_cta);
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  constexpr int kPer = kDR * kW / 512;  // elements per thread per matrix and stage
  double ra[kPer], rb_[kPer];
  auto load = [&](long rb) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + t * 512;
      const int rr = e % kDR, cc = e / kDR;  // a warp reads kDR consecutive rows of one column
      const long row = rb + rr;
      ra[t] = (row < r1 && cc < p) ? __ldg(A + (long)cc * m + row) : 0.0;
      rb_[t] = (row < r1 && cc < q) ? __ldg(B + (long)cc * m + row) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + t * 512;
      sa[(buf * kW + e / kDR) * kDP + e % kDR] = ra[t];
      sb[(buf * kW + e / kDR) * kDP + e % kDR] = rb_[t];
    }
  };
  int buf = 0;
  load(r0);
  store(0);
  __syncthreads();
  for (long rb = r0; rb < r1; rb += kDR) {
    const bool more = rb + kDR < r1;
    if (more) load(rb + kDR);
    const double* pa = sa + (buf * kW + 32 * wi + g) * kDP + t4;
    const double* pb = sb + (buf * kW + 32 * wj + g) * kDP + t4;
#pragma unroll
    for (int kk = 0; kk < kDR / 4; ++kk) {
      double va[4], vb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) va[a] = pa[8 * a * kDP + 4 * kk];
#pragma unroll
      for (int b = 0; b < 4; ++b) vb[b] = pb[8 * b * kDP + 4 * kk];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], va[a], vb[b]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  double* o = part + (long)blockIdx.x * kW * kW;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = 32 * wi + 8 * a + g, j = 32 * wj + 8 * b + 2 * t4;
      *reinterpret_cast<double2*>(o + i * kW + j) = make_double2(acc[a][b][0], acc[a][b][1]);
    }
}

__global__ void k_gram_wide_reduce(int nchunks, int p, int q, const double* __restrict__ part,
                                   double* __restrict__ C) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= kW * kW) return;
  const int i = e / kW, j = e % kW;
  if (i >= p || j >= q) return;
  double v = 0.0;
  for (int c = 0; c < nchunks; ++c) v += part[(long)c * kW * kW + e];
  C[(long)j * p + i] = v;  // column-major p x q
}

// Y (m x k) = A (m x n) M (n x k): 64-row tiles of A (transposed into shared
// memory) times M held in shared memory; 16 x 16 threads, 4 rows x 8 columns each.
__global__ void __launch_bounds__(256) k_rmul_wide(long m, int n, int k, const double* __restrict__ A,
                                                   const double* __restrict__ M, double* __restrict__ Y) {
  extern __shared__ double sm[];
  double* Ms = sm;                // [n][kW] row-major
  double* At = sm + n * kW;       // [n][64]
  for (int e = threadIdx.x; e < n * kW; e += blockDim.x) {
    const int l = e / kW, j = e % kW;
    Ms[e] = j < k ? M[(long)j * n + l] : 0.0;
  }
  const int tr = threadIdx.x & 15, tc = threadIdx.x >> 4;
  for (long rb = (long)blockIdx.x * 64; rb < m; rb += (long)gridDim.x * 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < n * 64; e += blockDim.x) {
      const int l = e / 64, rr = e % 64;
      const long row = rb + rr;
      At[e] = row < m ? A[(long)l * m + row] : 0.0;
    }
    __syncthreads();
    double acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
#pragma unroll 2
    for (int l = 0; l < n; ++l) {
      double va[4], vb[8];
#pragma unroll
      for (int a = 0; a < 4; ++a) va[a] = At[l * 64 + tr + 16 * a];
#pragma unroll
      for (int b = 0; b < 8; ++b) vb[b] = Ms[l * kW + tc + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fma(va[a], vb[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const long row = rb + tr + 16 * a;
      if (row >= m) continue;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int j = tc + 16 * b;
        if (j < k) Y[(long)j * m + row] = acc[a][b];
      }
    }
  }
}

// Y (m x k) = A (m x n) M (n x k) on the FP64 tensor cores, n, k <= 128:
// 64-row tiles; M (zero-padded to 128 columns) stays in shared memory, the A
// tile is staged column by column (the next tile prefetched into registers
// while this one multiplies); 16 warps = 2 row blocks x 8 column blocks, each
// 32 rows x 16 columns (4 x 2 m8n8 tiles: 8 DMMAs per 6 fragment loads).  The
// product tile goes back through shared memory so the global stores are
// whole 512-byte column segments.
constexpr int kRT = 64;        // rows per tile
constexpr int kRPA = kRT + 4;  // pitch of a staged A / Y column (conflict-free fragment reads)
constexpr int kRPM = kW + 4;   // pitch of a row of M

__global__ void __launch_bounds__(512, 1) k_rmul_dmma(long m, int n, int k, const double* __restrict__ A,
                                                      const double* __restrict__ M, double* __restrict__ Y) {
  extern __shared__ double sm[];
  double* Ms = sm;               // [kW][kRPM]: M[l][j], zero outside n x k
  double* At = sm + kW * kRPM;   // [kW][kRPA]: A tile by column, then the Y tile by column
  for (int e = threadIdx.x; e < kW * kW; e += blockDim.x) {
    const int l = e / kW, j = e % kW;
    Ms[l * kRPM + j] = (l < n && j < k) ? M[(long)j * n + l] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp & 1, wc = warp >> 1, g = lane >> 2, t4 = lane & 3;
  const int n4 = (n + 3) / 4;
  constexpr int kPer = kRT * kW / 512;
  double ra[kPer];
  auto load = [&](long rb) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + t * 512;
      const int rr = e % kRT, l = e / kRT;
      const long row = rb + rr;
      ra[t] = (row < m && l < n) ? __ldg(A + (long)l * m + row) : 0.0;
    }
  };
  long rb = (long)blockIdx.x * kRT;
  if (rb < m) load(rb);
  for (; rb < m; rb += (long)gridDim.x * kRT) {
    __syncthreads();  // the previous tile's Y columns have been written out
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + t * 512;
      At[(e / kRT) * kRPA + e % kRT] = ra[t];
    }
    __syncthreads();
    const long nxt = rb + (long)gridDim.x * kRT;
    if (nxt < m) load(nxt);
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const double* pa = At + t4 * kRPA + 32 * wr + g;
    const double* pb = Ms + t4 * kRPM + 16 * wc + g;
    for (int kk = 0; kk < n4; ++kk) {
      double va[4], vb[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) va[a] = pa[4 * kk * kRPA + 8 * a];
#pragma unroll
      for (int b = 0; b < 2; ++b) vb[b] = pb[4 * kk * kRPM + 8 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma884(acc[a][b][0], acc[a][b][1], va[a], vb[b]);
    }
    __syncthreads();  // every warp is done reading the A tile
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int row = 32 * wr + 8 * a + g, j = 16 * wc + 8 * b + 2 * t4;
        At[j * kRPA + row] = acc[a][b][0];
        At[(j + 1) * kRPA + row] = acc[a][b][1];
      }
    __syncthreads();
    for (int e = threadIdx.x; e < kRT * k; e += blockDim.x) {
      const int rr = e % kRT, j = e / kRT;
      const long row = rb + rr;
      if (row < m) Y[(long)j * m + row] = At[j * kRPA + rr];
    }
  }
}

// u_rho / u_iso: out[c][i] = sum_j wj U[c][j][i]
__global__ void k_block_sum(int r, int nv, long nd, const double* __restrict__ U, const double* __restrict__ w,
                            double* __restrict__ out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)r * nd) return;
  const long c = t / nd, i = t - c * nd;
  double v = 0.0;
  for (int j = 0; j < nv; ++j) v += (w ? w[j] : 1.0) * U[(c * nv + j) * nd + i];
  out[t] = v;
}

void gram(long m, int p, int q, const double* A, const double* B, double* C_dev, cudaStream_t st) {
  static const bool use_dmma = !(std::getenv("RTE_POD_DMMA") && std::atoi(std::getenv("RTE_POD_DMMA")) == 0);
  if (p <= kW && q <= kW && use_dmma) {
    // row ranges sized so the CTAs fill whole waves of the device (one CTA per SM)
    int sms = 148, dev = 0;
    RTE_CUDA(cudaGetDevice(&dev));
    RTE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long waves = std::max<long>(1, (m + (long)sms * 8192 - 1) / ((long)sms * 8192));
    long rows = (m + sms * waves - 1) / (sms * waves);
    rows = std::max<long>(kDR, (rows + kDR - 1) / kDR * kDR);
    const int nch = (int)((m + rows - 1) / rows);
    DBuf<double> part;
    part.alloc((size_t)nch * kW * kW);
    const int gsmem = (int)(sizeof(double) * 4 * kW * kDP);
    static bool dcfg = false;
    if (!dcfg) {
      RTE_CUDA(cudaFuncSetAttribute(k_gram_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, gsmem));
      dcfg = true;
    }
    k_gram_dmma<<<nch, 512, gsmem, st>>>(m, rows, p, q, A, B, part.p);
    k_gram_wide_reduce<<<kW * kW / 256, 256, 0, st>>>(nch, p, q, part.p, C_dev);
    RTE_CUDA(cudaGetLastError());
    RTE_CUDA(cudaStreamSynchronize(st));
    return;
  }
  if (p <= kW && q <= kW) {
    const int nch = (int)((m + kGChunk - 1) / kGChunk);
    DBuf<double> part;
    part.alloc((size_t)nch * kW * kW);
    const int gsmem = (int)(sizeof(double) * 4 * kGR * kW);
    static bool gcfg = false;
    if (!gcfg) {
      RTE_CUDA(cudaFuncSetAttribute(k_gram_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, gsmem));
      gcfg = true;
    }
    k_gram_wide<<<nch, 512, gsmem, st>>>(m, p, q, A, B, part.p);
    k_gram_wide_reduce<<<kW * kW / 256, 256, 0, st>>>(nch, p, q, part.p, C_dev);
    RTE_CUDA(cudaGetLastError());
    RTE_CUDA(cudaStreamSynchronize(st));
    return;
  }
  const int tiles = ((p + TT - 1) / TT) * ((q + TT - 1) / TT);
  const int nch = (int)((m + kRowChunk - 1) / kRowChunk);
  DBuf<double> part;
  part.alloc((size_t)nch * tiles * TT * TT);
  k_gram_partial<<<dim3(nch, tiles), 256, 0, st>>>(m, p, q, A, B, part.p);
  k_gram_reduce<<<tiles, 256, 0, st>>>(nch, p, q, part.p, C_dev);
  RTE_CUDA(cudaGetLastError());
  RTE_CUDA(cudaStreamSynchronize(st));
}

std::vector<double> gram_host(long m, int p, int q, const double* A, const double* B, cudaStream_t st) {
  DBuf<double> C;
  C.alloc((size_t)p * q);
  gram(m, p, q, A, B, C.p, st);
  std::vector<double> h((size_t)p * q);
  RTE_CUDA(cudaMemcpy(h.data(), C.p, sizeof(double) * p * q, cudaMemcpyDeviceToHost));
  return h;
}

void rmul(long m, int n, int k, const double* A, const std::vector<double>& M, double* Y, cudaStream_t st) {
  DBuf<double> dM;
  dM.upload(M.data(), M.size());
  static const bool use_dmma = !(std::getenv("RTE_POD_DMMA") && std::atoi(std::getenv("RTE_POD_DMMA")) == 0);
  if (n <= kW && k <= kW && use_dmma) {
    const size_t smem3 = sizeof(double) * ((size_t)kW * kRPM + (size_t)kW * kRPA);
    static bool cfg3 = false;
    if (!cfg3) {
      RTE_CUDA(cudaFuncSetAttribute(k_rmul_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
      cfg3 = true;
    }
    int sms = 148, dev = 0;
    RTE_CUDA(cudaGetDevice(&dev));
    RTE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long tiles = (m + kRT - 1) / kRT;
    k_rmul_dmma<<<(int)std::min<long>(tiles, (long)sms), 512, smem3, st>>>(m, n, k, A, dM.p, Y);
    RTE_CUDA(cudaGetLastError());
    RTE_CUDA(cudaStreamSynchronize(st));
    return;
  }
  if (n <= kW && k <= kW) {
    const size_t smem2 = sizeof(double) * ((size_t)n * kW + (size_t)n * 64);
    static bool cfg2 = false;
    if (!cfg2) {
      RTE_CUDA(cudaFuncSetAttribute(k_rmul_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      cfg2 = true;
    }
    int sms = 148, dev = 0;
    RTE_CUDA(cudaGetDevice(&dev));
    RTE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long tiles = (m + 63) / 64;
    k_rmul_wide<<<(int)std::min<long>(tiles, (long)sms * 2), 256, smem2, st>>>(m, n, k, A, dM.p, Y);
    RTE_CUDA(cudaGetLastError());
    RTE_CUDA(cudaStreamSynchronize(st));
    return;
  }
  const size_t smem = sizeof(double) * n * k;
  RTE_REQUIRE(smem <= 200 * 1024, RTE_ERR_UNSUPPORTED, "pod: too many columns");
  static bool cfg = false;
  if (!cfg) {
    RTE_CUDA(cudaFuncSetAttribute(k_rmul, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cfg = true;
  }
  k_rmul<<<(int)((m + 127) / 128), 128, smem, st>>>(m, n, k, A, dM.p, Y);
  RTE_CUDA(cudaGetLastError());
  RTE_CUDA(cudaStreamSynchronize(st));
}

// ---- host dense linear algebra (column-major n x n) ----------------------

// upper Cholesky G = R^T R; false if not positive definite
bool cholesky_upper(const std::vector<double>& G, int n, std::vector<double>& R) {
  R.assign((size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = G[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= R[(size_t)j * n + k] * R[(size_t)j * n + k];
    if (!(d > 0)) return false;
    const double rjj = std::sqrt(d);
    R[(size_t)j * n + j] = rjj;
    for (int i = j + 1; i < n; ++i) {
      double v = G[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) v -= R[(size_t)j * n + k] * R[(size_t)i * n + k];
      R[(size_t)i * n + j] = v / rjj;  // R(j, i) stored column-major at [i*n + j]
    }
  }
  return true;
}

// inverse of upper triangular R (column-major)
std::vector<double> inv_upper(const std::vector<double>& R, int n) {
  std::vector<double> X((size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    X[(size_t)j * n + j] = 1.0 / R[(size_t)j * n + j];
    for (int i = j - 1; i >= 0; --i) {
      double v = 0.0;
      for (int k = i + 1; k <= j; ++k) v += R[(size_t)k * n + i] * X[(size_t)j * n + k];
      X[(size_t)j * n + i] = -v / R[(size_t)i * n + i];
    }
  }
  return X;
}

std::vector<double> matmul_cm(const std::vector<double>& A, const std::vector<double>& B, int n) {
  std::vector<double> C((size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const double b = B[(size_t)j * n + k];
      if (b == 0) continue;
      for (int i = 0; i < n; ++i) C[(size_t)j * n + i] += A[(size_t)k * n + i] * b;
    }
  return C;
}

// One-sided Jacobi SVD of R (n x n, column-major): R = W diag(s) V^T.
// Applied to A = R^T: A J has orthogonal columns (norms = s), so the left
// singular vectors of R are the accumulated rotations J.
void jacobi_svd_left(const std::vector<double>& R, int n, std::vector<double>& s, std::vector<double>& W) {
  std::vector<double> A((size_t)n * n), J((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) A[(size_t)j * n + i] = R[(size_t)i * n + j];  // A = R^T
  for (int i = 0; i < n; ++i) J[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < n; ++i) {
          const double ap = A[(size_t)p * n + i], aq = A[(size_t)q * n + i];
          alpha += ap * ap;
          beta += aq * aq;
          gamma += ap * aq;
        }
        if (gamma == 0.0) continue;
        const double c0 = std::fabs(gamma) / std::sqrt(alpha * beta);
        off = std::max(off, c0);
        if (c0 < 1e-16) continue;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < n; ++i) {
          const double ap = A[(size_t)p * n + i], aq = A[(size_t)q * n + i];
          A[(size_t)p * n + i] = c * ap - sn * aq;
          A[(size_t)q * n + i] = sn * ap + c * aq;
          const double jp = J[(size_t)p * n + i], jq = J[(size_t)q * n + i];
          J[(size_t)p * n + i] = c * jp - sn * jq;
          J[(size_t)q * n + i] = sn * jp + c * jq;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> nrm(n);
  for (int j = 0; j < n; ++j) {
    double v = 0;
    for (int i = 0; i < n; ++i) v += A[(size_t)j * n + i] * A[(size_t)j * n + i];
    nrm[j] = std::sqrt(v);
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return nrm[a] > nrm[b]; });
  s.resize(n);
  W.assign((size_t)n * n, 0.0);
  for (int k = 0; k < n; ++k) {
    s[k] = nrm[ord[k]];
    for (int i = 0; i < n; ++i) W[(size_t)k * n + i] = J[(size_t)ord[k] * n + i];
  }
}

__global__ void k_sub(long n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) o[t] = a[t] - b[t];
}

}  // namespace

// Snapshot matrices (PrimarySource / CorrectionSource, snapshots.cpp:316-376):
// kind 0 = converged f of converged samples; kind 1 = f_conv - f^(l),
// l <= min(n_iter, window), converged samples only.  Returns column count.
int snapshot_columns(int S, int window, long kdim, const double* f_iter, const double* f_conv, const int* n_iter,
                     const int* conv, int kind, int window_limit, double* out, cudaStream_t st) {
  int col = 0;
  for (int s = 0; s < S; ++s) {
    if (!conv[s]) continue;
    if (kind == 0) {
      if (out) RTE_CUDA(cudaMemcpyAsync(out + (long)col * kdim, f_conv + (long)s * kdim, sizeof(double) * kdim,
                                        cudaMemcpyDeviceToDevice, st));
      ++col;
    } else {
      const int w = std::min(std::min(n_iter[s], window), window_limit);
      for (int l = 1; l <= w; ++l) {
        if (out)
          k_sub<<<(int)((kdim + 255) / 256), 256, 0, st>>>(kdim, f_conv + (long)s * kdim,
                                                           f_iter + ((long)s * window + l - 1) * kdim,
                                                           out + (long)col * kdim);
        ++col;
      }
    }
  }
  RTE_CUDA(cudaGetLastError());
  RTE_CUDA(cudaStreamSynchronize(st));
  return col;
}

// F: m x n column-major on device (m >= n).  sigma (n values) to host; the
// first rank_max left singular vectors to U (m x rank_max).
__global__ void k_transpose(long m, int n, const double* __restrict__ A, double* __restrict__ T) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * n) return;
  const long i = t % m, j = t / m;  // A(i, j), column-major m x n -> T(j, i), n x m
  T[i * n + j] = A[t];
}

// R (n x n, column-major) -> F = Q R with Q (m x n) orthonormal in *q_out
// (one of the two work buffers)
static std::vector<double> cholesky_qr(long m, int n, const double* F, DBuf<double>& Q1, DBuf<double>& Q2,
                                       const double** q_out, cudaStream_t st);

void pod(long m, int n, const double* F, int rank_max, double* U, double* sigma, cudaStream_t st) {
  RTE_REQUIRE(n >= 1 && n <= 128, RTE_ERR_UNSUPPORTED, "pod: 1..128 snapshot columns supported");
  RTE_REQUIRE(m >= 1, RTE_ERR_INVALID, "pod: empty snapshot matrix");
  RTE_REQUIRE(rank_max >= 0 && rank_max <= std::min<long>(m, n), RTE_ERR_INVALID, "pod: rank_max out of range");
  if (m < n) {
    // wide (more snapshots than unknowns, test_pod.cpp:183-193): F^T = Q R,
    // so F = R^T Q^T and the left singular vectors of F are those of R^T (m x m)
    DBuf<double> FT, Q1, Q2;
    FT.alloc((size_t)m * n);
    k_transpose<<<(int)((m * n + 255) / 256), 256, 0, st>>>(m, n, F, FT.p);
    RTE_CUDA(cudaGetLastError());
    const double* q = nullptr;
    std::vector<double> R = cholesky_qr(n, (int)m, FT.p, Q1, Q2, &q, st);
    const int k = (int)m;
    std::vector<double> RT((size_t)k * k);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) RT[(size_t)j * k + i] = R[(size_t)i * k + j];
    std::vector<double> s, W;
    jacobi_svd_left(RT, k, s, W);
    for (int i = 0; i < n; ++i) sigma[i] = i < k ? s[i] : 0.0;
    if (rank_max > 0)
      RTE_CUDA(cudaMemcpyAsync(U, W.data(), sizeof(double) * (size_t)k * rank_max, cudaMemcpyHostToDevice, st));
    RTE_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DBuf<double> Q1, Q2;
  const double* src = nullptr;
  std::vector<double> Rtot = cholesky_qr(m, n, F, Q1, Q2, &src, st);
  // F = Q Rtot, Rtot = W diag(s) V^T (one-sided Jacobi: high relative
  // accuracy), so the left singular vectors of F are Q W
  std::vector<double> s, W;
  jacobi_svd_left(Rtot, n, s, W);
  for (int k = 0; k < n; ++k) sigma[k] = s[k];
  if (rank_max > 0) {
    std::vector<double> Wr(W.begin(), W.begin() + (size_t)n * rank_max);
    rmul(m, n, rank_max, src, Wr, U, st);
  }
}

static std::vector<double> cholesky_qr(long m, int n, const double* F, DBuf<double>& Q1, DBuf<double>& Q2,
                                       const double** q_out, cudaStream_t st) {
  // Repeated CholeskyQR: a pass whose Gram is too ill-conditioned for a plain
  // Cholesky (kappa(Q) > 1e7, or breakdown) is shifted (Fukaya et al. 2020:
  // G + s I with s = 11 (m n + n (n + 1)) u ||Q||_F^2), which cuts the
  // condition number by ~sqrt(s) per pass; two plain passes (CholeskyQR2)
  // finish once it is below 1e7.  Snapshot matrices with decaying spectra
  // far past 1/u (the reference's POD KAT, test_pod.cpp:16-36: sigma_k =
  // 10^(-k/2), kappa 3e19) need two shifted passes; well-conditioned ones
  // run CholeskyQR2 directly.
  const double u = 1.1102230246251565e-16;
  Q1.alloc((size_t)m * n);
  Q2.alloc((size_t)m * n);
  std::vector<double> Rtot((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) Rtot[(size_t)i * n + i] = 1.0;
  const double* src = F;
  DBuf<double>* dst = &Q1;
  int plain = 0;
  for (int pass = 0; plain < 2; ++pass) {
    RTE_REQUIRE(pass < 10, RTE_ERR_RUNTIME, "pod: CholeskyQR did not reach an orthonormal basis in 10 passes");
    std::vector<double> G = gram_host(m, n, n, src, src, st);
    double fro2 = 0.0;
    for (int i = 0; i < n; ++i) fro2 += G[(size_t)i * n + i];
    RTE_REQUIRE(fro2 > 0 && std::isfinite(fro2), RTE_ERR_INVALID, "pod: snapshot matrix is zero or not finite");
    std::vector<double> R;
    bool ok = cholesky_upper(G, n, R);
    if (ok) {
      std::vector<double> sv, Wv;
      jacobi_svd_left(R, n, sv, Wv);
      ok = sv[n - 1] > 0 && sv[0] / sv[n - 1] <= 1e7;
    }
    if (ok) {
      ++plain;
    } else {
      plain = 0;
      const double shift = 11.0 * ((double)m * n + (double)n * (n + 1)) * u * fro2;
      for (int i = 0; i < n; ++i) G[(size_t)i * n + i] += shift;
      RTE_REQUIRE(cholesky_upper(G, n, R), RTE_ERR_RUNTIME, "pod: shifted CholeskyQR breakdown");
    }
    rmul(m, n, n, src, inv_upper(R, n), dst->p, st);
    Rtot = matmul_cm(R, Rtot, n);
    src = dst->p;
    dst = dst == &Q1 ? &Q2 : &Q1;
  }
  *q_out = src;
  return Rtot;
}

// build_reduced_model: U (kdim x r) on device, sample 0's discretization.
void build_rom(rte_ctx* ctx, int r, const double* U, const double* b_kin_host, double* u_rho, double* u_iso,
               double* a_r, double* b_r, cudaStream_t st) {
  RTE_REQUIRE(ctx->k_terms > 0, RTE_ERR_INVALID, "build_rom: rte_set_affine first");
  const long nd = ctx->ndof, kdim = (long)ctx->nv * nd;
  const int K = ctx->k_terms;
  DBuf<double> w, tmp;
  w.upload(ctx->w.data(), ctx->nv);
  tmp.alloc((size_t)r * nd);
  k_block_sum<<<(int)((r * nd + 255) / 256), 256, 0, st>>>(r, ctx->nv, nd, U, w.p, tmp.p);
  RTE_CUDA(cudaMemcpy(u_rho, tmp.p, sizeof(double) * r * nd, cudaMemcpyDeviceToHost));
  k_block_sum<<<(int)((r * nd + 255) / 256), 256, 0, st>>>(r, ctx->nv, nd, U, nullptr, tmp.p);
  RTE_CUDA(cudaMemcpy(u_iso, tmp.p, sizeof(double) * r * nd, cudaMemcpyDeviceToHost));
  DBuf<double> bk;
  bk.upload(b_kin_host, kdim);
  std::vector<double> br = gram_host(kdim, r, 1, U, bk.p, st);
  for (int c = 0; c < r; ++c) b_r[c] = br[c];
  DBuf<double> Y;
  Y.alloc((size_t)kdim * r);
  for (int k = 0; k < K; ++k) {
    apply_term_kinetic(ctx, k, r, U, Y.p, st);
    std::vector<double> a = gram_host(kdim, r, r, U, Y.p, st);
    std::copy(a.begin(), a.end(), a_r + (size_t)k * r * r);
  }
  std::vector<double> g = gram_host(kdim, r, r, U, U, st);
  double ortho = 0.0;
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) ortho = std::max(ortho, std::fabs(g[(size_t)j * r + i] - (i == j ? 1.0 : 0.0)));
  RTE_REQUIRE(ortho <= 1e-10, RTE_ERR_RUNTIME,
              "reduced model: basis columns are not orthonormal (defect " + std::to_string(ortho) + ")");
}

}  // namespace rte
