// gmres.cu -- batched restarted (P)GMRES on the device (gmres.cpp:15-124).
//
// Solves (I - L) rho = bbar for every parameter sample, optionally left
// preconditioned with P = I + C Ms (the consistent DSA operator), with the
// reference's algorithm per sample: modified Gram-Schmidt Arnoldi, Givens
// rotations, restart every m inner steps, and a true (preconditioned)
// residual at the start of every cycle that alone declares convergence.
//
// Batched form: each sample runs its own state machine (cycle start / inner
// step / done).  Both a cycle start (r = P(bbar - A rho)) and an inner step
// (w = P A v_j) cost exactly one transport sweep and one DSA solve, so every
// device "step" applies A and P once to a per-sample input vector -- rho or
// v_j -- and the per-sample scalar work (MGS coefficients, Hessenberg,
// rotations, back-substitution) follows in small kernels.  Samples that
// finish are masked.  Reductions are two-stage and fixed-order.
#include <cmath>
#include <cstdlib>
#include <string>
#include <cstring>
#include <vector>

#include "rte_internal.cuh"

namespace rte {

void dsa_apply(rte_ctx* ctx, const double* rhs, double* out, const int* kind, int apply_ms, cudaStream_t st);

namespace {

constexpr int kT = 256;       // threads per block of the vector kernels
enum { PH_START = 0, PH_INNER = 1, PH_DONE = 2 };

struct GmState {
  int phase, j, total, cols, hist_n, converged, steps, cycles;
  int pend_norm;      // V[pend_norm] = W * scale after the scalar step (-1: none)
  int pend_update;    // rho += V[0..pend_update) y (0: none)
  double bnorm, scale, final_res;
};

struct GmArgs {
  int S, m;
  long nd;
  GmState* st;
  double* V;          // [S][m+1][nd]
  double* H;          // [S][m+1][m] row-major (i, j)
  double* g;          // [S][m+1]
  double* cs;         // [S][m]
  double* sn;         // [S][m]
  double* y;          // [S][m]
  double* hist;       // [S][hcap]
  int hcap;
  double tol;
  int max_iters;
  int nblk;
};

__device__ __forceinline__ double* vcol(const GmArgs& a, int s, int k) { return a.V + ((long)s * (a.m + 1) + k) * a.nd; }

// fixed-order per-sample reduction of nblk partials (warp 0), broadcast to the block
__device__ __forceinline__ double reduce_part(const double* __restrict__ part, int s, int nblk) {
  __shared__ double sh;
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 32) v += part[(long)s * nblk + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) sh = v;
  }
  __syncthreads();
  const double r = sh;
  __syncthreads();
  return r;
}

__device__ __forceinline__ void block_part(double v, double* __restrict__ part, int s) {
  __shared__ double red[kT];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(long)s * gridDim.x + blockIdx.x] = red[0];
}

__device__ __forceinline__ double seq_sum(const double* __restrict__ part, int s, int nblk) {
  double v = 0.0;
  for (int b = 0; b < nblk; ++b) v += part[(long)s * nblk + b];
  return v;
}

// input of this step: rho (cycle start) or v_j (inner step); masks for the sweep and the DSA
__global__ void k_gm_stage(GmArgs a, const double* __restrict__ rho, double* __restrict__ U, int* __restrict__ act,
                           int* __restrict__ kind) {
  const int s = blockIdx.y;
  const GmState& g = a.st[s];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    act[s] = g.phase != PH_DONE;
    kind[s] = g.phase != PH_DONE ? KIND_DSA : KIND_IDLE;
  }
  if (g.phase == PH_DONE) return;
  const double* src = g.phase == PH_START ? rho + (long)s * a.nd : vcol(a, s, g.j);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < a.nd; i += (long)gridDim.x * blockDim.x)
    U[(long)s * a.nd + i] = src[i];
}

// Z = A U = U - L U (inner) or bbar - A rho (cycle start); max|Z| for the
// converged-residual report at cycle starts
__global__ void k_gm_z(GmArgs a, const double* __restrict__ U, const double* __restrict__ LU,
                       const double* __restrict__ bbar, double* __restrict__ Z, unsigned long long* __restrict__ zmax) {
  const int s = blockIdx.y;
  const GmState& g = a.st[s];
  if (g.phase == PH_DONE) return;
  const bool start = g.phase == PH_START;
  double m = 0.0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < a.nd; i += (long)gridDim.x * blockDim.x) {
    const long k = (long)s * a.nd + i;
    const double az = U[k] - LU[k];
    const double z = start ? bbar[k] - az : az;
    Z[k] = z;
    m = fmax(m, fabs(z));
  }
  if (start) {
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(zmax + s, (unsigned long long)__double_as_longlong(m));
  }
}

// MGS pass i (launched for i = 0 .. m + 1):
//   i == 0:        W = Z + C (P applied); partial (W, W) at a cycle start, (W, v_0) at an inner step
//   1 <= i <= j+1: h(i-1, j) = reduce(partials of pass i-1); W -= h v_{i-1};
//                  partial (W, v_i) for i <= j, (W, W) for i == j + 1
__global__ void __launch_bounds__(kT) k_gm_pass(GmArgs a, int i, const double* __restrict__ Z,
                                                const double* __restrict__ C, double* __restrict__ W,
                                                const double* __restrict__ part_in, double* __restrict__ part_out) {
  const int s = blockIdx.y;
  const GmState& g = a.st[s];
  if (g.phase == PH_DONE) return;
  const bool start = g.phase == PH_START;
  const int j = g.j;
  if (start ? i > 0 : i > j + 1) return;
  const long base = (long)s * a.nd;
  double coef = 0.0;
  const double* vprev = nullptr;
  if (i > 0) {
    coef = reduce_part(part_in, s, gridDim.x);
    vprev = vcol(a, s, i - 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.H[((long)s * (a.m + 1) + (i - 1)) * a.m + j] = coef;
  }
  const double* vdot = (!start && i <= j) ? vcol(a, s, i) : nullptr;
  double acc = 0.0;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < a.nd; t += (long)gridDim.x * blockDim.x) {
    double w;
    if (i == 0)
      w = C ? Z[base + t] + C[base + t] : Z[base + t];
    else
      w = W[base + t] - coef * vprev[t];
    W[base + t] = w;
    acc = vdot ? fma(w, vdot[t], acc) : fma(w, w, acc);
  }
  block_part(acc, part_out, s);
}

__device__ void push_hist(const GmArgs& a, int s, GmState& g, double v) {
  if (g.hist_n < a.hcap) a.hist[(long)s * a.hcap + g.hist_n] = v;
  ++g.hist_n;
}

// per-sample scalar step (thread per sample): gmres.cpp:50-111
// part0 / part1: partials of the even / odd MGS passes; a sample's last pass
// is pass 0 at a cycle start and pass j + 1 at inner step j
__global__ void k_gm_scalar(GmArgs a, const double* __restrict__ part0, const double* __restrict__ part1,
                            const unsigned long long* __restrict__ zmax, int* __restrict__ n_active) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  GmState& g = a.st[s];
  const double* part = (g.phase == PH_INNER && ((g.j + 1) & 1)) ? part1 : part0;
  g.pend_norm = -1;
  g.pend_update = 0;
  if (g.phase == PH_DONE) return;
  const int m = a.m;
  double* H = a.H + (long)s * (m + 1) * m;
  double* gg = a.g + (long)s * (m + 1);
  double* cs = a.cs + (long)s * m;
  double* sn = a.sn + (long)s * m;
  ++g.steps;
  if (g.phase == PH_START) {
    const double beta = sqrt(seq_sum(part, s, a.nblk));
    const double rel0 = beta / g.bnorm;
    push_hist(a, s, g, rel0);
    if (rel0 <= a.tol) {
      g.converged = 1;
      g.final_res = __longlong_as_double((long long)zmax[s]);
      g.phase = PH_DONE;
      return;
    }
    if (g.total >= a.max_iters) {
      g.phase = PH_DONE;
      return;
    }
    for (int k = 0; k <= m; ++k) gg[k] = 0.0;
    gg[0] = beta;
    g.j = 0;
    g.cols = 0;
    ++g.cycles;
    g.pend_norm = 0;
    g.scale = 1.0 / beta;
    g.phase = PH_INNER;
    atomicAdd(n_active, 1);
    return;
  }
  // inner step j: h(j+1, j) = ||w|| after MGS
  const int j = g.j;
  ++g.total;
  const double hj1 = sqrt(seq_sum(part, s, a.nblk));
  H[(j + 1) * m + j] = hj1;
  const bool breakdown = hj1 <= 1e-300;
  if (!breakdown) {
    g.pend_norm = j + 1;
    g.scale = 1.0 / hj1;
  }
  for (int i = 0; i < j; ++i) {
    const double tmp = cs[i] * H[i * m + j] + sn[i] * H[(i + 1) * m + j];
    H[(i + 1) * m + j] = -sn[i] * H[i * m + j] + cs[i] * H[(i + 1) * m + j];
    H[i * m + j] = tmp;
  }
  const double denom = hypot(H[j * m + j], H[(j + 1) * m + j]);
  cs[j] = denom == 0 ? 1.0 : H[j * m + j] / denom;
  sn[j] = denom == 0 ? 0.0 : H[(j + 1) * m + j] / denom;
  H[j * m + j] = denom;
  H[(j + 1) * m + j] = 0.0;
  gg[j + 1] = -sn[j] * gg[j];
  gg[j] = cs[j] * gg[j];
  g.cols = j + 1;
  const double rel = fabs(gg[j + 1]) / g.bnorm;
  push_hist(a, s, g, rel);
  const bool end = rel <= a.tol || breakdown || j + 1 >= m || g.total >= a.max_iters;
  if (end) {
    // back-substitute R y = g (gmres.cpp:102-110)
    double* y = a.y + (long)s * m;
    for (int i = g.cols - 1; i >= 0; --i) {
      double v = gg[i];
      for (int k = i + 1; k < g.cols; ++k) v -= H[i * m + k] * y[k];
      y[i] = v / H[i * m + i];
    }
    g.pend_update = g.cols;
    g.pend_norm = -1;
    g.phase = PH_START;
  } else {
    g.j = j + 1;
  }
  atomicAdd(n_active, 1);
}

// V[pend_norm] = W * scale; rho += V[0..cols) y
__global__ void k_gm_vec(GmArgs a, const double* __restrict__ W, double* __restrict__ rho) {
  const int s = blockIdx.y;
  const GmState& g = a.st[s];
  if (g.pend_norm < 0 && g.pend_update == 0) return;
  const long base = (long)s * a.nd;
  double* vn = g.pend_norm >= 0 ? vcol(a, s, g.pend_norm) : nullptr;
  const int cols = g.pend_update;
  const double* y = a.y + (long)s * a.m;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < a.nd; t += (long)gridDim.x * blockDim.x) {
    if (vn) vn[t] = W[base + t] * g.scale;
    if (cols) {
      double acc = rho[base + t];
      for (int k = 0; k < cols; ++k) acc = fma(y[k], vcol(a, s, k)[t], acc);
      rho[base + t] = acc;
    }
  }
}

__global__ void k_gm_init(GmArgs a, const double* __restrict__ part) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  GmState& g = a.st[s];
  g = GmState{};
  double bn = sqrt(seq_sum(part, s, a.nblk));
  if (bn == 0.0) bn = 1.0;
  g.bnorm = bn;
  g.phase = PH_START;
  g.pend_norm = -1;
  g.final_res = 0.0;
}

// W = Z + C and its partial squared norm (for ||P bbar||)
__global__ void k_gm_pb(int S, long nd, const double* __restrict__ Z, const double* __restrict__ C,
                        double* __restrict__ part) {
  const int s = blockIdx.y;
  double acc = 0.0;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nd; t += (long)gridDim.x * blockDim.x) {
    const double w = C ? Z[(long)s * nd + t] + C[(long)s * nd + t] : Z[(long)s * nd + t];
    acc = fma(w, w, acc);
  }
  block_part(acc, part, s);
}

}  // namespace

void romig(rte_ctx* ctx, double* rho0, int* status_dev, cudaStream_t st);

void gmres_solve(rte_ctx* ctx, const rte_gmres_config& cfg, double* rho, rte_gmres_report* reports, double* history,
                 int history_cap, cudaStream_t st) {
  RTE_REQUIRE(cfg.restart >= 1, RTE_ERR_INVALID, "gmres: restart must be >= 1");
  RTE_REQUIRE(cfg.max_iters >= 0, RTE_ERR_INVALID, "gmres: max_iters must be >= 0");
  RTE_REQUIRE(history_cap >= 0, RTE_ERR_INVALID, "gmres: negative history capacity");
  const int S = ctx->S, m = cfg.restart;
  const long nd = ctx->ndof;
  const bool pre = cfg.preconditioned != 0;
  if (pre && !ctx->dsa) dsa_setup(ctx, st);
  if (pre) {  // a solve does not depend on earlier calls' warm-start history
    dsa_history_reset(ctx, st);
    dsa_status_reset(ctx, st);
  }
  const int nblk = (int)std::min<long>(256, std::max<long>(1, (nd + 4095) / 4096));
  const dim3 vg(nblk, S);
  const int hcap = std::max(1, history_cap);

  // persistent per-context scratch (grow-only): no cudaMalloc per solve
  DBuf<double>(&dd)[15] = ctx->gm_d;
  DBuf<double>&V = dd[0], &H = dd[1], &gv = dd[2], &cs = dd[3], &sn = dd[4], &yv = dd[5], &hist = dd[6],
  &bbar = dd[7], &U = dd[8], &LU = dd[9], &Z = dd[10], &C = dd[11], &W = dd[12], &part0 = dd[13], &part1 = dd[14];
  DBuf<int>&act = ctx->gm_i[0], &kind = ctx->gm_i[1], &nact = ctx->gm_i[2];
  DBuf<unsigned long long>& zmax = ctx->gm_zmax;
  V.ensure((size_t)S * (m + 1) * nd);
  H.ensure((size_t)S * (m + 1) * m);
  H.zero(st);
  gv.ensure((size_t)S * (m + 1));
  cs.ensure((size_t)S * m);
  sn.ensure((size_t)S * m);
  yv.ensure((size_t)S * m);
  hist.ensure((size_t)S * hcap);
  for (DBuf<double>* b : {&bbar, &U, &LU, &Z, &W}) b->ensure((size_t)S * nd);
  if (pre) C.ensure((size_t)S * nd);
  part0.ensure((size_t)S * nblk);
  part1.ensure((size_t)S * nblk);
  ctx->gm_states.ensure(sizeof(GmState) * S);
  GmState* sts_p = reinterpret_cast<GmState*>(ctx->gm_states.p);
  act.ensure(S);
  kind.ensure(S);
  nact.ensure(1);
  zmax.ensure(S);
  GmArgs a{S, m, nd, sts_p, V.p, H.p, gv.p, cs.p, sn.p, yv.p, hist.p, hcap, cfg.rel_tol, cfg.max_iters, nblk};

  // initial guess
  if (cfg.guess == RTE_GUESS_ROMIG) {
    DBuf<int>& stat = ctx->gm_i[3];
    stat.ensure(S);
    romig(ctx, rho, stat.p, st);
    std::vector<int> hs(S);
    RTE_CUDA(cudaMemcpyAsync(hs.data(), stat.p, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
    RTE_CUDA(cudaStreamSynchronize(st));
    for (int s = 0; s < S; ++s)
      RTE_REQUIRE(hs[s] == 0, RTE_ERR_RUNTIME,
                  "reduced initial guess failed at sample " + std::to_string(s) +
                      (hs[s] == 1 ? " (reduced operator singular)" : " (Galerkin residual check)"));
  } else if (cfg.guess == RTE_GUESS_ZERO) {
    RTE_CUDA(cudaMemsetAsync(rho, 0, sizeof(double) * S * nd, st));
  } else {
    RTE_REQUIRE(cfg.guess == RTE_GUESS_SUPPLIED, RTE_ERR_INVALID, "gmres: unknown guess kind");
  }

  // bbar (1 sweep) and ||P bbar||
  transport_apply(ctx, SRC_G | SRC_BC, ctx->g.p, bbar.p, nullptr, nullptr, nullptr, nullptr, st);
  if (pre) dsa_apply(ctx, bbar.p, C.p, nullptr, 1, st);
  k_gm_pb<<<vg, kT, 0, st>>>(S, nd, bbar.p, pre ? C.p : nullptr, part0.p);
  k_gm_init<<<(S + 127) / 128, 128, 0, st>>>(a, part0.p);
  RTE_CUDA(cudaGetLastError());

  static const bool dbg = std::getenv("RTE_GMRES_DEBUG") != nullptr;
  auto chk = [&](const char* what) {
    if (!dbg) return;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw Error(RTE_ERR_CUDA, std::string("gmres debug: after ") + what + ": " +
                                                        cudaGetErrorString(e));
  };
  chk("init");
  if (!ctx->pinned_int) RTE_CUDA(cudaMallocHost(&ctx->pinned_int, sizeof(int)));
  int* nact_h = ctx->pinned_int;
  {
    for (;;) {
      k_gm_stage<<<vg, kT, 0, st>>>(a, rho, U.p, act.p, kind.p);
      RTE_CUDA(cudaGetLastError());
      chk("stage");
      transport_apply(ctx, SRC_MS_RHO, U.p, LU.p, act.p, nullptr, nullptr, nullptr, st);
      chk("sweep");
      RTE_CUDA(cudaMemsetAsync(zmax.p, 0, sizeof(unsigned long long) * S, st));
      k_gm_z<<<vg, kT, 0, st>>>(a, U.p, LU.p, bbar.p, Z.p, zmax.p);
      chk("z");
      if (pre) dsa_apply(ctx, Z.p, C.p, kind.p, 1, st);
      chk("dsa");
      // MGS passes; pass i reads the partials of pass i-1
      double* parts[2] = {part0.p, part1.p};
      for (int i = 0; i <= m + 1; ++i)
        k_gm_pass<<<vg, kT, 0, st>>>(a, i, Z.p, pre ? C.p : nullptr, W.p, parts[(i + 1) & 1], parts[i & 1]);
      RTE_CUDA(cudaGetLastError());
      chk("mgs");
      RTE_CUDA(cudaMemsetAsync(nact.p, 0, sizeof(int), st));
      k_gm_scalar<<<(S + 127) / 128, 128, 0, st>>>(a, part0.p, part1.p, zmax.p, nact.p);
      chk("scalar");
      k_gm_vec<<<vg, kT, 0, st>>>(a, W.p, rho);
      RTE_CUDA(cudaGetLastError());
      chk("vec");
      RTE_CUDA(cudaMemcpyAsync(nact_h, nact.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      RTE_CUDA(cudaStreamSynchronize(st));
      if (*nact_h == 0) break;
    }
  }

  std::vector<GmState> hs(S);
  RTE_CUDA(cudaMemcpyAsync(hs.data(), sts_p, sizeof(GmState) * S, cudaMemcpyDeviceToHost, st));
  RTE_CUDA(cudaStreamSynchronize(st));
  // non-converged samples: ||rho - L rho - bbar||_inf (uncounted sweep, gmres.cpp:116-119)
  bool any_nc = false;
  for (int s = 0; s < S; ++s) any_nc |= !hs[s].converged;
  std::vector<double> res_nc(S, 0.0);
  if (any_nc) {
    DBuf<unsigned long long>& bits = ctx->gm_bits;
    bits.ensure((size_t)2 * S);
    bits.zero(st);
    transport_apply(ctx, SRC_MS_RHO | SRC_G | SRC_BC, rho, U.p, nullptr, rho, LU.p, bits.p, st);
    std::vector<unsigned long long> hb(2 * S);
    RTE_CUDA(cudaMemcpyAsync(hb.data(), bits.p, sizeof(unsigned long long) * 2 * S, cudaMemcpyDeviceToHost, st));
    RTE_CUDA(cudaStreamSynchronize(st));
    for (int s = 0; s < S; ++s) std::memcpy(&res_nc[s], &hb[2 * s], sizeof(double));
  }
  std::vector<int> dstat(S, RTE_DSA_OK);
  if (pre) dsa_status_read(ctx, dstat.data(), st);
  if (reports) {
    for (int s = 0; s < S; ++s) {
      rte_gmres_report& r = reports[s];
      r.dsa_status = dstat[s];
      r.converged = hs[s].converged;
      r.iterations = hs[s].total;
      r.n_sweep = 1 + (long)hs[s].steps;  // bbar + one apply_A per cycle start and inner step
      r.cycles = hs[s].cycles;
      r.final_residual = hs[s].converged ? hs[s].final_res : res_nc[s];
      r.history_len = hs[s].hist_n;
    }
  }
  if (history && history_cap > 0)
    RTE_CUDA(cudaMemcpy(history, hist.p, sizeof(double) * S * history_cap, cudaMemcpyDeviceToHost));
  if (pre) dsa_status_check(ctx, st, "gmres: DSA preconditioner");
}

}  // namespace rte
