// capi.cu -- the C-ABI of include/rte_b200.h: context setup, transport
// operator entry points, the batched device-resident source-iteration driver
// (sisa.cpp:14-54 for S samples at once) and small bookkeeping kernels.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <utility>

#include "rte_internal.cuh"

using namespace rte;

namespace rte {
void dsa_apply(rte_ctx* ctx, const double* rhs, double* out, const int* kind, int apply_ms, cudaStream_t st);
int sweep2d_dirs_per_cta();
}

rte_ctx::~rte_ctx() {
  dsa_destroy(dsa);
  rom_destroy(rom[0]);
  rom_destroy(rom[1]);
}

namespace {

thread_local std::string g_create_err;

template <typename F>
int guarded(rte_ctx* ctx, F&& f) {
  try {
    f();
    if (ctx) ctx->err.clear();
    return RTE_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what();
    else g_create_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    else g_create_err = e.what();
    return RTE_ERR_RUNTIME;
  }
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------------------
// small kernels

__global__ void apply_block_kernel(int S, int ncells, int nl, int block, const double* __restrict__ m,
                                   const double* __restrict__ x, double* __restrict__ out) {
  const long nd = (long)ncells * nl;
  const long total = (long)S * nd;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
    const long s = t / nd, i = t - s * nd;
    const long c = i / nl;
    const int r = (int)(i - c * nl);
    if (block == 1) {
      out[t] = m[s * ncells + c] * x[t];
    } else {
      const double* mb = m + (s * ncells + c) * block + (long)r * nl;
      const double* xs = x + s * nd + c * nl;
      double v = mb[0] * xs[0];
      for (int k = 1; k < nl; ++k) v += mb[k] * xs[k];
      out[t] = v;
    }
  }
}

__global__ void density_kernel(int S, int nv, long nd, const double* __restrict__ w, const double* __restrict__ f,
                               double* __restrict__ rho) {
  const long total = (long)S * nd;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
    const long s = t / nd, i = t - s * nd;
    double v = 0.0;
    for (int j = 0; j < nv; ++j) v = v + w[j] * f[(s * nv + j) * nd + i];
    rho[t] = v;
  }
}

__device__ __forceinline__ double bits2d(unsigned long long b) { return __longlong_as_double((long long)b); }

__global__ void si_decide_kernel(int S, SiState st, int l, rte_si_config cfg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  if (!st.active[s]) {
    st.kind[s] = KIND_IDLE;
    return;
  }
  const double ch = bits2d(st.change_bits[2 * s]);
  const double rm = bits2d(st.change_bits[2 * s + 1]);
  double chn = ch;
  if (cfg.norm == RTE_NORM_REL && rm > 0) chn = ch / rm;
  st.history[(long)s * cfg.max_iters + l - 1] = chn;
  st.iters[s] = l;
  st.last_change[s] = chn;
  if (cfg.fixed_iters <= 0 && chn < cfg.eps) {  // sisa.cpp:123-127
    st.converged[s] = 1;
    st.active[s] = 0;
    st.kind[s] = KIND_ACCEPT;
    return;
  }
  int kind = KIND_ACCEPT;
  char lg = 0;
  switch (cfg.method) {
    case RTE_SI:
      break;
    case RTE_DSA:
    case RTE_ROMIG:
      kind = KIND_DSA;
      lg = 'D';
      break;
    case RTE_ROMSA:
      kind = st.singular[s] ? KIND_SINGULAR : KIND_ROMSA;
      lg = st.singular[s] ? 'S' : 'R';
      break;
    case RTE_CUSTOM:  // the caller's strategy decides; the log letter comes back from the callback
      kind = KIND_CUSTOM;
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
  }
  if (kind == KIND_DSA && st.switch_iter[s] < 0) st.switch_iter[s] = l;
  // inner tolerance relative to the outer stop test ("1e-2 eps_SISA"):
  // the correction only has to be accurate to dsa_inner * eps / ||delta||
  // and (dsa_floor) to the round-off floor of the iterate: below
  // 2^-53 ||rho*|| / ||delta|| relative, the correction cannot change rho*
  // beyond a few ulps times its gain
  if (st.dsa_tol && kind == KIND_DSA) {
    double t = (cfg.dsa_inner > 0 && cfg.fixed_iters <= 0) ? cfg.dsa_inner * cfg.eps / chn : 0.0;
    if (cfg.dsa_floor > 0) t = fmax(t, ch > 0 ? fmin(0.1, cfg.dsa_floor * 0x1p-53 * rm / ch) : 0.1);
    st.dsa_tol[s] = t;
  }
  st.kind[s] = kind;
  if (lg) st.log[(long)s * cfg.max_iters + l - 1] = lg;
  const int limit = cfg.fixed_iters > 0 ? cfg.fixed_iters : cfg.max_iters;
  if (l >= limit)
    st.active[s] = 0;
  else
    atomicAdd(st.n_active, 1);
}

// RTE_CUSTOM: record the callback's kind letters; 0 = no correction
__global__ void si_custom_kinds_kernel(int S, SiState st, int l, int max_iters, const char* kinds) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S || st.kind[s] != KIND_CUSTOM) return;
  const char c = kinds[s];
  if (c == 0) {
    st.kind[s] = KIND_ACCEPT;
    return;
  }
  st.log[(long)s * max_iters + l - 1] = c;
  if (c == 'D' && st.switch_iter[s] < 0) st.switch_iter[s] = l;
}

// rows [S][stride] -> packed [S][width] (history and log of rte_si_solve)
__global__ void compact_rows_kernel(int S, int stride, int width, const double* __restrict__ hist,
                                    double* __restrict__ hc, const char* __restrict__ lg, char* __restrict__ lc) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)S * width) return;
  const long s = t / width, l = t - s * width;
  hc[t] = hist[s * stride + l];
  lc[t] = lg[s * stride + l];
}

__global__ void si_finalize_kernel(int S, long nd, const int* __restrict__ kind, const double* __restrict__ rho_star,
                                   const double* __restrict__ corr, double* __restrict__ rho) {
  const int s = blockIdx.y;
  const int k = kind[s];
  if (k == KIND_IDLE) return;
  const bool add = (k == KIND_DSA || k == KIND_ROMSA || k == KIND_CUSTOM);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += (long)gridDim.x * blockDim.x) {
    const long t = (long)s * nd + i;
    rho[t] = add ? rho_star[t] + corr[t] : rho_star[t];
  }
}

__global__ void init_state_kernel(int S, SiState st, const int* sing, int method) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  st.active[s] = 1;
  st.iters[s] = 0;
  st.converged[s] = 0;
  st.switch_iter[s] = -1;
  st.singular[s] = sing ? sing[s] : 0;
  st.switched[s] = (method == RTE_ROMSAD && sing && sing[s]) ? 1 : 0;
  st.last_change[s] = 0.0;
}

// Slot tables (transport_system.cpp:194-202: slots keyed by (vx, vy)).
void build_slots(rte_ctx* c) {
  std::map<std::pair<double, double>, int> slot_of;
  c->dir_slot.assign(c->nv, -1);
  c->slot_vx.clear();
  c->slot_vy.clear();
  c->slot_w.clear();
  for (int j = 0; j < c->nv; ++j) {
    const auto key = std::make_pair(c->vx[j], c->geom == RTE_XY2D ? c->vy[j] : 0.0);
    auto it = slot_of.find(key);
    if (it == slot_of.end()) {
      it = slot_of.emplace(key, (int)slot_of.size()).first;
      c->slot_vx.push_back(key.first);
      c->slot_vy.push_back(key.second);
      c->slot_w.push_back(0.0);
    }
    c->dir_slot[j] = it->second;
    c->slot_w[it->second] += c->w[j];
  }
  c->nslots = (int)c->slot_vx.size();
  for (int q = 0; q < 4; ++q) c->q_slots[q].clear();
  for (int k = 0; k < c->nslots; ++k) {
    const int q = (c->slot_vx[k] > 0 ? 0 : 1) + 2 * (c->slot_vy[k] > 0 ? 0 : 1);
    c->q_slots[q].push_back(k);
  }
  for (int q = 0; q < 4; ++q) c->q_count[q] = (int)c->q_slots[q].size();
}

// Canonical slot constants; `single` >= 0 restricts to one slot with weight 1.
std::vector<Slot2D> slot_table(const rte_ctx* c, int dpl, int groups, int nq_pad, int single) {
  std::vector<Slot2D> t((size_t)4 * nq_pad);
  for (auto& e : t) e = Slot2D{1.0, 1.0, 0.0, 0.0, 0.0, -1, -1};
  const double hx = c->hx, hy = c->hy;
  for (int q = 0; q < 4; ++q) {
    int n = 0;
    for (int k : c->q_slots[q]) {
      if (single >= 0 && k != single) continue;
      const double vx = c->slot_vx[k], vy = c->slot_vy[k];
      Slot2D sl;
      sl.a = std::fabs(vx) / hx;
      sl.b = std::fabs(vy) / hy;
      sl.w = single >= 0 ? 1.0 : c->slot_w[k];
      // inflow ghost traces (transport_system.cpp:166-185), canonical basis
      const double gx = vx > 0 ? c->inflow[0] : c->inflow[1];
      const double gy = vy > 0 ? c->inflow[2] : c->inflow[3];
      sl.bcx = std::fabs(vx) * gx * (1.0 / std::sqrt(hx)) * std::sqrt(hy);
      sl.bcy = std::fabs(vy) * gy * (1.0 / std::sqrt(hy)) * std::sqrt(hx);
      sl.dir0 = sl.dir1 = -1;
      for (int j = 0; j < c->nv; ++j)
        if (c->dir_slot[j] == k) {
          if (sl.dir0 < 0)
            sl.dir0 = j;
          else if (sl.dir1 < 0)
            sl.dir1 = j;
        }
      t[(size_t)q * nq_pad + n] = sl;
      ++n;
    }
  }
  (void)dpl;
  (void)groups;
  return t;
}

struct Plan2D {
  int dpl, groups, nq_pad;
};

Plan2D plan2d(const rte_ctx* c, int single) {
  int mq = 0;
  for (int q = 0; q < 4; ++q) {
    int n = single >= 0 ? 1 : c->q_count[q];
    mq = std::max(mq, n);
  }
  const int nw = sweep2d_dirs_per_cta();
  const int nbands = (c->ny + 31) / 32;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  // development knob (read per call so tests can force each production plan)
  const char* dpl_env = std::getenv("RTE_SWEEP_DPL");
  const int force_dpl = dpl_env ? std::atoi(dpl_env) : 0;
  Plan2D best{1, 1, 0};
  for (int dpl : {8, 4, 2, 1}) {
    if (c->block == 16 && dpl > 2) continue;  // full-block cell solve: keep the register budget
    if (force_dpl > 0 && dpl != force_dpl) continue;
    const int groups = std::max(1, (mq + nw * dpl - 1) / (nw * dpl));
    best = Plan2D{dpl, groups, groups * nw * dpl};
    // padded direction slots cost as much as real ones: take a smaller
    // per-lane direction count rather than run more than 1/4 of the lanes
    // on padding (CL(16,8): 16 slots per quadrant -> 2 per lane, not 8)
    if (dpl > 1 && force_dpl == 0 && 4 * (best.nq_pad - mq) > mq) continue;
    const long items = (long)nbands * c->S * 4 * groups;
    if (items >= 4L * sms) break;
  }
  return best;
}

// Independent DFMA chains: 8 per thread, enough warps to saturate the pipe.
__global__ void dfma_probe_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

double probe_dfma_tflops() {
  int dev = 0, sms = 0;
  RTE_CUDA(cudaGetDevice(&dev));
  RTE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DBuf<double> out;
  out.alloc(1);
  const int threads = 512, blocks = sms * 4, iters = 4096;
  cudaEvent_t e0, e1;
  RTE_CUDA(cudaEventCreate(&e0));
  RTE_CUDA(cudaEventCreate(&e1));
  dfma_probe_kernel<<<blocks, threads>>>(out.p, iters, 0.999999, 1e-7);
  RTE_CUDA(cudaEventRecord(e0));
  for (int r = 0; r < 5; ++r) dfma_probe_kernel<<<blocks, threads>>>(out.p, iters, 0.999999, 1e-7);
  RTE_CUDA(cudaEventRecord(e1));
  RTE_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  RTE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double fmas = 5.0 * blocks * threads * (double)iters * 8;
  return 2.0 * fmas / (ms * 1e-3) / 1e12;
}

}  // namespace

namespace rte {

// mode: SrcMode bits.  2D: always through the band-wavefront kernel + the
// fixed-order partial reduction.  rho_prev/delta/change_bits: SI epilogue.
static void transport_apply_ex(rte_ctx* ctx, int mode, int single, const double* rho, double* out, const int* active,
                               const double* rho_prev, double* delta, unsigned long long* change_bits,
                               cudaStream_t st, double* fout = nullptr) {
  if (ctx->geom == RTE_SLAB1D) {
    Sweep1DArgs a{};
    a.S = ctx->S;
    a.N = ctx->ncells;
    a.nv = ctx->nv;
    a.ndof = ctx->ndof;
    a.width = ctx->width.p;
    a.vx = ctx->dvx.p;
    a.w = ctx->dw.p;
    a.block = ctx->block;
    a.mt = ctx->mt.p;
    a.ms = ctx->ms.p;
    a.g = ctx->g.p;
    a.g_shared = ctx->g_shared;
    a.rho = rho;
    a.inflow_l = ctx->inflow[0];
    a.inflow_r = ctx->inflow[1];
    a.mode = mode;
    a.j_single = single;
    a.out = single >= 0 ? nullptr : out;
    a.fout = single >= 0 ? out : fout;
    a.active = active;
    a.rho_prev = rho_prev;
    a.delta = delta;
    a.change_bits = change_bits;
    slab_cache_ensure(ctx, st);
    a.cache = ctx->slab_cache.p;
    a.cache_sc = ctx->slab_sc.p;
    ProfScope ps(ctx, RTE_PROF_SWEEP, st);
    launch_sweep1d(a, st);
    return;
  }
  const Plan2D pl = plan2d(ctx, single);
  const int slot_single = single >= 0 ? ctx->dir_slot[single] : -1;
  DBuf<Slot2D> tmp;
  const Slot2D* dtab = nullptr;
  if (single < 0) {
    if (ctx->slot_tab_dpl != pl.dpl * 1000 + pl.groups) {
      std::vector<Slot2D> tab = slot_table(ctx, pl.dpl, pl.groups, pl.nq_pad, -1);
      ctx->slot_tab.upload(tab.data(), tab.size());
      ctx->slot_tab_dpl = pl.dpl * 1000 + pl.groups;
    }
    dtab = ctx->slot_tab.p;
  } else {
    std::vector<Slot2D> tab = slot_table(ctx, pl.dpl, pl.groups, pl.nq_pad, slot_single);
    tmp.upload(tab.data(), tab.size());
    dtab = tmp.p;
  }
  const int nbands = (ctx->ny + 31) / 32;
  const int nparts = 4 * pl.groups;
  const int ndir_cta = pl.nq_pad / pl.groups;
  ctx->ws_part.alloc((size_t)nparts * ctx->S * ctx->ndof);
  ctx->ws_c.alloc((size_t)ctx->S * 4 * pl.groups * nbands * ctx->nx * ndir_cta * 2);
  ctx->ws_sync.alloc(1 + (size_t)ctx->S * 4 * pl.groups * nbands);
  ctx->ws_sync.zero(st);
  Sweep2DArgs a{};
  a.S = ctx->S;
  a.nx = ctx->nx;
  a.ny = ctx->ny;
  a.slots = dtab;
  a.nq_pad = pl.nq_pad;
  a.groups = pl.groups;
  a.sig_t = ctx->mt.p;
  a.sig_s = ctx->ms.p;
  a.g = ctx->g.p;
  a.g_shared = ctx->g_shared;
  a.rho = rho;
  a.mode = mode;
  a.part = ctx->ws_part.p;
  a.ybuf = ctx->ws_c.p;
  a.sync = ctx->ws_sync.p;
  a.active = active;
  a.fout = fout;
  a.nv = ctx->nv;
  if (ctx->block == 16) {
    a.mt_blk = ctx->mt.p;
    a.ms_blk = ctx->ms.p;
  }
  {
    ProfScope ps(ctx, RTE_PROF_SWEEP, st);
    launch_sweep2d(a, st);
  }
  {
    ProfScope ps(ctx, RTE_PROF_REDUCE, st);
    launch_reduce_partials(ctx->S, ctx->ndof, nparts, ctx->ws_part.p, out, rho_prev, delta, change_bits, active, st);
  }
  // a temporary slot table must outlive the kernels queued above
  if (single >= 0) RTE_CUDA(cudaStreamSynchronize(st));
}

void transport_apply(rte_ctx* ctx, int mode, const double* rho, double* out, const int* active,
                     const double* rho_prev, double* delta, unsigned long long* change_bits, cudaStream_t st) {
  transport_apply_ex(ctx, mode, -1, rho, out, active, rho_prev, delta, change_bits, st);
}

// one kinetic sweep: f (all original directions) and rho* = density(f), with
// the SI epilogue against rho (transport_system.cpp:420-441)
void kinetic_fixed_point(rte_ctx* ctx, const double* rho, double* rstar, double* f, const int* active,
                         double* delta, unsigned long long* bits, cudaStream_t st) {
  transport_apply_ex(ctx, SRC_MS_RHO | SRC_G | SRC_BC, -1, rho, rstar, active, rho, delta, bits, st, f);
}

void launch_apply_block(int S, int ncells, int nl, int block, const double* m, const double* x, double* out,
                        cudaStream_t st) {
  const long total = (long)S * ncells * nl;
  const int blocks = (int)std::min<long>((total + 255) / 256, 65535);
  apply_block_kernel<<<blocks, 256, 0, st>>>(S, ncells, nl, block, m, x, out);
  RTE_CUDA(cudaGetLastError());
}

void launch_density_of(int S, int nv, long nd, const double* w, const double* f, double* rho, cudaStream_t st) {
  const long total = (long)S * nd;
  const int blocks = (int)std::min<long>((total + 255) / 256, 65535);
  density_kernel<<<blocks, 256, 0, st>>>(S, nv, nd, w, f, rho);
  RTE_CUDA(cudaGetLastError());
}

}  // namespace rte

// ===========================================================================

// ---- guard mode (rte_internal.cuh, RTE_GUARD=1) ------------------------------
namespace rte {
namespace guard_detail {
struct GuardState {
  std::mutex mu;
  std::map<void*, size_t> live;  // base -> user bytes
  long violations = 0, checked = 0;
  std::string first;
};
GuardState& guard_state() {
  static GuardState* g = new GuardState();  // never destroyed: buffers may be released at exit
  return *g;
}
// 0 if both guard zones of the allocation at base still hold 0xFF bytes
int guard_zones_bad(void* base, size_t user_bytes) {
  std::vector<unsigned char> h(kGuardBytes);
  int bad = 0;
  const char* zones[2] = {static_cast<char*>(base), static_cast<char*>(base) + kGuardBytes + user_bytes};
  for (const char* z : zones) {
    if (cudaMemcpy(h.data(), z, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    for (unsigned char c : h)
      if (c != 0xFF) {
        ++bad;
        break;
      }
  }
  return bad;
}
void guard_note(GuardState& g, int bad, size_t bytes) {
  ++g.checked;
  if (!bad) return;
  g.violations += bad;
  if (g.first.empty()) g.first = "guard zone overwritten next to a " + std::to_string(bytes) + "-byte allocation";
}
}  // namespace guard_detail
using namespace guard_detail;

bool guard_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RTE_GUARD");
    return e && std::atoi(e) > 0;
  }();
  return on;
}
void guard_register(void* base, size_t user_bytes) {
  GuardState& g = guard_state();
  std::lock_guard<std::mutex> lk(g.mu);
  g.live[base] = user_bytes;
}
void guard_release(void* base) {
  GuardState& g = guard_state();
  std::lock_guard<std::mutex> lk(g.mu);
  auto it = g.live.find(base);
  if (it == g.live.end()) return;
  cudaDeviceSynchronize();
  guard_note(g, guard_zones_bad(base, it->second), it->second);
  g.live.erase(it);
}
}  // namespace rte

namespace rte {
void pool_init() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static bool done[64] = {false};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}
void* pool_alloc(size_t bytes) {
  pool_init();
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, nullptr);
  if (e != cudaSuccess) {  // the pool's reserve may be fragmented: hand it back and retry once
    cudaGetLastError();
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    cudaDeviceSynchronize();
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(&p, bytes, nullptr);
  }
  if (e != cudaSuccess)
    throw Error(RTE_ERR_CUDA, std::string("cudaMallocAsync(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  return p;
}
void pool_free(void* p) {
  if (p) cudaFreeAsync(p, nullptr);
}
size_t device_free_bytes() {
  size_t fr = 0, tot = 0;
  RTE_CUDA(cudaMemGetInfo(&fr, &tot));
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long res = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    if (res > used) fr += (size_t)(res - used);
  }
  return fr;
}
}  // namespace rte

namespace rte {
__global__ void guard_selftest_kernel(double* p, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) p[n] = 1.0;  // one element past the end
}
}  // namespace rte

extern "C" {

int rte_create(const rte_problem* p, int device, rte_ctx** out) {
  return guarded(nullptr, [&] {
    RTE_REQUIRE(p && out, RTE_ERR_INVALID, "rte_create: null argument");
    RTE_REQUIRE(p->geometry == RTE_SLAB1D || p->geometry == RTE_XY2D, RTE_ERR_INVALID, "rte_create: bad geometry");
    RTE_REQUIRE(p->nx >= 1 && (p->geometry == RTE_SLAB1D || p->ny >= 1), RTE_ERR_INVALID, "invalid mesh");
    RTE_REQUIRE(p->n_dirs >= 1 && p->dirs && p->weights, RTE_ERR_INVALID, "rte_create: empty quadrature");
    RTE_REQUIRE(p->n_samples >= 1, RTE_ERR_INVALID, "rte_create: n_samples must be >= 1");
    RTE_REQUIRE(p->mt && p->ms, RTE_ERR_INVALID, "rte_create: mass blocks missing");
    auto* c = new rte_ctx();
    std::unique_ptr<rte_ctx> hold(c);
    c->device = device;
    DeviceGuard dg(device);
    c->geom = p->geometry;
    c->nx = p->nx;
    c->ny = p->geometry == RTE_SLAB1D ? 1 : p->ny;
    c->ncells = c->nx * c->ny;
    c->nl = p->geometry == RTE_SLAB1D ? 2 : 4;
    c->ndof = (long)c->ncells * c->nl;
    c->S = p->n_samples;
    c->nv = p->n_dirs;
    for (int j = 0; j < c->nv; ++j) {
      c->vx.push_back(p->dirs[3 * j]);
      c->vy.push_back(p->dirs[3 * j + 1]);
      c->vz.push_back(p->dirs[3 * j + 2]);
      c->w.push_back(p->weights[j]);
    }
    for (int k = 0; k < 4; ++k) c->inflow[k] = p->inflow[k];
    c->block = p->block;
    if (c->geom == RTE_SLAB1D) {
      RTE_REQUIRE(p->bounds, RTE_ERR_INVALID, "slab mesh needs boundaries");
      RTE_REQUIRE(c->block == 1 || c->block == 4, RTE_ERR_INVALID, "slab: block must be 1 or 4");
      c->bounds.assign(p->bounds, p->bounds + c->nx + 1);
      std::vector<double> wd(c->nx);
      for (int i = 0; i < c->nx; ++i) {
        RTE_REQUIRE(c->bounds[i] < c->bounds[i + 1], RTE_ERR_INVALID, "slab mesh boundaries must be strictly increasing");
        wd[i] = c->bounds[i + 1] - c->bounds[i];
      }
      c->width.upload(wd.data(), wd.size());
      c->dvx.upload(c->vx.data(), c->nv);
      c->dw.upload(c->w.data(), c->nv);
    } else {
      RTE_REQUIRE(c->block == 1 || c->block == 16, RTE_ERR_INVALID,
                  "xy: block must be 1 (sigma I per cell) or 16 (full 4x4 per-cell blocks)");
      RTE_REQUIRE(p->x0 < p->x1 && p->y0 < p->y1, RTE_ERR_INVALID, "invalid rectangular mesh");
      c->hx = (p->x1 - p->x0) / c->nx;
      c->hy = (p->y1 - p->y0) / c->ny;
    }
    build_slots(c);
    if (c->geom == RTE_XY2D) {
      // the 2D sweep writes kinetic output for at most two original directions
      // per (vx, vy) slot (the +/-vz pair of a product quadrature)
      std::vector<int> per_slot(c->nslots, 0);
      for (int j = 0; j < c->nv; ++j) ++per_slot[c->dir_slot[j]];
      for (int k = 0; k < c->nslots; ++k)
        RTE_REQUIRE(per_slot[k] <= 2, RTE_ERR_UNSUPPORTED,
                    "rte_create: more than two directions share one (vx, vy) slot");
    }
    const size_t nblk = (size_t)c->S * c->ncells * c->block;
    c->mt.upload(p->mt, nblk);
    c->ms.upload(p->ms, nblk);
    c->g_shared = p->source_shared ? 1 : 0;
    const size_t ng = (size_t)(c->g_shared ? 1 : c->S) * c->ndof;
    if (p->source) {
      c->g.upload(p->source, ng);
    } else {
      std::vector<double> z(ng, 0.0);
      c->g.upload(z.data(), ng);
    }
    RTE_CUDA(cudaDeviceSynchronize());
    *out = hold.release();
  });
}

void rte_destroy(rte_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dg(ctx->device);
  if (ctx->pinned_int) cudaFreeHost(ctx->pinned_int);
  if (ctx->pinned_hist) cudaFreeHost(ctx->pinned_hist);
  delete ctx;
}

const char* rte_last_error(const rte_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
long rte_n_dof(const rte_ctx* ctx) { return ctx->ndof; }
int rte_n_samples(const rte_ctx* ctx) { return ctx->S; }
int rte_n_slots(const rte_ctx* ctx) { return ctx->nslots; }

int rte_sweep_plan(rte_ctx* ctx, int* dpl, int* groups) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(dpl && groups, RTE_ERR_INVALID, "sweep_plan: null argument");
    *dpl = *groups = 0;
    if (ctx->geom != RTE_XY2D) return;
    const Plan2D p = plan2d(ctx, -1);
    *dpl = p.dpl;
    *groups = p.groups;
  });
}

int rte_apply_L(rte_ctx* ctx, const double* rho, double* out, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    transport_apply(ctx, SRC_MS_RHO, rho, out, nullptr, nullptr, nullptr, nullptr, as_stream(stream));
  });
}

int rte_assemble_rhs(rte_ctx* ctx, double* out, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    transport_apply(ctx, SRC_G | SRC_BC, ctx->g.p, out, nullptr, nullptr, nullptr, nullptr, as_stream(stream));
  });
}

int rte_fixed_point(rte_ctx* ctx, const double* rho, double* out, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    transport_apply(ctx, SRC_MS_RHO | SRC_G | SRC_BC, rho, out, nullptr, nullptr, nullptr, nullptr,
                    as_stream(stream));
  });
}

int rte_sweep_direction(rte_ctx* ctx, int j, const double* rhs, double* f, void* stream) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(j >= 0 && j < ctx->nv, RTE_ERR_INVALID, "sweep_direction: bad direction index");
    DeviceGuard dg(ctx->device);
    transport_apply_ex(ctx, SRC_RAW, j, rhs, f, nullptr, nullptr, nullptr, nullptr, as_stream(stream));
  });
}

int rte_kinetic_sweep(rte_ctx* ctx, const double* rho, double* f, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    ctx->ws_b.alloc((size_t)ctx->S * ctx->ndof);
    transport_apply_ex(ctx, SRC_MS_RHO | SRC_G | SRC_BC, -1, rho, ctx->ws_b.p, nullptr, nullptr, nullptr, nullptr,
                       as_stream(stream), f);
  });
}

int rte_density_of(rte_ctx* ctx, const double* f, double* rho, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    DBuf<double> w;
    w.upload(ctx->w.data(), ctx->nv);
    launch_density_of(ctx->S, ctx->nv, ctx->ndof, w.p, f, rho, as_stream(stream));
    RTE_CUDA(cudaStreamSynchronize(as_stream(stream)));
  });
}

int rte_apply_Ms(rte_ctx* ctx, const double* x, double* out, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    launch_apply_block(ctx->S, ctx->ncells, ctx->nl, ctx->block, ctx->ms.p, x, out, as_stream(stream));
  });
}

int rte_apply_Mt(rte_ctx* ctx, const double* x, double* out, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    launch_apply_block(ctx->S, ctx->ncells, ctx->nl, ctx->block, ctx->mt.p, x, out, as_stream(stream));
  });
}

int rte_set_affine(rte_ctx* ctx, const rte_affine* aff) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(aff && aff->k_terms >= 1 && aff->psi, RTE_ERR_INVALID, "set_affine: bad arguments");
    DeviceGuard dg(ctx->device);
    for (int s = 0; s < ctx->S; ++s)
      RTE_REQUIRE(aff->psi[(size_t)s * aff->k_terms] == 1.0, RTE_ERR_INVALID,
                  "transport system: term 0 must be parameter independent (psi == 1)");
    ctx->k_terms = aff->k_terms;
    ctx->psi_h.assign(aff->psi, aff->psi + (size_t)ctx->S * aff->k_terms);
    ctx->psi.upload(aff->psi, (size_t)ctx->S * aff->k_terms);
    const size_t nb = (size_t)aff->k_terms * ctx->ncells * ctx->block;
    if (aff->term_mt) ctx->term_mt.upload(aff->term_mt, nb);
    if (aff->term_ms) ctx->term_ms.upload(aff->term_ms, nb);
  });
}

int rte_apply_term_kinetic(rte_ctx* ctx, int k, int n_cols, const double* u, double* out, void* stream) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(u && out && u != out, RTE_ERR_INVALID, "apply_term_kinetic: null or aliased buffers");
    DeviceGuard dg(ctx->device);
    apply_term_kinetic(ctx, k, n_cols, u, out, as_stream(stream));
  });
}

int rte_collect_snapshots(rte_ctx* ctx, int window, double eps_train, int max_iters, double* f_iter_dev,
                          double* f_conv_dev, double* drho_dev, int* converged_host, int* n_iter_host) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(window >= 1 && max_iters >= 1, RTE_ERR_INVALID, "collect_snapshots: bad window / max_iters");
    DeviceGuard dg(ctx->device);
    collect_snapshots(ctx, window, eps_train, max_iters, f_iter_dev, f_conv_dev, drho_dev, converged_host,
                      n_iter_host, nullptr);
  });
}

int rte_dsa_setup(rte_ctx* ctx, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    dsa_setup(ctx, as_stream(stream));
  });
}

int rte_dsa_solve_density(rte_ctx* ctx, const double* rhs, double* out, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    RTE_REQUIRE(ctx->dsa, RTE_ERR_INVALID, "dsa: rte_dsa_setup was not called");
    dsa_status_reset(ctx, as_stream(stream));
    dsa_apply(ctx, rhs, out, nullptr, 0, as_stream(stream));
    dsa_status_check(ctx, as_stream(stream), "dsa: solve_density");
  });
}

int rte_dsa_correct(rte_ctx* ctx, const double* delta, double* out, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    RTE_REQUIRE(ctx->dsa, RTE_ERR_INVALID, "dsa: rte_dsa_setup was not called");
    dsa_status_reset(ctx, as_stream(stream));
    dsa_apply(ctx, delta, out, nullptr, 1, as_stream(stream));
    dsa_status_check(ctx, as_stream(stream), "dsa: correct");
  });
}

int rte_dsa_reset_history(rte_ctx* ctx, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    RTE_REQUIRE(ctx->dsa, RTE_ERR_INVALID, "dsa: rte_dsa_setup was not called");
    dsa_history_reset(ctx, as_stream(stream));
  });
}

int rte_dsa_apply_eliminated(rte_ctx* ctx, const double* x, double* out, void* stream) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(x != out, RTE_ERR_INVALID, "dsa: apply_eliminated input and output must not alias");
    DeviceGuard dg(ctx->device);
    dsa_apply_eliminated(ctx, x, out, as_stream(stream));
  });
}

long rte_dsa_coupled_dim(const rte_ctx* ctx) { return dsa_coupled_dim(ctx); }

int rte_dsa_set_tolerance(rte_ctx* ctx, double tol, int max_iters) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(ctx->geom == RTE_XY2D, RTE_ERR_INVALID, "dsa: tolerance applies to the xy (iterative) solver only");
    DeviceGuard dg(ctx->device);
    if (!ctx->dsa) dsa_setup(ctx, nullptr);
    dsa2d_set_tolerance(ctx, tol, max_iters);
  });
}

int rte_dsa_last_iterations(const rte_ctx* ctx) { return ctx->geom == RTE_XY2D ? dsa2d_last_iters(ctx) : 0; }

int rte_dsa_iteration_log(const rte_ctx* ctx, int* out, int cap) {
  if (!ctx || ctx->geom != RTE_XY2D || (cap > 0 && !out)) return 0;
  return dsa2d_iteration_log(ctx, out, cap);
}

int rte_rom_load(rte_ctx* ctx, int which, const rte_rom* rom) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    rom_load(ctx, which, rom);
  });
}

int rte_romig(rte_ctx* ctx, double* rho0, int* status_host, void* stream) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    DBuf<int> stat;
    stat.alloc(ctx->S);
    romig(ctx, rho0, stat.p, as_stream(stream));
    if (status_host) RTE_CUDA(cudaMemcpy(status_host, stat.p, sizeof(int) * ctx->S, cudaMemcpyDeviceToHost));
  });
}

int rte_gmres_solve(rte_ctx* ctx, const rte_gmres_config* cfg, double* rho, rte_gmres_report* reports,
                    double* history, int history_cap) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(cfg && rho, RTE_ERR_INVALID, "gmres: null argument");
    DeviceGuard dg(ctx->device);
    gmres_solve(ctx, *cfg, rho, reports, history, history_cap, nullptr);
  });
}

int rte_si_solve(rte_ctx* ctx, const rte_si_config* cfg_in, double* rho, rte_si_report* reports, double* history,
                 char* log) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(cfg_in && rho, RTE_ERR_INVALID, "si_solve: null argument");
    DeviceGuard dg(ctx->device);
    rte_si_config cfg = *cfg_in;
    RTE_REQUIRE(cfg.max_iters >= 1, RTE_ERR_INVALID, "si_solve: max_iters must be >= 1");
    // history_host / log_host rows are max_iters long
    RTE_REQUIRE(cfg.fixed_iters <= cfg.max_iters, RTE_ERR_INVALID, "si_solve: fixed_iters must not exceed max_iters");
    const int every = cfg.check_every > 0 ? cfg.check_every : 4;
    cudaStream_t st = nullptr;
    const int S = ctx->S;
    const long nd = ctx->ndof;
    const bool need_dsa = cfg.method == RTE_DSA || cfg.method == RTE_ROMSAD || cfg.method == RTE_ROMIG;
    const bool need_rom = cfg.method == RTE_ROMSA || cfg.method == RTE_ROMSAD;
    if (need_dsa && !ctx->dsa) dsa_setup(ctx, st);
    if (need_dsa) {  // a solve does not depend on earlier calls' warm-start history
      dsa_history_reset(ctx, st);
      dsa_status_reset(ctx, st);
    }
    DBuf<int>& ibuf = ctx->si_ibuf;
    ibuf.ensure((size_t)S * 8 + 1);
    SiState sst{};
    sst.active = ibuf.p;
    sst.iters = ibuf.p + S;
    sst.switched = ibuf.p + 2 * S;
    sst.kind = ibuf.p + 3 * S;
    sst.converged = ibuf.p + 4 * S;
    sst.singular = ibuf.p + 5 * S;
    sst.switch_iter = ibuf.p + 6 * S;
    DBuf<int>& sing = ctx->si_int;
    if (need_rom) {
      sing.ensure(S);
      rom_setup(ctx, 1, sing.p, st);
    }
    sst.n_active = ibuf.p + 8 * S;
    DBuf<double>& hist = ctx->si_hist;
    DBuf<double>& lastc = ctx->si_lastc;
    hist.ensure((size_t)S * cfg.max_iters);
    RTE_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(double) * S * cfg.max_iters, st));
    lastc.ensure(S);
    sst.history = hist.p;
    sst.last_change = lastc.p;
    DBuf<char>& lg = ctx->si_log;
    lg.ensure((size_t)S * cfg.max_iters);
    RTE_CUDA(cudaMemsetAsync(lg.p, 0, (size_t)S * cfg.max_iters, st));
    sst.log = lg.p;
    DBuf<unsigned long long>& bits = ctx->si_bits;
    bits.ensure((size_t)2 * S);
    sst.change_bits = bits.p;
    DBuf<double>& dtol = ctx->si_dsatol;
    RTE_REQUIRE(cfg.dsa_floor >= 0, RTE_ERR_INVALID, "si_solve: dsa_floor must be >= 0");
    const bool inner = ((cfg.dsa_inner > 0 && cfg.fixed_iters <= 0) || cfg.dsa_floor > 0) && ctx->geom == RTE_XY2D &&
                       need_dsa;
    if (inner) {
      RTE_REQUIRE(cfg.dsa_inner < 1.0, RTE_ERR_INVALID, "si_solve: dsa_inner must be in [0, 1)");
      dtol.ensure(S);
      sst.dsa_tol = dtol.p;
    }
    struct TolScope {  // the per-sample tolerances apply to this solve only
      rte_ctx* c;
      ~TolScope() { c->dsa_tol_s = nullptr; }
    } tol_scope{ctx};
    ctx->dsa_tol_s = inner ? dtol.p : nullptr;
    init_state_kernel<<<(S + 127) / 128, 128, 0, st>>>(S, sst, need_rom ? sing.p : nullptr, cfg.method);
    RTE_CUDA(cudaGetLastError());

    if (cfg.method == RTE_ROMIG) {
      DBuf<int> stat;
      stat.alloc(S);
      romig(ctx, rho, stat.p, st);
      std::vector<int> hs(S);
      RTE_CUDA(cudaMemcpy(hs.data(), stat.p, sizeof(int) * S, cudaMemcpyDeviceToHost));
      for (int s = 0; s < S; ++s) {
        if (hs[s] == 1)
          throw Error(RTE_ERR_RUNTIME, "reduced initial guess: reduced operator is singular at sample " +
                                           std::to_string(s));
        if (hs[s] == 2)
          throw Error(RTE_ERR_RUNTIME, "reduced initial guess: Galerkin residual check failed at sample " +
                                           std::to_string(s));
      }
    } else if (!cfg.use_guess) {
      RTE_CUDA(cudaMemsetAsync(rho, 0, sizeof(double) * S * nd, st));
    }

    DBuf<double>& rstar = ctx->ws_a;
    DBuf<double>& delta = ctx->ws_b;
    DBuf<double>& corr = ctx->ws_d;
    rstar.alloc((size_t)S * nd);
    delta.alloc((size_t)S * nd);
    corr.alloc((size_t)S * nd);
    RTE_REQUIRE(cfg.method != RTE_CUSTOM || cfg.correct, RTE_ERR_INVALID, "si_solve: RTE_CUSTOM needs a callback");
    std::vector<int> kinds_h(S), active_h(S);
    std::vector<char> letters_h(S);
    DBuf<char>& letters_d = ctx->si_letters;
    letters_d.ensure(S);
    if (!ctx->pinned_int) RTE_CUDA(cudaMallocHost(&ctx->pinned_int, sizeof(int)));
    int* n_active_host = ctx->pinned_int;
    const int fin_bx = (int)std::min<long>((nd + 255) / 256, std::max(1, 8192 / S));
    // slab: the whole loop in one launch (si1d.cu) when a sample fits one CTA
    static const bool fuse1d = [] {
      const char* e = std::getenv("RTE_SI1D_FUSED");
      return !e || std::atoi(e) != 0;
    }();
    bool fused = false;
    if (fuse1d && ctx->geom == RTE_SLAB1D && cfg.method != RTE_CUSTOM) {
      Si1DArgs fa{};
      Sweep1DArgs& a = fa.sw;
      a.S = S;
      a.N = ctx->ncells;
      a.nv = ctx->nv;
      a.ndof = nd;
      a.width = ctx->width.p;
      a.vx = ctx->dvx.p;
      a.w = ctx->dw.p;
      a.block = ctx->block;
      a.mt = ctx->mt.p;
      a.ms = ctx->ms.p;
      a.g = ctx->g.p;
      a.g_shared = ctx->g_shared;
      a.inflow_l = ctx->inflow[0];
      a.inflow_r = ctx->inflow[1];
      a.mode = SRC_MS_RHO | SRC_G | SRC_BC;
      a.j_single = -1;
      slab_cache_ensure(ctx, st);
      a.cache = ctx->slab_cache.p;
      a.cache_sc = ctx->slab_sc.p;
      fa.st = sst;
      fa.cfg = cfg;
      fa.rho = rho;
      fa.fac = need_dsa ? ctx->dsa->fac_c.p : nullptr;
      if (need_rom) rom_fill_si1d(ctx, fa);
      static const bool clk = std::getenv("RTE_SI1D_CLOCKS") != nullptr;  // development: phase clocks
      DBuf<long long> pc;
      if (clk) {
        pc.alloc(4);
        pc.zero(st);
        fa.phase_clk = pc.p;
      }
      {
        ProfScope ps(ctx, RTE_PROF_OTHER, st, 1);
        fused = si1d_fused(fa, st);
      }
      if (clk && fused) {
        long long h[4];
        RTE_CUDA(cudaMemcpy(h, pc.p, sizeof(h), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[si1d] sample 0 clocks: sweep %lld, epilogue+decide %lld, correction %lld, total %lld\n",
                     h[0], h[1], h[2], h[3]);
      }
    }
    int l = fused ? cfg.max_iters + 1 : 1;
    try {
      for (; l <= cfg.max_iters; ++l) {
        bits.zero(st);
        transport_apply(ctx, SRC_MS_RHO | SRC_G | SRC_BC, rho, rstar.p, sst.active, rho, delta.p, bits.p, st);
        RTE_CUDA(cudaMemsetAsync(sst.n_active, 0, sizeof(int), st));
        {
          ProfScope ps(ctx, RTE_PROF_OTHER, st);
          si_decide_kernel<<<(S + 127) / 128, 128, 0, st>>>(S, sst, l, cfg);
          RTE_CUDA(cudaGetLastError());
        }
        if (need_dsa) {
          ProfScope ps(ctx, RTE_PROF_DSA, st, ctx->geom == RTE_XY2D ? 0 : 1);
          dsa_apply(ctx, delta.p, corr.p, sst.kind, 1, st);
          if (ctx->geom == RTE_XY2D && ctx->prof) ctx->prof_n[RTE_PROF_DSA] += dsa2d_take_launches(ctx);
        }
        if (need_rom) {
          ProfScope ps(ctx, RTE_PROF_ROM, st);
          rom_correct(ctx, delta.p, corr.p, sst.kind, st);
        }
        if (cfg.method == RTE_CUSTOM) {
          // host round trip: which samples need a correction, then the callback
          RTE_CUDA(cudaMemcpyAsync(kinds_h.data(), sst.kind, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
          RTE_CUDA(cudaStreamSynchronize(st));
          for (int s = 0; s < S; ++s) {
            active_h[s] = kinds_h[s] == KIND_CUSTOM ? 1 : 0;
            letters_h[s] = 0;
          }
          const int rc = cfg.correct(cfg.correct_user, l, S, nd, active_h.data(), delta.p, corr.p, letters_h.data(),
                                     st);
          RTE_REQUIRE(rc == 0, RTE_ERR_RUNTIME, "si_solve: correction callback failed (" + std::to_string(rc) + ")");
          for (int s = 0; s < S; ++s)
            if (!active_h[s]) letters_h[s] = 0;
          RTE_CUDA(cudaMemcpyAsync(letters_d.p, letters_h.data(), S, cudaMemcpyHostToDevice, st));
          si_custom_kinds_kernel<<<(S + 127) / 128, 128, 0, st>>>(S, sst, l, cfg.max_iters, letters_d.p);
          RTE_CUDA(cudaGetLastError());
        }
        {
          ProfScope ps(ctx, RTE_PROF_OTHER, st, 1);
          si_finalize_kernel<<<dim3(fin_bx, S), 256, 0, st>>>(S, nd, sst.kind, rstar.p, corr.p, rho);
          RTE_CUDA(cudaGetLastError());
        }
        if (l % every == 0 || l == cfg.max_iters || (cfg.fixed_iters > 0 && l >= cfg.fixed_iters)) {
          RTE_CUDA(cudaMemcpyAsync(n_active_host, sst.n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
          RTE_CUDA(cudaStreamSynchronize(st));
          if (*n_active_host == 0) break;
        }
      }
    } catch (...) {
      throw;
    }

    // Readback in (at most) two synchronisations: the report state, the
    // residuals, the DSA status and -- when small -- the full history / log
    // rows go to pinned staging in one batch; a large history is packed on the
    // device to the batch's largest iteration count and copied second.
    if (cfg.compute_residual) {
      bits.zero(st);
      transport_apply(ctx, SRC_MS_RHO | SRC_G | SRC_BC, rho, rstar.p, nullptr, rho, delta.p, bits.p, st);
    }
    const int* dfail = need_dsa ? dsa_status_dev(ctx) : nullptr;
    const size_t nrow = (size_t)S * cfg.max_iters;
    const bool rows_now = (history || log) && nrow * (sizeof(double) + 1) <= ((size_t)1 << 20);
    const size_t b_bits = sizeof(unsigned long long) * 2 * S, b_int = sizeof(int) * S * 8, b_last = sizeof(double) * S,
                 b_fail = sizeof(int) * S, b_rows = rows_now ? nrow * (sizeof(double) + 1) : 0;
    const size_t need0 = b_bits + b_int + b_last + b_fail + b_rows;
    auto staging = [&](size_t need) -> char* {
      if (ctx->pinned_hist_bytes < need) {
        if (ctx->pinned_hist) cudaFreeHost(ctx->pinned_hist);
        ctx->pinned_hist = nullptr;
        ctx->pinned_hist_bytes = 0;
        RTE_CUDA(cudaMallocHost(&ctx->pinned_hist, need));
        ctx->pinned_hist_bytes = need;
      }
      return static_cast<char*>(ctx->pinned_hist);
    };
    char* h0 = staging(need0);
    unsigned long long* hb = reinterpret_cast<unsigned long long*>(h0);
    int* hi = reinterpret_cast<int*>(h0 + b_bits);
    double* hl = reinterpret_cast<double*>(h0 + b_bits + b_int);
    int* hf = reinterpret_cast<int*>(h0 + b_bits + b_int + b_last);
    double* hrow = reinterpret_cast<double*>(h0 + b_bits + b_int + b_last + b_fail);
    char* lrow = reinterpret_cast<char*>(hrow + (rows_now ? nrow : 0));
    if (cfg.compute_residual) RTE_CUDA(cudaMemcpyAsync(hb, bits.p, b_bits, cudaMemcpyDeviceToHost, st));
    RTE_CUDA(cudaMemcpyAsync(hi, ibuf.p, b_int, cudaMemcpyDeviceToHost, st));
    RTE_CUDA(cudaMemcpyAsync(hl, lastc.p, b_last, cudaMemcpyDeviceToHost, st));
    if (dfail) RTE_CUDA(cudaMemcpyAsync(hf, dfail, b_fail, cudaMemcpyDeviceToHost, st));
    if (rows_now) {
      RTE_CUDA(cudaMemcpyAsync(hrow, hist.p, sizeof(double) * nrow, cudaMemcpyDeviceToHost, st));
      RTE_CUDA(cudaMemcpyAsync(lrow, lg.p, nrow, cudaMemcpyDeviceToHost, st));
    }
    RTE_CUDA(cudaStreamSynchronize(st));
    std::vector<double> resid(S, 0.0);
    if (cfg.compute_residual)
      for (int s = 0; s < S; ++s) std::memcpy(&resid[s], &hb[2 * s], sizeof(double));
    std::vector<int> dstat(S, RTE_DSA_OK);
    if (dfail) std::copy(hf, hf + S, dstat.begin());
    if (reports) {
      for (int s = 0; s < S; ++s) {
        rte_si_report& r = reports[s];
        r.converged = hi[4 * S + s];
        r.iterations = hi[S + s];
        r.n_sweep = 1 + (long)r.iterations;  // sisa.cpp:112 (bbar) + one per iteration
        r.switch_iter = hi[6 * S + s];
        r.singular = hi[5 * S + s];
        r.final_residual = resid[s];
        r.last_change = hl[s];
        r.dsa_status = dstat[s];
      }
    }
    // history / log rows: only the first `width` entries (the batch's largest
    // iteration count) are written
    int width = 0;
    for (int s = 0; s < S; ++s) width = std::max(width, hi[S + s]);
    if ((history || log) && width > 0) {
      const double* hh = hrow;
      const char* lh = lrow;
      size_t rstride = (size_t)cfg.max_iters;
      if (!rows_now) {  // pack on the device, then one more copy
        const size_t nh = (size_t)S * width;
        DBuf<double>& hc = ctx->si_hist_c;
        DBuf<char>& lc = ctx->si_log_c;
        hc.ensure(nh);
        lc.ensure(nh);
        compact_rows_kernel<<<(unsigned)((nh + 255) / 256), 256, 0, st>>>(S, cfg.max_iters, width, hist.p, hc.p,
                                                                            lg.p, lc.p);
        RTE_CUDA(cudaGetLastError());
        char* h1 = staging(nh * (sizeof(double) + 1));  // the first batch has been consumed above
        double* hp = reinterpret_cast<double*>(h1);
        char* lp = reinterpret_cast<char*>(hp + nh);
        RTE_CUDA(cudaMemcpyAsync(hp, hc.p, sizeof(double) * nh, cudaMemcpyDeviceToHost, st));
        RTE_CUDA(cudaMemcpyAsync(lp, lc.p, nh, cudaMemcpyDeviceToHost, st));
        RTE_CUDA(cudaStreamSynchronize(st));
        hh = hp;
        lh = lp;
        rstride = (size_t)width;
      }
      for (int s = 0; s < S; ++s) {
        if (history) std::memcpy(history + (size_t)s * cfg.max_iters, hh + (size_t)s * rstride, sizeof(double) * width);
        if (log) std::memcpy(log + (size_t)s * cfg.max_iters, lh + (size_t)s * rstride, width);
      }
    }
    for (int s = 0; s < S; ++s)
      if (dstat[s] != RTE_DSA_OK) {
        static const char* why[] = {"ok", "iteration cap reached", "breakdown", "non-finite residual"};
        throw Error(RTE_ERR_RUNTIME, std::string("si_solve: DSA correction: coupled moment system solve failed at "
                                                 "sample ") + std::to_string(s) + " (" + why[dstat[s] & 3] + ")");
      }
  });
}

int rte_snapshot_columns(rte_ctx* ctx, int window, const double* f_iter, const double* f_conv, const int* n_iter,
                         const int* conv, int kind, int window_limit, double* out, int* n_cols) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    *n_cols = snapshot_columns(ctx->S, window, (long)ctx->nv * ctx->ndof, f_iter, f_conv, n_iter, conv, kind,
                               window_limit > 0 ? window_limit : (1 << 30), out, nullptr);
  });
}

int rte_pod(int device, long m, int n, const double* F, int rank_max, double* U, double* sigma, void* stream) {
  return guarded(nullptr, [&] {
    DeviceGuard dg(device);
    pod(m, n, F, rank_max, U, sigma, as_stream(stream));
  });
}

int rte_truncation_rank(const double* s, int n, double eps_pod) {
  // pod.cpp:117-139: modes below 1e-14 sigma_1 are exact zeros; smallest l
  // with partial/total >= 1 - eps.  -1 for a zero matrix.
  if (n <= 0 || !(s[0] > 0)) return -1;
  const double guard = 1e-14 * s[0];
  int kept = 0;
  double total = 0;
  for (int k = 0; k < n; ++k) {
    if (s[k] >= guard) {
      total += s[k];
      kept = k + 1;
    } else {
      break;
    }
  }
  double partial = 0;
  for (int l = 0; l < kept; ++l) {
    partial += s[l];
    if (partial / total >= 1.0 - eps_pod) return l + 1;
  }
  return kept;
}

namespace {
// kinetic right-hand side b_j = G + g_j^bc of sample s (transport_system.cpp:615-624, 142-187)
std::vector<double> kinetic_rhs_host(rte_ctx* ctx, int s) {
  const long nd = ctx->ndof;
  std::vector<double> g(nd);
  RTE_CUDA(cudaMemcpy(g.data(), ctx->g.p + (ctx->g_shared ? 0 : (size_t)s * nd), sizeof(double) * nd,
                      cudaMemcpyDeviceToHost));
  std::vector<double> b((size_t)ctx->nv * nd);
  const double s3 = kSqrt3;
  for (int j = 0; j < ctx->nv; ++j) {
    double* bj = b.data() + (size_t)j * nd;
    std::copy(g.begin(), g.end(), bj);
    const double vx = ctx->vx[j], vy = ctx->vy[j];
    if (ctx->geom == RTE_SLAB1D) {
      const int n = ctx->nx;
      if (vx > 0 && ctx->inflow[0] != 0) {
        const double a = vx * ctx->inflow[0] / std::sqrt(ctx->bounds[1] - ctx->bounds[0]);
        bj[0] += a;
        bj[1] += -s3 * a;
      } else if (vx < 0 && ctx->inflow[1] != 0) {
        const double a = -vx * ctx->inflow[1] / std::sqrt(ctx->bounds[n] - ctx->bounds[n - 1]);
        bj[2 * (n - 1)] += a;
        bj[2 * (n - 1) + 1] += s3 * a;
      }
      continue;
    }
    const int nx = ctx->nx, ny = ctx->ny;
    const double sx = 1.0 / std::sqrt(ctx->hx), sy = 1.0 / std::sqrt(ctx->hy);
    if (vx > 0 && ctx->inflow[0] != 0) {
      const double a = vx * ctx->inflow[0] * sx * std::sqrt(ctx->hy);
      for (int iy = 0; iy < ny; ++iy) { bj[4L * (nx * iy)] += a; bj[4L * (nx * iy) + 1] += -s3 * a; }
    }
    if (vx < 0 && ctx->inflow[1] != 0) {
      const double a = -vx * ctx->inflow[1] * sx * std::sqrt(ctx->hy);
      for (int iy = 0; iy < ny; ++iy) { bj[4L * (nx - 1 + nx * iy)] += a; bj[4L * (nx - 1 + nx * iy) + 1] += s3 * a; }
    }
    if (vy > 0 && ctx->inflow[2] != 0) {
      const double a = vy * ctx->inflow[2] * sy * std::sqrt(ctx->hx);
      for (int ix = 0; ix < nx; ++ix) { bj[4L * ix] += a; bj[4L * ix + 2] += -s3 * a; }
    }
    if (vy < 0 && ctx->inflow[3] != 0) {
      const double a = -vy * ctx->inflow[3] * sy * std::sqrt(ctx->hx);
      for (int ix = 0; ix < nx; ++ix) { bj[4L * (ix + nx * (ny - 1))] += a; bj[4L * (ix + nx * (ny - 1)) + 2] += s3 * a; }
    }
  }
  return b;
}
}  // namespace

int rte_build_rom(rte_ctx* ctx, int r, const double* U, double* u_rho, double* u_iso, double* a_r, double* b_r) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    const std::vector<double> b = kinetic_rhs_host(ctx, 0);
    build_rom(ctx, r, U, b.data(), u_rho, u_iso, a_r, b_r, nullptr);
  });
}

int rte_kinetic_rhs(rte_ctx* ctx, double* out, void* stream) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(out, RTE_ERR_INVALID, "kinetic_rhs: null argument");
    DeviceGuard dg(ctx->device);
    const size_t kdim = (size_t)ctx->nv * ctx->ndof;
    for (int s = 0; s < ctx->S; ++s) {
      const std::vector<double> b = kinetic_rhs_host(ctx, s);
      RTE_CUDA(cudaMemcpyAsync(out + s * kdim, b.data(), sizeof(double) * kdim, cudaMemcpyHostToDevice,
                               as_stream(stream)));
      RTE_CUDA(cudaStreamSynchronize(as_stream(stream)));
    }
  });
}

int rte_apply_streaming_collision(rte_ctx* ctx, int j, const double* f, double* out, void* stream) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(f && out, RTE_ERR_INVALID, "apply_streaming_collision: null argument");
    RTE_REQUIRE(f != out, RTE_ERR_INVALID, "apply_streaming_collision: out must not alias f");
    RTE_REQUIRE(j >= 0 && j < ctx->nv, RTE_ERR_INVALID, "apply_streaming_collision: bad direction");
    DeviceGuard dg(ctx->device);
    apply_streaming_collision(ctx, j, f, out, as_stream(stream));
  });
}

int rte_apply_kinetic(rte_ctx* ctx, const double* u, double* out, void* stream) {
  return guarded(ctx, [&] {
    RTE_REQUIRE(u && out, RTE_ERR_INVALID, "apply_kinetic: null argument");
    RTE_REQUIRE(u != out, RTE_ERR_INVALID, "apply_kinetic: out must not alias u");
    DeviceGuard dg(ctx->device);
    apply_kinetic(ctx, u, out, as_stream(stream));
  });
}

// ---- measurement ------------------------------------------------------------

int rte_profile_enable(rte_ctx* ctx, int on) {
  return guarded(ctx, [&] {
    // launches counted while profiling was off do not belong to the profile
    if (on && !ctx->prof && ctx->geom == RTE_XY2D) dsa2d_take_launches(ctx);
    ctx->prof = on != 0;
  });
}

int rte_profile_read(rte_ctx* ctx, double* ms, long* n) {
  return guarded(ctx, [&] {
    DeviceGuard dg(ctx->device);
    for (auto& e : ctx->prof_ev) {
      RTE_CUDA(cudaEventSynchronize(e.b));
      float t = 0;
      RTE_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
      ctx->prof_ms[e.kind] += t;
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    ctx->prof_ev.clear();
    for (int k = 0; k < RTE_PROF_KINDS; ++k) {
      if (ms) ms[k] = ctx->prof_ms[k];
      if (n) n[k] = ctx->prof_n[k];
      ctx->prof_ms[k] = 0;
      ctx->prof_n[k] = 0;
    }
  });
}

int rte_probe_dfma(int device, double* tflops) {
  return guarded(nullptr, [&] {
    DeviceGuard dg(device);
    *tflops = probe_dfma_tflops();
  });
}

// ---- host-side discretization helpers ---------------------------------------

int rte_gauss_legendre_nodes(int n, double* x, double* w);
int rte_unit_draws(unsigned long long seed, long n, double* out) {
  return guarded(nullptr, [&] {
    std::mt19937_64 gen(seed);
    for (long i = 0; i < n; ++i) out[i] = static_cast<double>(gen() >> 11) * 0x1p-53;
  });
}


int rte_guard_check(long* violations, long* checked) {
  return guarded(nullptr, [&] {
    using namespace rte;
    GuardState& g = guard_state();
    std::lock_guard<std::mutex> lk(g.mu);
    if (guard_enabled()) {
      RTE_CUDA(cudaDeviceSynchronize());
      for (auto& kv : g.live) guard_note(g, guard_zones_bad(kv.first, kv.second), kv.second);
    }
    if (violations) *violations = g.violations;
    if (checked) *checked = g.checked;
    RTE_REQUIRE(guard_enabled(), RTE_ERR_UNSUPPORTED, "guard: RTE_GUARD is not set for this process");
  });
}

int rte_guard_selftest(int device) {
  return guarded(nullptr, [&] {
    DeviceGuard dg(device);
    rte::DBuf<double> b;
    b.alloc(10);
    rte::guard_selftest_kernel<<<1, 32>>>(b.p, 10);
    RTE_CUDA(cudaDeviceSynchronize());
  });
}

}  // extern "C"
