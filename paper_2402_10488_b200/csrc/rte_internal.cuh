// rte_internal.cuh -- shared declarations of the B200 implementation behind
// include/rte_b200.h.  Host-side context, device kernels' argument blocks and
// launch helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/rte_b200.h"

namespace rte {

constexpr double kSqrt3 = 1.7320508075688772935;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define RTE_CUDA(call)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw ::rte::Error(RTE_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define RTE_REQUIRE(cond, code, msg) \
  do {                               \
    if (!(cond)) throw ::rte::Error((code), (msg)); \
  } while (0)

// Guard mode (RTE_GUARD=1, read once): every device allocation gets a 4 KB
// guard zone on each side filled with 0xFF bytes (NaN as fp64/fp32, -1 as
// int) and its user region is filled with the same pattern, so an
// out-of-bounds write is found by the guard check (rte_guard_check, and at
// release) and an out-of-bounds or uninitialised read turns into NaN that the
// parity tests see.  This is the bounds checking the GPU pool allows
// (compute-sanitizer is not available there).
constexpr size_t kGuardBytes = 4096;
bool guard_enabled();
void guard_register(void* base, size_t user_bytes);
void guard_release(void* base);

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync
// on the legacy stream) with an unbounded release threshold: memory a released
// context returns stays mapped for the next one, so per-parameter setups and
// solves do not pay the driver's page mapping again.  Frees are ordered after
// all prior work (the private DSA stream is joined back into the caller's
// stream at the end of every solve).
void pool_init();
void* pool_alloc(size_t bytes);
void pool_free(void* p);
// free device memory including what the pool holds but does not use
size_t device_free_bytes();

// Owning device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) {
      if (guard_enabled()) {
        char* base = reinterpret_cast<char*>(p) - kGuardBytes;
        guard_release(base);
        cudaFree(base);
      } else {
        pool_free(p);
      }
    }
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    if (guard_enabled()) {
      char* base = nullptr;
      const size_t bytes = count * sizeof(T);
      RTE_CUDA(cudaMalloc(&base, bytes + 2 * kGuardBytes));
      RTE_CUDA(cudaMemset(base, 0xFF, bytes + 2 * kGuardBytes));
      RTE_CUDA(cudaDeviceSynchronize());
      guard_register(base, bytes);
      p = reinterpret_cast<T*>(base + kGuardBytes);
    } else {
      p = static_cast<T*>(pool_alloc(count * sizeof(T)));
    }
    n = count;
  }
  // grow-only variant for per-context scratch reused across calls
  void ensure(size_t count) {
    if (p && count <= n) return;
    alloc(count);
  }
  void upload(const T* host, size_t count) {
    alloc(count);
    if (count) RTE_CUDA(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
  }
  void zero(cudaStream_t s) {
    if (n) RTE_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

// Source-assembly modes shared by the 1D and 2D sweeps.
enum SrcMode : int {
  SRC_MS_RHO = 1,  // q += Ms rho
  SRC_G = 2,       // q += G
  SRC_BC = 4,      // inflow ghost traces (boundary sources, transport_system.cpp:142-187)
  SRC_RAW = 8      // q = rhs given (single-direction sweeps)
};

// Per-sample SI bookkeeping kinds (rte_si_solve).
enum Kind : int { KIND_IDLE = 0, KIND_ACCEPT = 1, KIND_DSA = 2, KIND_ROMSA = 3, KIND_SINGULAR = 4, KIND_CUSTOM = 5 };

// 2D sweep direction table entry: canonical (reflected) constants of one
// unique (vx, vy) slot.
struct Slot2D {
  double a, b;   // |vx|/hx, |vy|/hy
  double w;      // folded quadrature weight (sum over the slot's directions)
  double bcx, bcy;  // inflow ghost traces (already scaled), see sweep2d.cu
  int dir0, dir1;   // original direction indices sharing the slot (-1: none)
};

struct DsaState {
  int nf = 2;
  long dim = 0;
  double m1 = 0, m2 = 0, m3 = 0;
  DBuf<double> fac;         // slab: [S][sum of CR level sizes][48] block cyclic reduction factors
  DBuf<double> fac_c;       // slab: the same factors in the compact layout (slab_dev.cuh crc_*), fused SI
  DBuf<double> fac_t;       // slab: CR factors of the current block T (apply_eliminated, lazy)
  void* impl2d = nullptr;   // xy: multigrid/Krylov state (dsa2d.cu)
};
struct RomState;

}  // namespace rte

struct rte_ctx {
  int device = 0;
  int geom = 0, nx = 0, ny = 1, ncells = 0, nl = 2;
  long ndof = 0;
  int S = 0;
  int nv = 0;
  std::vector<double> vx, vy, vz, w;
  double inflow[4] = {0, 0, 0, 0};
  int block = 1;
  double hx = 0, hy = 0;
  std::vector<double> bounds;

  // device problem data
  rte::DBuf<double> width;   // slab widths [N]
  rte::DBuf<double> slab_cache, slab_sc;  // slab sweep cache (Sweep1DArgs::cache)
  bool slab_cache_tried = false;
  rte::DBuf<double> dvx, dw; // slab directions [nv]
  rte::DBuf<double> mt, ms;  // [S][cells][block]
  rte::DBuf<double> g;       // [S or 1][ndof]
  int g_shared = 0;

  // 2D direction tables
  int nslots = 0;
  std::vector<int> dir_slot;          // direction -> slot
  std::vector<double> slot_vx, slot_vy, slot_w;
  int q_count[4] = {0, 0, 0, 0};      // slots per quadrant
  std::vector<int> q_slots[4];

  // workspace (lazily sized)
  rte::DBuf<double> ws_a, ws_b, ws_c, ws_d, ws_e, ws_part;
  // SI driver scratch reused across rte_si_solve calls (no cudaMalloc per solve)
  rte::DBuf<int> si_ibuf, si_int;
  rte::DBuf<double> si_hist, si_lastc, si_dsatol;
  rte::DBuf<char> si_log, si_letters;
  rte::DBuf<double> si_hist_c;  // packed history rows (rte_si_solve readback)
  rte::DBuf<char> si_log_c;
  rte::DBuf<unsigned long long> si_bits;
  int* pinned_int = nullptr;  // cudaMallocHost, one int for the active-count poll
  void* pinned_hist = nullptr;  // cudaMallocHost staging of the packed SI history / log
  size_t pinned_hist_bytes = 0;
  // PGMRES scratch reused across rte_gmres_solve calls (grow-only)
  rte::DBuf<double> gm_d[15];
  rte::DBuf<int> gm_i[4];
  rte::DBuf<unsigned long long> gm_zmax, gm_bits;
  rte::DBuf<char> gm_states;
  rte::DBuf<unsigned long long> ws_bits;
  rte::DBuf<unsigned int> ws_sync;
  rte::DBuf<rte::Slot2D> slot_tab;  // cached all-slot sweep table (2D)
  int slot_tab_dpl = 0;

  // affine terms
  int k_terms = 0;
  rte::DBuf<double> term_mt, term_ms, psi;
  std::vector<double> psi_h;

  // profiling (rte_profile_enable)
  bool prof = false;
  struct ProfEv { int kind; cudaEvent_t a, b; };
  std::vector<ProfEv> prof_ev;
  double prof_ms[RTE_PROF_KINDS] = {0, 0, 0, 0, 0, 0};
  long prof_n[RTE_PROF_KINDS] = {0, 0, 0, 0, 0, 0};

  rte::DsaState* dsa = nullptr;
  // per-sample relative tolerances for the iterative (xy) DSA solve, set by
  // rte_si_solve for the duration of a solve when rte_si_config.dsa_inner > 0
  // (nullptr: the DSA's own tolerance for every sample)
  const double* dsa_tol_s = nullptr;
  rte::RomState* rom[2] = {nullptr, nullptr};

  std::string err;
  ~rte_ctx();
};

namespace rte {

// RAII scope that brackets the kernels launched inside it with CUDA events
// on `st` when the context profiles (rte_profile_enable).
struct ProfScope {
  rte_ctx* c;
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  int launches;
  ProfScope(rte_ctx* ctx, int k, cudaStream_t s, int n = 1) : c(ctx), kind(k), st(s), launches(n) {
    if (c && c->prof) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (c && c->prof) {
      cudaEventRecord(b, st);
      c->prof_ev.push_back({kind, a, b});
      c->prof_n[kind] += launches;
    }
  }
};

// ---- kernel launchers (implemented in the .cu files) ----------------------

struct Sweep1DArgs {
  int S, N, nv;
  long ndof;
  const double* width;
  const double* vx;
  const double* w;
  int block;
  const double* mt;
  const double* ms;
  const double* g;
  int g_shared;
  const double* rho;   // Ms rho source, or raw rhs in SRC_RAW mode
  double inflow_l, inflow_r;
  int mode;            // SrcMode bits
  int j_single;        // -1 all directions, else only this one (weight 1)
  double* out;         // [S][ndof] sum_j w_j f_j (may be null)
  double* fout;        // kinetic [S][nv][ndof] or single-dir [S][ndof] (may be null)
  const int* active;   // [S] mask (may be null)
  // fused SI epilogue (may be null): delta = out - rho_prev, per-sample
  // max|delta| and max|out| as ordered bit patterns
  const double* rho_prev;
  double* delta;
  unsigned long long* change_bits;  // [S][2]
  // per-context sweep cache (slab_cache_ensure; null: cell blocks on the fly):
  // cache [S][nv][5][32 * CPL] = B^-1 (4) and the trace gain beta of the cell at
  // sweep position p = lane * CPL + k stored at k * 32 + lane; cache_sc [N] = h^-1/2
  const double* cache;
  const double* cache_sc;
};
void launch_sweep1d(const Sweep1DArgs& a, cudaStream_t st);
int sweep1d_cpl(int N);  // cells per lane of the slab sweep (0: unsupported)
// Builds the slab sweep cache once per context (the reference's per-slot
// inverse cache, build_sweep_cache transport_system.cpp:189-227, plus the
// trace gains); leaves it empty when it would exceed the memory budget.
void slab_cache_ensure(rte_ctx* ctx, cudaStream_t st);

struct Sweep2DArgs {
  int S, nx, ny;
  const Slot2D* slots;   // [4][nq_pad] canonical slot table per quadrant
  int nq_pad;            // padded slots per quadrant (multiple of D*NW)
  int groups;            // direction groups per quadrant
  const double* sig_t;   // [S][cells]
  const double* sig_s;   // [S][cells]
  const double* g;       // [S or 1][ndof]
  int g_shared;
  const double* rho;     // [S][ndof] (Ms rho source, or raw rhs)
  int mode;
  double* part;          // [4*groups][S][ndof] partial sums
  double* ybuf;          // band-boundary traces
  unsigned int* sync;    // progress counters + ticket
  const int* active;
  double* fout;          // kinetic output [S][nv][ndof] (null: no kinetic store)
  int nv;
  const double* mt_blk;  // full per-cell 4x4 blocks [S][cells][16] (intra-cell-varying
  const double* ms_blk;  // coefficients), or null: sigma * I from sig_t / sig_s
};
void launch_sweep2d(const Sweep2DArgs& a, cudaStream_t st);

// sum of partials (fixed order) + optional SI epilogue
void launch_reduce_partials(int S, long ndof, int nparts, const double* part, double* out,
                            const double* rho_prev, double* delta, unsigned long long* change_bits,
                            const int* active, cudaStream_t st);

void launch_apply_block(int S, int ncells, int nl, int block, const double* m, const double* x, double* out,
                        cudaStream_t st);
void launch_density_of(int S, int nv, long ndof, const double* w, const double* f, double* rho,
                       cudaStream_t st);

// SI bookkeeping
struct SiState {
  int* active;
  int* iters;
  int* switched;
  int* kind;
  int* converged;
  int* singular;
  double* history;     // [S][max_iters]
  char* log;           // [S][max_iters]
  int* switch_iter;
  unsigned long long* change_bits;  // [S][2]: max|delta|, max|rho*|
  double* last_change;
  int* n_active;
  double* dsa_tol;     // [S] per-sample relative DSA tolerance (rte_si_config.dsa_inner > 0), else nullptr
};
void launch_si_decide(int S, const SiState& st, int l, const rte_si_config& cfg, cudaStream_t s);
void launch_si_finalize(int S, long ndof, const SiState& st, const double* rho_star, const double* corr,
                        double* rho, cudaStream_t s);
void launch_residual(int S, long ndof, const double* rho, const double* rho_star, double* resid,
                     cudaStream_t s);

// Fused slab SI loop (si1d.cu): one CTA per sample runs every iteration of
// rte_si_solve (sweep, stop test / strategy choice, DSA or ROMSA correction)
// with its state in shared memory.
struct Si1DArgs {
  Sweep1DArgs sw;  // mode SRC_MS_RHO | SRC_G | SRC_BC; rho is read from shared memory
  SiState st;
  rte_si_config cfg;
  double* rho;        // [S][ndof] initial guess in, solution out
  const double* fac;  // [S][crc_doubles(N)] DSA factors, compact layout (null: no DSA)
  // ROMSA correction model (r = 0: none)
  int r;
  const double* u_rho;
  const double* u_iso;
  const double* lu;
  const int* rp;
  const int* cp;
  long long* phase_clk;  // optional [4]: summed SM clocks of sample 0's sweep / decide / correction / total
};
bool si1d_fused(const Si1DArgs& a, cudaStream_t st);  // false: does not fit one CTA
void rom_fill_si1d(rte_ctx* ctx, Si1DArgs& a);          // the correction model's device arrays

// DSA
void dsa_setup(rte_ctx* ctx, cudaStream_t st);
void dsa_solve_density(rte_ctx* ctx, const double* rhs, double* out, const int* kind_mask, cudaStream_t st);
void dsa_destroy(DsaState* d);
int dsa2d_last_iters(const rte_ctx* ctx);
int dsa2d_iteration_log(const rte_ctx* ctx, int* out, int cap);
long dsa2d_take_launches(rte_ctx* ctx);
void dsa2d_set_tolerance(rte_ctx* ctx, double tol, int maxit);
long dsa_coupled_dim(const rte_ctx* ctx);
void dsa_apply_eliminated(rte_ctx* ctx, const double* x, double* out, cudaStream_t st);
void dsa_status_reset(rte_ctx* ctx, cudaStream_t st);
void dsa_status_read(rte_ctx* ctx, int* host, cudaStream_t st);  // [S] rte_dsa_status
const int* dsa_status_dev(rte_ctx* ctx);  // device [S] rte_dsa_status, or null (all OK / direct slab solve)
void dsa_status_check(rte_ctx* ctx, cudaStream_t st, const char* what);
void dsa_history_reset(rte_ctx* ctx, cudaStream_t st);

// ROM
void rom_load(rte_ctx* ctx, int which, const rte_rom* rom);
void rom_setup(rte_ctx* ctx, int which, int* singular_dev, cudaStream_t st);
void rom_correct(rte_ctx* ctx, const double* ms_delta, double* corr, const int* kind, cudaStream_t st);
void romig(rte_ctx* ctx, double* rho0, int* status_dev, cudaStream_t st);
void rom_destroy(RomState* r);

// kinetic operators and training (kinetic.cu)
void apply_term_kinetic(rte_ctx* ctx, int k, int ncols, const double* u, double* out, cudaStream_t st);
void apply_streaming_collision(rte_ctx* ctx, int j, const double* f, double* out, cudaStream_t st);
void apply_kinetic(rte_ctx* ctx, const double* u, double* out, cudaStream_t st);
void collect_snapshots(rte_ctx* ctx, int window, double eps, int max_iters, double* f_iter, double* f_conv,
                       double* drho_iter, int* conv_h, int* n_iter_h, cudaStream_t st);

// POD / reduced-model projections (pod.cu)
void pod(long m, int n, const double* F, int rank_max, double* U, double* sigma, cudaStream_t st);
void build_rom(rte_ctx* ctx, int r, const double* U, const double* b_kin_host, double* u_rho, double* u_iso,
               double* a_r, double* b_r, cudaStream_t st);
int snapshot_columns(int S, int window, long kdim, const double* f_iter, const double* f_conv, const int* n_iter,
                     const int* conv, int kind, int window_limit, double* out, cudaStream_t st);

// (P)GMRES (gmres.cu)
void gmres_solve(rte_ctx* ctx, const rte_gmres_config& cfg, double* rho, rte_gmres_report* reports, double* history,
                 int history_cap, cudaStream_t st);

// transport helpers used by the C-ABI (capi.cu)
void transport_apply(rte_ctx* ctx, int mode, const double* rho, double* out, const int* active,
                     const double* rho_prev, double* delta, unsigned long long* change_bits, cudaStream_t st);

}  // namespace rte
