// rte_b200.hpp -- header-only C++ host API over the C-ABI (rte_b200.h).
//
// Mirrors the reference core library's entry points for the hot path
// (namespace rte, /root/reference/proj/core/include/rte): problem setup
// (TransportSystem ctor, transport_system.hpp:32-34), the DSA operator
// (dsa.hpp:29-56), reduced models (reduced_model.hpp:19-44) and the solver
// driver sisa_solve (solvers.hpp:70-72) with SolveConfig / SolveReport
// (solvers.hpp:13-33) -- batched over parameter samples.  Errors are thrown
// as std::invalid_argument / std::runtime_error like the reference.
//
// Link: -lrte_b200 (paper_2402_10488_b200/librte_b200.so) -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rte_b200.h"

namespace rte_b200 {

inline void check(int code, const rte_ctx* ctx) {
  if (code == RTE_OK) return;
  const std::string msg = rte_last_error(ctx);
  if (code == RTE_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct AngularQuadrature {  // quadrature.hpp:19-35
  int geometry = RTE_SLAB1D;
  std::vector<std::array<double, 3>> directions;
  std::vector<double> weights;
  int n() const { return static_cast<int>(weights.size()); }
};

inline AngularQuadrature gauss_legendre(int n) {  // quadrature.cpp:41-52
  std::vector<double> x(n), w(n);
  check(rte_gauss_legendre_nodes(n, x.data(), w.data()), nullptr);
  AngularQuadrature q;
  for (int j = 0; j < n; ++j) {
    q.directions.push_back({x[j], 0.0, 0.0});
    q.weights.push_back(0.5 * w[j]);
  }
  return q;
}

inline AngularQuadrature chebyshev_legendre(int n_phi, int n_vz) {  // quadrature.cpp:54-73
  std::vector<double> z(n_vz), wz(n_vz);
  check(rte_gauss_legendre_nodes(n_vz, z.data(), wz.data()), nullptr);
  AngularQuadrature q;
  q.geometry = RTE_XY2D;
  const double pi = 3.14159265358979323846;
  for (int j2 = 0; j2 < n_vz; ++j2) {
    const double s = std::sqrt(std::max(0.0, 1.0 - z[j2] * z[j2]));
    for (int j1 = 1; j1 <= n_phi; ++j1) {
      const double phi = 2.0 * j1 * pi / n_phi - pi / n_phi;
      q.directions.push_back({std::cos(phi) * s, std::sin(phi) * s, z[j2]});
      q.weights.push_back((1.0 / n_phi) * (0.5 * wz[j2]));
    }
  }
  return q;
}

// ---- problem setup (problem.hpp:10-44, mesh.hpp:12-36) ----------------------

using Params = std::vector<double>;
using SpatialFn = std::function<double(double, double)>;  // (x, y); y ignored in slab
using ParamFn = std::function<double(const Params&)>;

// problem.hpp:24-29: sigma_a += psi(mu) absorption_weight(x), sigma_s +=
// psi(mu) scattering_weight(x); terms[0] must have psi == 1.
struct CoefficientTerm {
  ParamFn psi;
  SpatialFn absorption_weight;
  SpatialFn scattering_weight;
  std::string name;
};

struct ProblemDefinition {  // problem.hpp:31-44
  int geometry = RTE_SLAB1D;
  std::vector<CoefficientTerm> terms;
  SpatialFn source;  // isotropic source G(x)
  double inflow_left = 0, inflow_right = 0, inflow_bottom = 0, inflow_top = 0;
  int n_params = 0;
  std::vector<std::pair<double, double>> param_ranges;
};

constexpr int kCellRule = 6;  // per-axis Gauss points of the cell rules (transport_system.cpp:18)

struct Mesh {  // mesh.hpp:12-36
  int geometry = RTE_SLAB1D;
  std::vector<double> bounds;  // slab boundaries
  double x0 = 0, x1 = 1, y0 = 0, y1 = 1;
  int nx = 0, ny = 1;

  static Mesh slab(std::vector<double> b) {
    if (b.size() < 2) throw std::invalid_argument("slab mesh needs at least one cell");
    for (size_t i = 1; i < b.size(); ++i)
      if (!(b[i - 1] < b[i])) throw std::invalid_argument("slab mesh boundaries must be strictly increasing");
    Mesh m;
    m.nx = (int)b.size() - 1;
    m.bounds = std::move(b);
    return m;
  }
  static Mesh slab_uniform(double a, double b, int n) {
    if (n < 1 || !(a < b)) throw std::invalid_argument("invalid slab mesh");
    std::vector<double> x(n + 1);
    for (int i = 0; i <= n; ++i) x[i] = a + (b - a) * i / n;
    x[n] = b;
    return slab(std::move(x));
  }
  static Mesh rect_uniform(double x0, double x1, int nx, double y0, double y1, int ny) {
    if (nx < 1 || ny < 1 || !(x0 < x1) || !(y0 < y1)) throw std::invalid_argument("invalid rectangular mesh");
    Mesh m;
    m.geometry = RTE_XY2D;
    m.x0 = x0, m.x1 = x1, m.y0 = y0, m.y1 = y1, m.nx = nx, m.ny = ny;
    return m;
  }
  int cell_count() const { return geometry == RTE_SLAB1D ? nx : nx * ny; }
  int n_local() const { return geometry == RTE_SLAB1D ? 2 : 4; }
  long n_dof() const { return (long)cell_count() * n_local(); }
  int points_per_cell(int nq = kCellRule) const { return geometry == RTE_SLAB1D ? nq : nq * nq; }
  const double* bounds_ptr() const { return bounds.empty() ? nullptr : bounds.data(); }
  // Gauss points of every cell's rule, cell-major (rte_cell_points).
  void cell_points(std::vector<double>& px, std::vector<double>& py, int nq = kCellRule) const {
    px.assign((size_t)cell_count() * points_per_cell(nq), 0.0);
    py.assign(px.size(), 0.0);
    check(rte_cell_points(geometry, nx, ny, bounds_ptr(), x0, x1, y0, y1, nq, px.data(), py.data()), nullptr);
  }
  // weighted_mass (transport_system.cpp:17-55) from values at the cell points.
  std::vector<double> weighted_mass(const std::vector<double>& wvals, int nq = kCellRule) const {
    std::vector<double> out((size_t)cell_count() * n_local() * n_local());
    check(rte_weighted_mass(geometry, nx, ny, bounds_ptr(), x0, x1, y0, y1, nq, wvals.data(), out.data()), nullptr);
    return out;
  }
  // project (dg_space.cpp:31-71) from values at the cell points.
  std::vector<double> project(const std::vector<double>& fvals, int nq = kCellRule) const {
    std::vector<double> out((size_t)n_dof());
    check(rte_project(geometry, nx, ny, bounds_ptr(), x0, x1, y0, y1, nq, fvals.data(), out.data()), nullptr);
    return out;
  }
};

namespace detail {
// Per-cell blocks [cells][nl*nl] -> scalars when every block is d0 I to
// 1e-12 (the closed-form XY cell solve needs sigma I); false otherwise.
inline bool scalar_blocks(const std::vector<double>& m, int nl, std::vector<double>& out) {
  const size_t nb = (size_t)nl * nl, nc = m.size() / nb;
  out.assign(nc, 0.0);
  for (size_t c = 0; c < nc; ++c) {
    const double* f = m.data() + c * nb;
    const double d0 = f[0];
    double err = 0.0, scale = 1e-300;
    for (int i = 0; i < nl; ++i)
      for (int j = 0; j < nl; ++j) {
        err = std::max(err, std::fabs(f[i * nl + j] - (i == j ? d0 : 0.0)));
        if (i == j) scale = std::max(scale, std::fabs(f[i * nl + j]));
      }
    if (err > 1e-12 * scale) return false;
    out[c] = d0;
  }
  return true;
}

// build_masses accumulation (transport_system.cpp:133-138): out_s = sum_k psi_sk term_k, k ascending.
inline std::vector<double> combine_terms(const std::vector<std::vector<double>>& terms, const std::vector<double>& psi,
                                         int S) {
  const int K = (int)terms.size();
  const size_t n = terms[0].size();
  std::vector<double> out((size_t)S * n, 0.0);
  for (int s = 0; s < S; ++s)
    for (int k = 0; k < K; ++k) {
      const double p = psi[(size_t)s * K + k];
      double* o = out.data() + (size_t)s * n;
      const double* t = terms[k].data();
      for (size_t e = 0; e < n; ++e) {
        const double v = p * t[e];
        o[e] = o[e] + v;
      }
    }
  return out;
}

inline std::vector<double> flatten(const std::vector<std::vector<double>>& v) {
  std::vector<double> out;
  for (const auto& x : v) out.insert(out.end(), x.begin(), x.end());
  return out;
}
}  // namespace detail

// Device buffer of S x n doubles (sample-major).
class DeviceVector {
 public:
  DeviceVector() = default;
  DeviceVector(long n) : n_(n) {
    if (cudaMalloc(&p_, sizeof(double) * n) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
  }
  ~DeviceVector() {
    if (p_) cudaFree(p_);
  }
  DeviceVector(DeviceVector&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
  DeviceVector(const DeviceVector&) = delete;
  double* data() { return p_; }
  const double* data() const { return p_; }
  long size() const { return n_; }
  std::vector<double> to_host() const {
    std::vector<double> h(n_);
    if (cudaMemcpy(h.data(), p_, sizeof(double) * n_, cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("DeviceVector: device-to-host copy failed");
    return h;
  }
  void from_host(const std::vector<double>& h) {
    if ((long)h.size() != n_) throw std::invalid_argument("DeviceVector: host vector has the wrong size");
    if (cudaMemcpy(p_, h.data(), sizeof(double) * n_, cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("DeviceVector: host-to-device copy failed");
  }

 private:
  double* p_ = nullptr;
  long n_ = 0;
};

// TransportSystem (transport_system.hpp:30-142) for S samples, built from
// per-cell coefficients (slab: full 2x2 blocks or scalars; xy: scalars).
class TransportBatch {
 public:
  TransportBatch(const rte_problem& p, int device = 0) : n_dirs_(p.n_dirs), device_(device) {
    check(rte_create(&p, device, &ctx_), nullptr);
  }
  // The reference constructor (transport_system.cpp:82-109) for a batch of
  // parameter samples mus: evaluates psi_k(mu) and the coefficient closures
  // at the 6x6 (slab: 6) Gauss points, forms the per-term mass blocks
  // (weighted_mass) and the source load vector (project), combines the
  // samples' blocks in build_masses order and uploads everything.  XY
  // problems whose blocks are all sigma I per cell use the closed-form cell
  // solves (per-cell scalars); intra-cell-varying coefficients (or
  // force_full_blocks) use full 4x4 blocks.  Same inputs, same arithmetic as
  // rte.TransportBatch (paper_2402_10488_b200/rte.py).
  TransportBatch(const ProblemDefinition& problem, const Mesh& mesh, const AngularQuadrature& quad,
                 const std::vector<Params>& mus, int device = 0, bool force_full_blocks = false)
      : n_dirs_(quad.n()), device_(device) {
    if (problem.geometry != mesh.geometry || mesh.geometry != quad.geometry)
      throw std::invalid_argument("transport system: geometry mismatch");
    if (problem.terms.empty()) throw std::invalid_argument("transport system: no coefficient terms");
    if (mus.empty()) throw std::invalid_argument("transport system: no parameter samples");
    const int S = (int)mus.size(), K = (int)problem.terms.size();
    std::vector<double> psi((size_t)S * K);
    for (int s = 0; s < S; ++s)
      for (int k = 0; k < K; ++k) {
        const auto& t = problem.terms[k];
        psi[(size_t)s * K + k] = t.psi ? t.psi(mus[s]) : 1.0;
      }
    for (int s = 0; s < S; ++s)
      if (std::abs(psi[(size_t)s * K] - 1.0) > 0)
        throw std::invalid_argument("transport system: term 0 must be parameter independent (psi == 1)");
    std::vector<double> px, py;
    mesh.cell_points(px, py);
    const size_t np = px.size();
    std::vector<std::vector<double>> tmt(K), tms(K);
    std::vector<double> tot(np), sc(np);
    for (int k = 0; k < K; ++k) {
      const auto& t = problem.terms[k];
      for (size_t i = 0; i < np; ++i) {
        const double a = t.absorption_weight ? t.absorption_weight(px[i], py[i]) : 0.0;
        sc[i] = t.scattering_weight ? t.scattering_weight(px[i], py[i]) : 0.0;
        double v = 0.0;  // transport_system.cpp:125-130
        if (t.absorption_weight) v += a;
        if (t.scattering_weight) v += sc[i];
        tot[i] = v;
      }
      tmt[k] = mesh.weighted_mass(tot);
      tms[k] = mesh.weighted_mass(sc);
    }
    std::vector<double> g((size_t)mesh.n_dof(), 0.0);
    if (problem.source) {
      std::vector<double> f(np);
      for (size_t i = 0; i < np; ++i) f[i] = problem.source(px[i], py[i]);
      g = mesh.project(f);
    }
    int block = mesh.geometry == RTE_SLAB1D ? 4 : 16;
    if (mesh.geometry == RTE_XY2D && !force_full_blocks) {
      std::vector<std::vector<double>> st(K), ss(K);
      bool scalar = true;
      for (int k = 0; k < K && scalar; ++k)
        scalar = detail::scalar_blocks(tmt[k], 4, st[k]) && detail::scalar_blocks(tms[k], 4, ss[k]);
      if (scalar) {
        block = 1;
        tmt = std::move(st);
        tms = std::move(ss);
      }
    }
    const std::vector<double> mt = detail::combine_terms(tmt, psi, S), ms = detail::combine_terms(tms, psi, S);
    std::vector<double> dirs;
    for (const auto& d : quad.directions) dirs.insert(dirs.end(), d.begin(), d.end());
    rte_problem p{};
    p.geometry = mesh.geometry;
    p.nx = mesh.nx;
    p.ny = std::max(mesh.ny, 1);
    p.bounds = mesh.bounds_ptr();
    p.x0 = mesh.x0, p.x1 = mesh.x1, p.y0 = mesh.y0, p.y1 = mesh.y1;
    p.n_dirs = quad.n();
    p.dirs = dirs.data();
    p.weights = quad.weights.data();
    p.inflow[0] = problem.inflow_left;
    p.inflow[1] = problem.inflow_right;
    p.inflow[2] = problem.inflow_bottom;
    p.inflow[3] = problem.inflow_top;
    p.n_samples = S;
    p.block = block;
    p.mt = mt.data();
    p.ms = ms.data();
    p.source = g.data();
    p.source_shared = 1;
    check(rte_create(&p, device, &ctx_), nullptr);
    set_affine(K, detail::flatten(tmt), detail::flatten(tms), psi);
  }
  // Affine decomposition (problem.hpp:24-29): per-term total / scattering
  // mass blocks [K][cells][block] and psi [S][K] with psi[s][0] == 1; needed
  // by the kinetic term operators and the reduced models.
  void set_affine(int k_terms, const std::vector<double>& term_mt, const std::vector<double>& term_ms,
                  const std::vector<double>& psi) {
    rte_affine a{k_terms, term_mt.data(), term_ms.data(), psi.data()};
    check(rte_set_affine(ctx_, &a), ctx_);
    k_terms_ = k_terms;
  }
  int n_dirs() const { return n_dirs_; }
  long kinetic_dim() const { return (long)n_dirs_ * n_dof(); }
  int k_terms() const { return k_terms_; }
  int device() const { return device_; }
  ~TransportBatch() {
    if (ctx_) rte_destroy(ctx_);
  }
  TransportBatch(const TransportBatch&) = delete;
  TransportBatch(TransportBatch&& o) noexcept
      : ctx_(o.ctx_), n_dirs_(o.n_dirs_), device_(o.device_), k_terms_(o.k_terms_) {
    o.ctx_ = nullptr;
  }
  rte_ctx* handle() const { return ctx_; }
  long n_dof() const { return rte_n_dof(ctx_); }
  int n_samples() const { return rte_n_samples(ctx_); }

  void apply_L(const DeviceVector& rho, DeviceVector& out) const {  // transport_system.cpp:393
    check(rte_apply_L(ctx_, rho.data(), out.data(), nullptr), ctx_);
  }
  void assemble_rhs(DeviceVector& out) const {  // transport_system.cpp:406
    check(rte_assemble_rhs(ctx_, out.data(), nullptr), ctx_);
  }
  void apply_Ms(const DeviceVector& x, DeviceVector& out) const {  // transport_system.cpp:373
    check(rte_apply_Ms(ctx_, x.data(), out.data(), nullptr), ctx_);
  }
  void apply_Mt(const DeviceVector& x, DeviceVector& out) const {  // transport_system.cpp:383
    check(rte_apply_Mt(ctx_, x.data(), out.data(), nullptr), ctx_);
  }
  // rho* = L rho + bbar in one sweep (the SI fixed-point map)
  void fixed_point(const DeviceVector& rho, DeviceVector& out) const {
    check(rte_fixed_point(ctx_, rho.data(), out.data(), nullptr), ctx_);
  }
  void sweep_direction(int j, const DeviceVector& rhs, DeviceVector& f) const {  // transport_system.hpp:53
    check(rte_sweep_direction(ctx_, j, rhs.data(), f.data(), nullptr), ctx_);
  }
  void apply_streaming_collision(int j, const DeviceVector& f, DeviceVector& out) const {  // :482-558
    check(rte_apply_streaming_collision(ctx_, j, f.data(), out.data(), nullptr), ctx_);
  }
  // kinetic vectors are [S][n_dirs * n_dof]
  void kinetic_sweep(const DeviceVector& rho, DeviceVector& f) const {  // transport_system.cpp:420
    check(rte_kinetic_sweep(ctx_, rho.data(), f.data(), nullptr), ctx_);
  }
  void density_of(const DeviceVector& f, DeviceVector& rho) const {  // transport_system.cpp:433
    check(rte_density_of(ctx_, f.data(), rho.data(), nullptr), ctx_);
  }
  void apply_kinetic(const DeviceVector& u, DeviceVector& out) const {  // transport_system.cpp:598
    check(rte_apply_kinetic(ctx_, u.data(), out.data(), nullptr), ctx_);
  }
  void kinetic_rhs(DeviceVector& out) const {  // transport_system.cpp:615
    check(rte_kinetic_rhs(ctx_, out.data(), nullptr), ctx_);
  }

 private:
  rte_ctx* ctx_ = nullptr;
  int n_dirs_ = 0, device_ = 0, k_terms_ = 0;
};

class DsaOperator {  // dsa.hpp:29-56
 public:
  explicit DsaOperator(TransportBatch& b) : b_(&b) { check(rte_dsa_setup(b.handle(), nullptr), b.handle()); }
  void correct(const DeviceVector& delta, DeviceVector& out) const {
    check(rte_dsa_correct(b_->handle(), delta.data(), out.data(), nullptr), b_->handle());
  }
  void solve_density(const DeviceVector& rhs, DeviceVector& out) const {
    check(rte_dsa_solve_density(b_->handle(), rhs.data(), out.data(), nullptr), b_->handle());
  }
  // dsa.cpp:279-293: S x = A_rr x - A_rJ T^-1 A_Jr x
  void apply_eliminated(const DeviceVector& x, DeviceVector& out) const {
    check(rte_dsa_apply_eliminated(b_->handle(), x.data(), out.data(), nullptr), b_->handle());
  }
  long coupled_dim() const { return rte_dsa_coupled_dim(b_->handle()); }
  // XY: relative residual of the iterative coupled solve (default 1e-12)
  void set_tolerance(double tol, int max_iters = 0) const {
    check(rte_dsa_set_tolerance(b_->handle(), tol, max_iters), b_->handle());
  }
  int last_iterations() const { return rte_dsa_last_iterations(b_->handle()); }
  /* Krylov iteration counts of the XY DSA solves of the last solve call, one per correction */
  std::vector<int> iteration_log() const {
    std::vector<int> v(4096);
    const int n = rte_dsa_iteration_log(b_->handle(), v.data(), (int)v.size());
    v.resize(n < 0 ? 0 : std::min<size_t>((size_t)n, v.size()));
    return v;
  }

 private:
  TransportBatch* b_;
};

struct SolveConfig {  // solvers.hpp:13-19 (+ batch options)
  double eps_sisa = 1e-11;
  int max_iters = 2000;
  int method = RTE_DSA;
  int norm = RTE_NORM_ABS;
  int theta = 3;
  double eps_romsad = 0.0;
  int fixed_iters = 0;
  const std::vector<double>* initial_guess = nullptr;  // S * n_dof, host
  int gmres_restart = 25;        // solvers.hpp:16
  double gmres_rel_tol = 1e-11;  // solvers.hpp:17
  double dsa_inner = 0.0;        // xy DSA inner tolerance factor (rte_si_config.dsa_inner)
  double dsa_floor = 0.0;        // xy DSA round-off floor factor (rte_si_config.dsa_floor)
  rte_correction_fn correct = nullptr;  // RTE_CUSTOM (see the CorrectionStrategy overload of sisa_solve)
  void* correct_user = nullptr;
};

struct SolveReport {  // solvers.hpp:21-33 (per sample)
  bool converged = false;
  long n_sweep = 0;
  int iterations = 0;
  std::vector<double> change_history;
  double final_residual = 0;
  std::string correction_log;
  int switch_iter = -1;
  std::string strategy;  // label of a caller strategy (CorrectionStrategy overload)
  int dsa_status = RTE_DSA_OK;  // worst rte_dsa_status of the sample's DSA corrections
};

// sisa_solve (solvers.hpp:70-72) for all samples: returns rho [S * n_dof].
inline std::pair<std::vector<double>, std::vector<SolveReport>> sisa_solve(TransportBatch& b, const SolveConfig& c) {
  const int S = b.n_samples();
  const long nd = b.n_dof();
  DeviceVector rho((long)S * nd);
  if (c.initial_guess) rho.from_host(*c.initial_guess);
  rte_si_config cfg{c.method, c.eps_sisa, c.norm, c.max_iters, c.fixed_iters, c.theta, c.eps_romsad,
                    c.initial_guess ? 1 : 0, 1, 4};
  cfg.dsa_inner = c.dsa_inner;
  cfg.dsa_floor = c.dsa_floor;
  cfg.correct = c.correct;
  cfg.correct_user = c.correct_user;
  const int mi = c.max_iters;  // rte_si_solve rejects fixed_iters > max_iters
  std::vector<rte_si_report> reps(S);
  std::vector<double> hist((size_t)S * mi);
  std::vector<char> log((size_t)S * mi);
  check(rte_si_solve(b.handle(), &cfg, rho.data(), reps.data(), hist.data(), log.data()), b.handle());
  std::vector<SolveReport> out(S);
  for (int s = 0; s < S; ++s) {
    SolveReport& r = out[s];
    r.converged = reps[s].converged != 0;
    r.n_sweep = reps[s].n_sweep;
    r.iterations = reps[s].iterations;
    r.change_history.assign(hist.begin() + (long)s * mi, hist.begin() + (long)s * mi + r.iterations);
    r.final_residual = reps[s].final_residual;
    r.switch_iter = reps[s].switch_iter;
    r.dsa_status = reps[s].dsa_status;
    for (int l = 0; l < r.iterations; ++l)
      if (log[(size_t)s * mi + l]) r.correction_log.push_back(log[(size_t)s * mi + l]);
  }
  return {rho.to_host(), out};
}

// The reference's plugin point (solvers.hpp:38-51), one instance per sample:
// setup() before the solve; correct(l, delta) once per SI iteration with
// delta = rho* - rho (host vector, n_dof) returns the correction; last_kind()
// is the correction-log letter (0: no correction).  Existing host-side
// strategies port unchanged; the device loop calls them through RTE_CUSTOM.
class CorrectionStrategy {
 public:
  virtual ~CorrectionStrategy() = default;
  virtual void setup(TransportBatch& /*batch*/, int /*sample*/) {}
  virtual std::vector<double> correct(int l, const std::vector<double>& delta) = 0;
  virtual char last_kind() const = 0;
  virtual std::string label() const = 0;
};

namespace detail {
struct StrategyCall {
  std::vector<CorrectionStrategy*>* strategies;
  std::string error;
};
inline int strategy_trampoline(void* user, int l, int n_samples, long n_dof, const int* active, const double* delta,
                               double* corr, char* kind, void* stream) {
  auto* call = static_cast<StrategyCall*>(user);
  try {
    std::vector<double> d((size_t)n_dof);
    for (int s = 0; s < n_samples; ++s) {
      if (!active[s]) continue;
      CorrectionStrategy* st = (*call->strategies)[s];
      cudaMemcpyAsync(d.data(), delta + (long)s * n_dof, sizeof(double) * n_dof, cudaMemcpyDeviceToHost,
                      static_cast<cudaStream_t>(stream));
      cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
      const std::vector<double> c = st->correct(l, d);
      if ((long)c.size() != n_dof) throw std::invalid_argument("strategy: correction has the wrong size");
      cudaMemcpyAsync(corr + (long)s * n_dof, c.data(), sizeof(double) * n_dof, cudaMemcpyHostToDevice,
                      static_cast<cudaStream_t>(stream));
      cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
      kind[s] = st->last_kind();
    }
    return 0;
  } catch (const std::exception& e) {
    call->error = e.what();
    return 1;
  }
}
}  // namespace detail

// sisa_solve (solvers.hpp:70-72) with one caller strategy per sample (RTE_CUSTOM).
inline std::pair<std::vector<double>, std::vector<SolveReport>> sisa_solve(TransportBatch& b,
                                                                           std::vector<CorrectionStrategy*> strategies,
                                                                           SolveConfig c) {
  const int S = b.n_samples();
  if ((int)strategies.size() != S) throw std::invalid_argument("sisa_solve: one strategy per sample");
  for (int s = 0; s < S; ++s) strategies[s]->setup(b, s);
  detail::StrategyCall call{&strategies, {}};
  c.method = RTE_CUSTOM;
  c.correct = detail::strategy_trampoline;
  c.correct_user = &call;
  try {
    auto res = sisa_solve(b, c);
    for (int s = 0; s < S; ++s) res.second[s].strategy = strategies[s]->label();
    return res;
  } catch (const std::runtime_error&) {
    if (!call.error.empty()) throw std::runtime_error(call.error);
    throw;
  }
}

// gmres_solve (solvers.hpp:80-82, gmres.cpp:15-124) for all samples:
// preconditioned = PGMRES with the context's DSA operator; romig_guess =
// PGMRES-ROMIG (runner.cpp:202-205).  Returns rho [S * n_dof].
inline std::pair<std::vector<double>, std::vector<SolveReport>> gmres_solve(TransportBatch& b, bool preconditioned,
                                                                            const SolveConfig& c,
                                                                            bool romig_guess = false) {
  const int S = b.n_samples();
  const long nd = b.n_dof();
  DeviceVector rho((long)S * nd);
  if (c.initial_guess) rho.from_host(*c.initial_guess);
  rte_gmres_config cfg{preconditioned ? 1 : 0, c.gmres_restart, c.gmres_rel_tol, c.max_iters,
                       romig_guess ? RTE_GUESS_ROMIG : (c.initial_guess ? RTE_GUESS_SUPPLIED : RTE_GUESS_ZERO)};
  const int cap = 2 * c.max_iters + 2;
  std::vector<rte_gmres_report> reps(S);
  std::vector<double> hist((size_t)S * cap);
  check(rte_gmres_solve(b.handle(), &cfg, rho.data(), reps.data(), hist.data(), cap), b.handle());
  std::vector<SolveReport> out(S);
  for (int s = 0; s < S; ++s) {
    SolveReport& r = out[s];
    r.converged = reps[s].converged != 0;
    r.n_sweep = reps[s].n_sweep;
    r.iterations = reps[s].iterations;
    const int n = std::min(reps[s].history_len, cap);
    r.change_history.assign(hist.begin() + (long)s * cap, hist.begin() + (long)s * cap + n);
    r.final_residual = reps[s].final_residual;
  }
  return {rho.to_host(), out};
}

// ---- reduced models: offline stage and online strategies -------------------

// ReducedModel (reduced_model.hpp:19-44), column-major like the reference's
// Eigen storage: u_rho / u_iso n_dof x r, a_r K blocks of r x r.
struct ReducedModel {
  int rank = 0, k_affine = 0;
  std::vector<double> u_rho, u_iso, a_r, b_r;
  std::vector<double> singular_values;  // the first `rank` POD singular values
  double eps_pod = 0.0, eps_train = 0.0;
  double discarded_fraction = 0.0;      // sum_{k > r} sigma_k / sum sigma_k
};

// RomsadStrategy tolerance eta * max(eps_train, eps_pod) (strategies.cpp:30-32).
inline double romsad_tolerance(double eps_train, double eps_pod, double eta = 0.1) {
  return eta * std::max(eps_train, eps_pod);
}

// Upload a model: which = 0 primary (ROMIG), 1 correction (ROMSA / ROMSAD).
inline void load_rom(TransportBatch& b, int which, const ReducedModel& m) {
  rte_rom r{m.rank, m.k_affine, m.u_rho.data(), m.u_iso.data(), m.a_r.data(), m.b_r.data(), m.eps_pod, m.eps_train};
  check(rte_rom_load(b.handle(), which, &r), b.handle());
}

// romig (strategies.cpp:8-28) for every sample: rho0 [S * n_dof]; throws
// std::runtime_error for a singular reduced operator or a failed Galerkin
// residual check, as the reference does.
inline std::vector<double> romig(TransportBatch& b) {
  const int S = b.n_samples();
  DeviceVector rho((long)S * b.n_dof());
  std::vector<int> status(S);
  check(rte_romig(b.handle(), rho.data(), status.data(), nullptr), b.handle());
  for (int s = 0; s < S; ++s) {
    if (status[s] == 1) throw std::runtime_error("romig: reduced operator is singular at sample " + std::to_string(s));
    if (status[s] == 2) throw std::runtime_error("romig: Galerkin residual check failed at sample " + std::to_string(s));
  }
  return rho.to_host();
}

// collect_snapshots (snapshots.cpp:118-194) for every training sample of the
// batch at once, kept in device memory.
struct Snapshots {
  int window = 0;
  DeviceVector f_iter, f_conv, drho;  // [S][window][kdim], [S][kdim], [S][window][n_dof]
  std::vector<int> converged, n_iter;
};

inline Snapshots collect_snapshots(TransportBatch& b, int window, double eps_train, int max_iters = 2000) {
  const int S = b.n_samples();
  const long kdim = b.kinetic_dim();
  Snapshots sn{window, DeviceVector((long)S * window * kdim), DeviceVector((long)S * kdim),
               DeviceVector((long)S * window * b.n_dof()), std::vector<int>(S), std::vector<int>(S)};
  if (cudaMemset(sn.f_iter.data(), 0, sizeof(double) * sn.f_iter.size()) != cudaSuccess ||
      cudaMemset(sn.drho.data(), 0, sizeof(double) * sn.drho.size()) != cudaSuccess)
    throw std::runtime_error("collect_snapshots: cudaMemset failed");
  check(rte_collect_snapshots(b.handle(), window, eps_train, max_iters, sn.f_iter.data(), sn.f_conv.data(),
                              sn.drho.data(), sn.converged.data(), sn.n_iter.data()),
        b.handle());
  return sn;
}

// Training matrix (PrimarySource / CorrectionSource, snapshots.cpp:316-376):
// correction = false: converged solutions; true: f - f^(l).  Column-major
// kdim x n_cols on the device; *n_cols receives the column count.
inline DeviceVector snapshot_matrix(TransportBatch& b, Snapshots& sn, bool correction, int* n_cols,
                                    int window_limit = 0) {
  int n = 0;
  const int kind = correction ? 1 : 0;
  check(rte_snapshot_columns(b.handle(), sn.window, sn.f_iter.data(), sn.f_conv.data(), sn.n_iter.data(),
                             sn.converged.data(), kind, window_limit, nullptr, &n),
        b.handle());
  DeviceVector F((long)n * b.kinetic_dim());
  check(rte_snapshot_columns(b.handle(), sn.window, sn.f_iter.data(), sn.f_conv.data(), sn.n_iter.data(),
                             sn.converged.data(), kind, window_limit, F.data(), &n),
        b.handle());
  *n_cols = n;
  return F;
}

// POD (pod.cpp): the first rank_max left singular vectors of F (m x n,
// column-major, device) and all n singular values.
inline std::pair<DeviceVector, std::vector<double>> pod(const DeviceVector& F, long m, int n, int rank_max,
                                                        int device = 0) {
  DeviceVector U((long)rank_max * m);
  std::vector<double> sigma(n);
  cudaDeviceSynchronize();
  check(rte_pod(device, m, n, F.data(), rank_max, U.data(), sigma.data(), nullptr), nullptr);
  return {std::move(U), sigma};
}

// truncation_rank (pod.cpp:117-139).
inline int truncation_rank(const std::vector<double>& sigma, double eps_pod) {
  const int r = rte_truncation_rank(sigma.data(), (int)sigma.size(), eps_pod);
  if (r < 0) throw std::runtime_error("pod: snapshot matrix is zero");
  return r;
}

// build_reduced_model (reduced_model.cpp:106-199) from a rank-r basis U
// (kdim x r, column-major, device) with the batch's affine term operators.
inline ReducedModel build_reduced_model(TransportBatch& b, const DeviceVector& U, int r,
                                        const std::vector<double>& all_singular_values, double eps_pod,
                                        double eps_train) {
  const long nd = b.n_dof();
  const int K = b.k_terms();
  ReducedModel m;
  m.rank = r;
  m.k_affine = K;
  m.u_rho.resize((size_t)r * nd);
  m.u_iso.resize((size_t)r * nd);
  m.a_r.resize((size_t)K * r * r);
  m.b_r.resize(r);
  cudaDeviceSynchronize();
  check(rte_build_rom(b.handle(), r, U.data(), m.u_rho.data(), m.u_iso.data(), m.a_r.data(), m.b_r.data()),
        b.handle());
  m.eps_pod = eps_pod;
  m.eps_train = eps_train;
  double total = 0.0, tail = 0.0;
  for (size_t k = 0; k < all_singular_values.size(); ++k) {
    total += all_singular_values[k];
    if ((int)k >= r) tail += all_singular_values[k];
  }
  m.singular_values.assign(all_singular_values.begin(),
                           all_singular_values.begin() + std::min<size_t>(r, all_singular_values.size()));
  m.discarded_fraction = total > 0 ? tail / total : 0.0;
  return m;
}

}  // namespace rte_b200
