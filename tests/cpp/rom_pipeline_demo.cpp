// C++ host-API ROM pipeline (include/rte_b200.hpp): the reference's offline
// stage (collect_snapshots, POD, build_reduced_model) and online ROMSAD solve
// on a parametric slab (test_rom.cpp:12-31 style: sigma_s = 0.5 + 0.3 mu,
// sigma_a = 0.2, q = 1, inflow 0.3 on the left), all through the C++ wrapper.
// Prints the test solves as JSON for tests/test_gpu_cpp_host.py.
#include <cstdio>
#include <vector>

#include "rte_b200.hpp"

namespace {

struct Slab {
  int N;
  std::vector<double> bounds, px, py;
  std::vector<double> mass(const std::vector<double>& w) const {  // weighted_mass on the 6-point rule
    std::vector<double> m((size_t)N * 4);
    rte_b200::check(rte_weighted_mass(RTE_SLAB1D, N, 1, bounds.data(), 0, 1, 0, 1, 6, w.data(), m.data()), nullptr);
    return m;
  }
};

rte_b200::TransportBatch make_batch(const Slab& sl, const rte_b200::AngularQuadrature& q,
                                    const std::vector<double>& mus, const std::vector<double> tmt[2],
                                    const std::vector<double> tms[2], const std::vector<double>& g,
                                    std::vector<double> dirs) {
  const int S = (int)mus.size();
  const size_t nb = (size_t)sl.N * 4;
  std::vector<double> mt(S * nb, 0.0), ms(S * nb, 0.0), psi(2 * S);
  for (int s = 0; s < S; ++s) {
    psi[2 * s] = 1.0;
    psi[2 * s + 1] = mus[s];
    for (int k = 0; k < 2; ++k)  // build_masses accumulation order (transport_system.cpp:136-137)
      for (size_t e = 0; e < nb; ++e) {
        mt[s * nb + e] += psi[2 * s + k] * tmt[k][e];
        ms[s * nb + e] += psi[2 * s + k] * tms[k][e];
      }
  }
  rte_problem p{};
  p.geometry = RTE_SLAB1D;
  p.nx = sl.N;
  p.ny = 1;
  p.bounds = sl.bounds.data();
  p.n_dirs = q.n();
  p.dirs = dirs.data();
  p.weights = q.weights.data();
  p.inflow[0] = 0.3;
  p.n_samples = S;
  p.block = 4;
  p.mt = mt.data();
  p.ms = ms.data();
  p.source = g.data();
  p.source_shared = 1;
  rte_b200::TransportBatch b(p, 0);
  std::vector<double> t_mt(tmt[0]), t_ms(tms[0]);
  t_mt.insert(t_mt.end(), tmt[1].begin(), tmt[1].end());
  t_ms.insert(t_ms.end(), tms[1].begin(), tms[1].end());
  b.set_affine(2, t_mt, t_ms, psi);
  return b;
}

// test_solvers.cpp:30-62's stub: no correction, log letter 'Z'
class ZeroCorrection : public rte_b200::CorrectionStrategy {
 public:
  std::vector<double> correct(int, const std::vector<double>& delta) override {
    return std::vector<double>(delta.size(), 0.0);
  }
  char last_kind() const override { return 'Z'; }
  std::string label() const override { return "ZERO"; }
};

}  // namespace

int main() {
  Slab sl{64, std::vector<double>(65), {}, {}};
  for (int i = 0; i <= sl.N; ++i) sl.bounds[i] = 1.0 * i / sl.N;
  sl.px.resize(sl.N * 6);
  sl.py.resize(sl.N * 6);
  rte_b200::check(rte_cell_points(RTE_SLAB1D, sl.N, 1, sl.bounds.data(), 0, 1, 0, 1, 6, sl.px.data(), sl.py.data()),
                  nullptr);
  const size_t nq = sl.px.size();
  // term 0: sigma_a 0.2, sigma_s 0.5 (total 0.7); term 1 (psi = mu): sigma_s 0.3
  std::vector<double> tmt[2] = {sl.mass(std::vector<double>(nq, 0.7)), sl.mass(std::vector<double>(nq, 0.3))};
  std::vector<double> tms[2] = {sl.mass(std::vector<double>(nq, 0.5)), sl.mass(std::vector<double>(nq, 0.3))};
  std::vector<double> g((size_t)sl.N * 2), one(nq, 1.0);
  rte_b200::check(rte_project(RTE_SLAB1D, sl.N, 1, sl.bounds.data(), 0, 1, 0, 1, 6, one.data(), g.data()), nullptr);
  const auto quad = rte_b200::gauss_legendre(8);
  std::vector<double> dirs;
  for (auto& d : quad.directions) dirs.insert(dirs.end(), d.begin(), d.end());

  // offline: training solves, correction snapshots, POD, Galerkin projections
  const double eps_train = 1e-10;
  const std::vector<double> train = {0.1, 0.3, 0.5, 0.7, 0.9};
  auto tb = make_batch(sl, quad, train, tmt, tms, g, dirs);
  auto snaps = rte_b200::collect_snapshots(tb, 3, eps_train);
  int ncols = 0;
  auto F = rte_b200::snapshot_matrix(tb, snaps, true, &ncols);
  const int r = 4;
  auto U_sigma = rte_b200::pod(F, tb.kinetic_dim(), ncols, r);
  double total = 0.0, tail = 0.0;
  for (int k = 0; k < ncols; ++k) {
    total += U_sigma.second[k];
    if (k >= r) tail += U_sigma.second[k];
  }
  const double eps_pod = tail / total;
  auto model = rte_b200::build_reduced_model(tb, U_sigma.first, r, U_sigma.second, eps_pod, eps_train);

  // online: ROMSAD on test samples
  const std::vector<double> test = {0.2, 0.45, 0.8};
  auto b = make_batch(sl, quad, test, tmt, tms, g, dirs);
  rte_b200::load_rom(b, 1, model);
  rte_b200::DsaOperator dsa(b);
  rte_b200::SolveConfig cfg;
  cfg.method = RTE_ROMSAD;
  cfg.eps_sisa = 1e-10;
  cfg.theta = 3;
  cfg.eps_romsad = rte_b200::romsad_tolerance(eps_train, eps_pod);
  auto res = rte_b200::sisa_solve(b, cfg);
  std::printf("{\"n_cols\": %d, \"eps_pod\": %.17g, \"sigma\": [", ncols, eps_pod);
  for (int k = 0; k < ncols; ++k) std::printf(k ? ", %.17g" : "%.17g", U_sigma.second[k]);
  std::printf("], \"samples\": [");
  const long nd = b.n_dof();
  for (size_t s = 0; s < test.size(); ++s) {
    const auto& rp = res.second[s];
    std::printf("%s{\"converged\": %d, \"iterations\": %d, \"log\": \"%s\", \"switch_iter\": %d, \"rho\": [",
                s ? ", " : "", rp.converged, rp.iterations, rp.correction_log.c_str(), rp.switch_iter);
    for (long i = 0; i < nd; ++i) std::printf(i ? ", %.17g" : "%.17g", res.first[s * nd + i]);
    std::printf("]}");
  }
  // the plugin point: per-sample ZeroCorrection strategies reproduce plain SI
  rte_b200::SolveConfig scfg;
  scfg.method = RTE_SI;
  scfg.eps_sisa = 1e-10;
  auto si = rte_b200::sisa_solve(b, scfg);
  std::vector<ZeroCorrection> zs(test.size());
  std::vector<rte_b200::CorrectionStrategy*> zp;
  for (auto& z : zs) zp.push_back(&z);
  auto zr = rte_b200::sisa_solve(b, zp, scfg);
  bool same = si.first == zr.first;
  for (size_t s = 0; s < test.size(); ++s)
    same = same && si.second[s].iterations == zr.second[s].iterations &&
           zr.second[s].correction_log == std::string(si.second[s].iterations - 1, 'Z') &&
           zr.second[s].strategy == "ZERO";
  std::printf("], \"zero_strategy_equals_si\": %s, \"si_iterations\": %d}\n", same ? "true" : "false",
              si.second[0].iterations);
  return 0;
}
