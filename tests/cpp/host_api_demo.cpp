// C++ host-API demo/test (include/rte_b200.hpp): BASELINE configs[0] (C1) --
// slab [0,1], 256 cells, S16, sigma_t = 100, c = 0.9999, q = 1, vacuum -- solved
// with SI-DSA to eps (argv[1]); prints iterations and the solution as JSON.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rte_b200.hpp"

int main(int argc, char** argv) {
  const double eps = argc > 1 ? std::atof(argv[1]) : 1e-10;
  const int N = 256;
  std::vector<double> bounds(N + 1);
  for (int i = 0; i <= N; ++i) bounds[i] = 1.0 * i / N;
  bounds[N] = 1.0;
  const auto quad = rte_b200::gauss_legendre(16);
  std::vector<double> dirs, w = quad.weights;
  for (auto& d : quad.directions) dirs.insert(dirs.end(), d.begin(), d.end());
  // mass blocks from the coefficient closures (weighted_mass, 6-point Gauss)
  const int nq = 6;
  std::vector<double> px(N * nq), py(N * nq);
  rte_b200::check(rte_cell_points(RTE_SLAB1D, N, 1, bounds.data(), 0, 1, 0, 1, nq, px.data(), py.data()), nullptr);
  std::vector<double> wt(N * nq, 100.0), ws(N * nq, 100.0 * 0.9999), one(N * nq, 1.0);
  std::vector<double> mt(N * 4), ms(N * 4), g(2 * N);
  rte_b200::check(rte_weighted_mass(RTE_SLAB1D, N, 1, bounds.data(), 0, 1, 0, 1, nq, wt.data(), mt.data()), nullptr);
  rte_b200::check(rte_weighted_mass(RTE_SLAB1D, N, 1, bounds.data(), 0, 1, 0, 1, nq, ws.data(), ms.data()), nullptr);
  rte_b200::check(rte_project(RTE_SLAB1D, N, 1, bounds.data(), 0, 1, 0, 1, nq, one.data(), g.data()), nullptr);
  rte_problem p{};
  p.geometry = RTE_SLAB1D;
  p.nx = N;
  p.ny = 1;
  p.bounds = bounds.data();
  p.n_dirs = quad.n();
  p.dirs = dirs.data();
  p.weights = w.data();
  p.n_samples = 1;
  p.block = 4;
  p.mt = mt.data();
  p.ms = ms.data();
  p.source = g.data();
  p.source_shared = 1;
  rte_b200::TransportBatch batch(p, 0);
  rte_b200::DsaOperator dsa(batch);
  rte_b200::SolveConfig cfg;
  cfg.eps_sisa = eps;
  cfg.method = RTE_DSA;
  auto res = rte_b200::sisa_solve(batch, cfg);
  const auto& r = res.second[0];
  std::printf("{\"converged\": %d, \"iterations\": %d, \"n_sweep\": %ld, \"log\": \"%s\", \"rho\": [", r.converged,
              r.iterations, r.n_sweep, r.correction_log.c_str());
  for (size_t i = 0; i < res.first.size(); ++i) std::printf(i ? ", %.17g" : "%.17g", res.first[i]);
  // PGMRES on the same system (gmres.cpp:15-124)
  rte_b200::SolveConfig gcfg;
  gcfg.gmres_rel_tol = 1e-11;
  auto gres = rte_b200::gmres_solve(batch, true, gcfg);
  const auto& gr = gres.second[0];
  std::printf("], \"pgmres_converged\": %d, \"pgmres_iterations\": %d, \"pgmres_n_sweep\": %ld, \"pgmres_rho\": [",
              gr.converged, gr.iterations, gr.n_sweep);
  for (size_t i = 0; i < gres.first.size(); ++i) std::printf(i ? ", %.17g" : "%.17g", gres.first[i]);
  std::printf("]}\n");
  return r.converged && gr.converged ? 0 : 1;
}
