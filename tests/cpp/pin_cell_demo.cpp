// C++ host-API problem setup (include/rte_b200.hpp): BASELINE configs[3]
// (C4) -- the parametric pin cell -- declared as a ProblemDefinition with
// affine CoefficientTerms (problem.hpp:24-44) and built by
// TransportBatch(problem, mesh, quad, mus) exactly like the reference's
// TransportSystem constructor (transport_system.cpp:82-109), then solved with
// SI-DSA through the C-ABI.
//
//   pin_cell_demo NX N_TEST EPS OUT.bin [DSA_INNER] [N_TRAIN]
//
// With N_TRAIN > 0 it also runs the reference's offline stage in C++
// (collect_snapshots, correction snapshot matrix, POD rank 20,
// build_reduced_model on the first N_TRAIN parameter vectors; snapshots.cpp
// 118-194, pod.cpp, reduced_model.cpp:106-199) and ROMSAD (theta = 5) on the
// test samples, writing that flux to OUT.bin.romsad.
//
// Parameters: std::mt19937_64 unit draws (cases.cpp:11-13 via rte_unit_draws),
// 40 training vectors first, then N_TEST test vectors, collisions re-drawn
// (cases.cpp:297-313), mu = (sigma_pin ~ U[1,10], eps ~ logU[1e-3,1e-1],
// c ~ U[0.9,0.9999]).  Writes the test solutions to OUT.bin ([S][n_dof]
// doubles) and prints the parameters and per-sample reports as JSON.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rte_b200.hpp"

namespace {

std::vector<rte_b200::Params> c4_params(int n_train, int n_test, bool training = false) {
  const unsigned long long seed = 20260821ULL;
  const long need = (long)(n_train + n_test) * 3 * 4 + 64;
  std::vector<double> u(need);
  rte_b200::check(rte_unit_draws(seed, need, u.data()), nullptr);
  long k = 0;
  auto uni = [](double a, double b, double x) { return a + (b - a) * x; };
  auto logu = [](double a, double b, double x) { return std::exp(std::log(a) + (std::log(b) - std::log(a)) * x); };
  std::vector<rte_b200::Params> out;
  while ((int)out.size() < n_train + n_test) {
    rte_b200::Params p = {uni(1.0, 10.0, u[k]), logu(1e-3, 1e-1, u[k + 1]), uni(0.9, 0.9999, u[k + 2])};
    k += 3;
    bool dup = false;
    for (const auto& q : out) dup = dup || q == p;
    if (!dup) out.push_back(p);
  }
  if (training) return std::vector<rte_b200::Params>(out.begin(), out.begin() + n_train);
  return std::vector<rte_b200::Params>(out.begin() + n_train, out.end());
}

// configs[3]: pin = cells whose centroid lies within r = 0.3 of (0.5, 0.5);
// the closures classify a point by its cell's centroid (per-cell constant).
rte_b200::ProblemDefinition pin_cell(int nx) {
  const double h = 1.0 / nx;
  auto chiP = [h](double x, double y) {
    const double cx = (std::floor(x / h) + 0.5) * h, cy = (std::floor(y / h) + 0.5) * h;
    return (cx - 0.5) * (cx - 0.5) + (cy - 0.5) * (cy - 0.5) <= 0.09 ? 1.0 : 0.0;
  };
  auto chiM = [chiP](double x, double y) { return 1.0 - chiP(x, y); };
  rte_b200::ProblemDefinition p;
  p.geometry = RTE_XY2D;
  p.terms = {
      {nullptr, nullptr, nullptr, "floor"},
      {[](const rte_b200::Params& m) { return m[0]; }, chiP, nullptr, "pin total"},
      {[](const rte_b200::Params& m) { return m[2] * m[0]; }, [chiP](double x, double y) { return -chiP(x, y); },
       chiP, "pin scattering"},
      {[](const rte_b200::Params& m) { return 1.0 / m[1]; }, chiM, nullptr, "moderator total"},
      {[](const rte_b200::Params& m) { return m[2] / m[1]; }, [chiM](double x, double y) { return -chiM(x, y); },
       chiM, "moderator scattering"},
  };
  p.source = chiP;
  p.n_params = 3;
  p.param_ranges = {{1.0, 10.0}, {1e-3, 1e-1}, {0.9, 0.9999}};
  return p;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: pin_cell_demo NX N_TEST EPS OUT.bin [DSA_INNER] [N_TRAIN]\n");
    return 2;
  }
  const int nx = std::atoi(argv[1]), n_test = std::atoi(argv[2]);
  const double eps = std::atof(argv[3]);
  const double dsa_inner = argc > 5 ? std::atof(argv[5]) : 0.0;
  const auto mus = c4_params(40, n_test);
  const auto mesh = rte_b200::Mesh::rect_uniform(0.0, 1.0, nx, 0.0, 1.0, nx);
  const auto quad = rte_b200::chebyshev_legendre(16, 8);
  rte_b200::TransportBatch batch(pin_cell(nx), mesh, quad, mus, 0);
  rte_b200::DsaOperator dsa(batch);
  rte_b200::SolveConfig cfg;
  cfg.eps_sisa = eps;
  cfg.method = RTE_DSA;
  cfg.dsa_inner = dsa_inner;
  auto res = rte_b200::sisa_solve(batch, cfg);
  FILE* f = std::fopen(argv[4], "wb");
  if (!f || std::fwrite(res.first.data(), sizeof(double), res.first.size(), f) != res.first.size()) return 3;
  std::fclose(f);
  std::printf("{\"n_dof\": %ld, \"k_terms\": %d, \"samples\": [", batch.n_dof(), batch.k_terms());
  for (size_t s = 0; s < mus.size(); ++s) {
    const auto& r = res.second[s];
    std::printf("%s{\"mu\": [%.17g, %.17g, %.17g], \"converged\": %d, \"iterations\": %d, \"n_sweep\": %ld, "
                "\"log\": \"%s\"}",
                s ? ", " : "", mus[s][0], mus[s][1], mus[s][2], r.converged, r.iterations, r.n_sweep,
                r.correction_log.c_str());
  }
  std::printf("]");
  const int n_train = argc > 6 ? std::atoi(argv[6]) : 0;
  if (n_train > 0) {
    // offline stage on the training parameters (40 are drawn first, as configs[3] does)
    const double eps_train = 1e-8;
    const int rank = 20;
    auto train = c4_params(40, n_test, true);
    train.resize(std::min<size_t>(train.size(), (size_t)n_train));
    rte_b200::TransportBatch tb(pin_cell(nx), mesh, quad, train, 0);
    auto sn = rte_b200::collect_snapshots(tb, 3, eps_train);
    int ncols = 0;
    auto F = rte_b200::snapshot_matrix(tb, sn, true, &ncols);
    auto pod = rte_b200::pod(F, tb.kinetic_dim(), ncols, rank);
    double total = 0.0, tail = 0.0;
    for (int k = 0; k < ncols; ++k) {
      total += pod.second[k];
      if (k >= rank) tail += pod.second[k];
    }
    auto model = rte_b200::build_reduced_model(tb, pod.first, rank, pod.second, tail / total, eps_train);
    rte_b200::load_rom(batch, 1, model);
    rte_b200::SolveConfig rc;
    rc.eps_sisa = eps;
    rc.method = RTE_ROMSAD;
    rc.theta = 5;
    rc.max_iters = 500;
    rc.dsa_inner = dsa_inner;
    rc.eps_romsad = rte_b200::romsad_tolerance(eps_train, model.discarded_fraction);
    auto rr = rte_b200::sisa_solve(batch, rc);
    const std::string path = std::string(argv[4]) + ".romsad";
    FILE* g = std::fopen(path.c_str(), "wb");
    if (!g || std::fwrite(rr.first.data(), sizeof(double), rr.first.size(), g) != rr.first.size()) return 3;
    std::fclose(g);
    std::printf(", \"pod_cols\": %d, \"discarded_fraction\": %.17g, \"romsad\": [", ncols, model.discarded_fraction);
    for (size_t s = 0; s < rr.second.size(); ++s) {
      const auto& r = rr.second[s];
      std::printf("%s{\"converged\": %d, \"iterations\": %d, \"switch_iter\": %d, \"log\": \"%s\"}", s ? ", " : "",
                  r.converged, r.iterations, r.switch_iter, r.correction_log.c_str());
    }
    std::printf("]");
  }
  std::printf("}\n");
  return 0;
}
