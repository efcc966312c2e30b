// rte_oracle.cpp -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// A plain-C++ (no Eigen) restatement of the reference's discrete transport
// operator and consistent-DSA assembly, used by tests/ and by bench.py's
// cpu_baseline / --impl reference leg as the checker.  It is never linked into
// or called by the product path (paper_2402_10488_b200/).
//
// Every function cites the reference file:line it restates
// (paths relative to /root/reference/proj/core/src/).  The reference itself
// cannot be compiled here (Eigen3 and LAPACKE are absent), so
// this restatement is pinned against the reference's own known-answer tests
// (tests/test_oracle_*.py).
//
// Layouts follow the reference: DOF vectors are cell-major with the local
// index fastest (dg_space.hpp:24); kinetic vectors are direction-major blocks
// of n_dof (transport_system.hpp:73-89).
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr double kS3 = 1.7320508075688772935;

thread_local std::string g_err;

// ---------------------------------------------------------------------------
// quadrature.cpp:8-39 -- Gauss-Legendre nodes by Newton iteration in long
// double, ascending order, odd middle node forced to zero.
void gl_nodes(int n, double* x, double* w) {
  const long double pi = 3.141592653589793238462643383279502884L;
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    long double z = std::cos(pi * (i + 0.75L) / (n + 0.5L));
    long double dp = 0.0L;
    for (int it = 0; it < 100; ++it) {
      long double pm1 = 1.0L, pcur = z;
      for (int k = 2; k <= n; ++k) {
        long double pn = ((2.0L * k - 1.0L) * z * pcur - (k - 1.0L) * pm1) / k;
        pm1 = pcur;
        pcur = pn;
      }
      dp = n * (z * pcur - pm1) / (z * z - 1.0L);
      long double step = pcur / dp;
      z -= step;
      if (std::abs(step) < 1e-19L) break;
    }
    const long double wt = 2.0L / ((1.0L - z * z) * dp * dp);
    x[i] = static_cast<double>(-z);
    w[i] = static_cast<double>(wt);
    x[n - 1 - i] = static_cast<double>(z);
    w[n - 1 - i] = static_cast<double>(wt);
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

struct Mesh {
  int geom = 0;  // 0 slab, 1 xy
  int nx = 0, ny = 1;
  std::vector<double> b;  // slab boundaries
  double x0 = 0, x1 = 1, y0 = 0, y1 = 1;
  int cells() const { return geom == 0 ? nx : nx * ny; }
  double width(int i) const { return b[i + 1] - b[i]; }
  double center(int i) const { return 0.5 * (b[i] + b[i + 1]); }
  double hx() const { return (x1 - x0) / nx; }
  double hy() const { return (y1 - y0) / ny; }
  double cx0(int ix) const { return x0 + ix * hx(); }
  double cy0(int iy) const { return y0 + iy * hy(); }
};

// Evaluation points of the per-cell nq-point tensor Gauss rule, in the order
// weighted_mass (transport_system.cpp:23-53) and project (dg_space.cpp:35-69)
// visit them: slab q; 2D qy outer, qx inner.
void cell_points(const Mesh& m, int nq, const double* gx, double* px, double* py) {
  long k = 0;
  if (m.geom == 0) {
    for (int i = 0; i < m.nx; ++i) {
      const double h = m.width(i), xc = m.center(i);
      for (int q = 0; q < nq; ++q) {
        px[k] = xc + 0.5 * h * gx[q];
        py[k] = 0.0;
        ++k;
      }
    }
    return;
  }
  const double hx = m.hx(), hy = m.hy();
  for (int iy = 0; iy < m.ny; ++iy)
    for (int ix = 0; ix < m.nx; ++ix) {
      const double xc = m.cx0(ix) + 0.5 * hx, yc = m.cy0(iy) + 0.5 * hy;
      for (int qy = 0; qy < nq; ++qy) {
        const double y = yc + 0.5 * hy * gx[qy];
        for (int qx = 0; qx < nq; ++qx) {
          px[k] = xc + 0.5 * hx * gx[qx];
          py[k] = y;
          ++k;
        }
      }
    }
}

// Per-cell basis values at the cell's Gauss points (dg_space.cpp:22-28 and
// transport_system.cpp:28-49).  Returns nl values per point.
void basis_at(const Mesh& m, int cell, int nq, const double* gx, std::vector<double>& phi) {
  if (m.geom == 0) {
    const double h = m.width(cell), xc = m.center(cell);
    phi.resize(2 * nq);
    for (int q = 0; q < nq; ++q) {
      const double x = xc + 0.5 * h * gx[q];
      phi[2 * q] = 1.0 / std::sqrt(h);
      phi[2 * q + 1] = std::sqrt(12.0 / (h * h * h)) * (x - xc);
    }
    return;
  }
  const double hx = m.hx(), hy = m.hy();
  const int ix = cell % m.nx, iy = cell / m.nx;
  const double xc = m.cx0(ix) + 0.5 * hx, yc = m.cy0(iy) + 0.5 * hy;
  phi.resize(4 * nq * nq);
  int k = 0;
  for (int qy = 0; qy < nq; ++qy) {
    const double y = yc + 0.5 * hy * gx[qy];
    const double py0 = 1.0 / std::sqrt(hy), py1 = std::sqrt(12.0 / (hy * hy * hy)) * (y - yc);
    for (int qx = 0; qx < nq; ++qx) {
      const double x = xc + 0.5 * hx * gx[qx];
      const double px0 = 1.0 / std::sqrt(hx), px1 = std::sqrt(12.0 / (hx * hx * hx)) * (x - xc);
      phi[4 * k + 0] = px0 * py0;
      phi[4 * k + 1] = px1 * py0;
      phi[4 * k + 2] = px0 * py1;
      phi[4 * k + 3] = px1 * py1;
      ++k;
    }
  }
}

// Quadrature weight factor of point k in the cell (the ww prefactor without
// the coefficient value): transport_system.cpp:27 / :45, dg_space.cpp:41 / :59.
double point_weight(const Mesh& m, int cell, int nq, const double* gw, int k) {
  if (m.geom == 0) return 0.5 * m.width(cell) * gw[k];
  const int qy = k / nq, qx = k % nq;
  return 0.25 * m.hx() * m.hy() * gw[qx] * gw[qy];
}

// 2x2 inverse in the closed form a fixed-size inverse uses (adjugate / det).
void inv2(const double* a, double* o) {
  const double det = a[0] * a[3] - a[2] * a[1];
  const double id = 1.0 / det;
  o[0] = a[3] * id;
  o[1] = -a[1] * id;
  o[2] = -a[2] * id;
  o[3] = a[0] * id;
}

// 4x4 inverse by cofactor expansion (row-major in/out).
void inv4(const double* m, double* inv) {
  double c[16];
  c[0] = m[5] * m[10] * m[15] - m[5] * m[11] * m[14] - m[9] * m[6] * m[15] + m[9] * m[7] * m[14] +
         m[13] * m[6] * m[11] - m[13] * m[7] * m[10];
  c[4] = -m[4] * m[10] * m[15] + m[4] * m[11] * m[14] + m[8] * m[6] * m[15] - m[8] * m[7] * m[14] -
         m[12] * m[6] * m[11] + m[12] * m[7] * m[10];
  c[8] = m[4] * m[9] * m[15] - m[4] * m[11] * m[13] - m[8] * m[5] * m[15] + m[8] * m[7] * m[13] +
         m[12] * m[5] * m[11] - m[12] * m[7] * m[9];
  c[12] = -m[4] * m[9] * m[14] + m[4] * m[10] * m[13] + m[8] * m[5] * m[14] - m[8] * m[6] * m[13] -
          m[12] * m[5] * m[10] + m[12] * m[6] * m[9];
  c[1] = -m[1] * m[10] * m[15] + m[1] * m[11] * m[14] + m[9] * m[2] * m[15] - m[9] * m[3] * m[14] -
         m[13] * m[2] * m[11] + m[13] * m[3] * m[10];
  c[5] = m[0] * m[10] * m[15] - m[0] * m[11] * m[14] - m[8] * m[2] * m[15] + m[8] * m[3] * m[14] +
         m[12] * m[2] * m[11] - m[12] * m[3] * m[10];
  c[9] = -m[0] * m[9] * m[15] + m[0] * m[11] * m[13] + m[8] * m[1] * m[15] - m[8] * m[3] * m[13] -
         m[12] * m[1] * m[11] + m[12] * m[3] * m[9];
  c[13] = m[0] * m[9] * m[14] - m[0] * m[10] * m[13] - m[8] * m[1] * m[14] + m[8] * m[2] * m[13] +
          m[12] * m[1] * m[10] - m[12] * m[2] * m[9];
  c[2] = m[1] * m[6] * m[15] - m[1] * m[7] * m[14] - m[5] * m[2] * m[15] + m[5] * m[3] * m[14] +
         m[13] * m[2] * m[7] - m[13] * m[3] * m[6];
  c[6] = -m[0] * m[6] * m[15] + m[0] * m[7] * m[14] + m[4] * m[2] * m[15] - m[4] * m[3] * m[14] -
         m[12] * m[2] * m[7] + m[12] * m[3] * m[6];
  c[10] = m[0] * m[5] * m[15] - m[0] * m[7] * m[13] - m[4] * m[1] * m[15] + m[4] * m[3] * m[13] +
          m[12] * m[1] * m[7] - m[12] * m[3] * m[5];
  c[14] = -m[0] * m[5] * m[14] + m[0] * m[6] * m[13] + m[4] * m[1] * m[14] - m[4] * m[2] * m[13] -
          m[12] * m[1] * m[6] + m[12] * m[2] * m[5];
  c[3] = -m[1] * m[6] * m[11] + m[1] * m[7] * m[10] + m[5] * m[2] * m[11] - m[5] * m[3] * m[10] -
         m[9] * m[2] * m[7] + m[9] * m[3] * m[6];
  c[7] = m[0] * m[6] * m[11] - m[0] * m[7] * m[10] - m[4] * m[2] * m[11] + m[4] * m[3] * m[10] +
         m[8] * m[2] * m[7] - m[8] * m[3] * m[6];
  c[11] = -m[0] * m[5] * m[11] + m[0] * m[7] * m[9] + m[4] * m[1] * m[11] - m[4] * m[3] * m[9] -
          m[8] * m[1] * m[7] + m[8] * m[3] * m[5];
  c[15] = m[0] * m[5] * m[10] - m[0] * m[6] * m[9] - m[4] * m[1] * m[10] + m[4] * m[2] * m[9] +
          m[8] * m[1] * m[6] - m[8] * m[2] * m[5];
  const double det = m[0] * c[0] + m[1] * c[4] + m[2] * c[8] + m[3] * c[12];
  const double id = 1.0 / det;
  for (int i = 0; i < 16; ++i) inv[i] = c[i] * id;
}

// transport_system.cpp:58-78 -- upwind per-cell 1D streaming block for speed v
// on width h (row-major 2x2): v>0: v(E_R - S); v<=0: v(-E_L - S).
void stream_block(double v, double h, double* o) {
  if (v > 0) {
    o[0] = v * (1.0 / h - 0.0);
    o[1] = v * (kS3 / h - 0.0);
    o[2] = v * (kS3 / h - 2.0 * kS3 / h);
    o[3] = v * (3.0 / h - 0.0);
  } else {
    o[0] = v * (-(1.0 / h) - 0.0);
    o[1] = v * (-(-kS3 / h) - 0.0);
    o[2] = v * (-(-kS3 / h) - 2.0 * kS3 / h);
    o[3] = v * (-(3.0 / h) - 0.0);
  }
}

// Largest per-slot inverse cache (bytes) the oracle builds (ro_set_cache_budget).
double g_cache_budget = 4.0e9;

struct BcEntry {
  int cell;
  double v[4];
};

struct System {
  Mesh mesh;
  int nl = 2;
  long ndof = 0;
  int nv = 0;
  std::vector<double> vx, vy, vz, w;
  int nterms = 0;
  std::vector<double> psi;
  std::vector<double> tmt, tms;  // [k][cell][nl*nl]
  std::vector<double> mt, ms;    // [cell][nl*nl]
  std::vector<double> g;         // n_dof
  double inflow[4] = {0, 0, 0, 0};
  std::vector<std::vector<BcEntry>> bc;
  std::vector<int> slot;
  int nslots = 0;
  std::vector<std::vector<double>> inv;   // per slot: cached inverses, or empty (computed per cell on the fly)
  std::vector<std::array<double, 16>> gm; // xy: per-slot streaming block g (transport_system.cpp:239-250)
  std::vector<double> trL, trR;  // slab: [cell][2]
  double bxL[2], bxR[2], byL[2], byR[2];

  int nb() const { return nl * nl; }

  // transport_system.cpp:142-187
  void build_bc() {
    bc.assign(nv, {});
    if (mesh.geom == 0) {
      const int n = mesh.cells();
      const double h0 = mesh.width(0), hn = mesh.width(n - 1);
      for (int j = 0; j < nv; ++j) {
        const double v = vx[j];
        if (v > 0 && inflow[0] != 0) {
          const double a = v * inflow[0] / std::sqrt(h0);
          bc[j].push_back({0, {a, -kS3 * a, 0, 0}});
        } else if (v < 0 && inflow[1] != 0) {
          const double a = -v * inflow[1] / std::sqrt(hn);
          bc[j].push_back({n - 1, {a, kS3 * a, 0, 0}});
        }
      }
      return;
    }
    const int nx = mesh.nx, ny = mesh.ny;
    const double hx = mesh.hx(), hy = mesh.hy();
    const double sx = 1.0 / std::sqrt(hx), sy = 1.0 / std::sqrt(hy);
    for (int j = 0; j < nv; ++j) {
      if (vx[j] > 0 && inflow[0] != 0) {
        const double a = vx[j] * inflow[0] * sx * std::sqrt(hy);
        for (int iy = 0; iy < ny; ++iy) bc[j].push_back({nx * iy, {a, -kS3 * a, 0, 0}});
      }
      if (vx[j] < 0 && inflow[1] != 0) {
        const double a = -vx[j] * inflow[1] * sx * std::sqrt(hy);
        for (int iy = 0; iy < ny; ++iy) bc[j].push_back({nx - 1 + nx * iy, {a, kS3 * a, 0, 0}});
      }
      if (vy[j] > 0 && inflow[2] != 0) {
        const double a = vy[j] * inflow[2] * sy * std::sqrt(hx);
        for (int ix = 0; ix < nx; ++ix) bc[j].push_back({ix, {a, 0, -kS3 * a, 0}});
      }
      if (vy[j] < 0 && inflow[3] != 0) {
        const double a = -vy[j] * inflow[3] * sy * std::sqrt(hx);
        for (int ix = 0; ix < nx; ++ix) bc[j].push_back({ix + nx * (ny - 1), {a, 0, kS3 * a, 0}});
      }
    }
  }

  // transport_system.cpp:189-261 -- slots keyed by (vx,vy), first-appearance
  // numbering; per slot and cell the explicit inverse of (streaming + Mt).
  void build_cache() {
    const int nc = mesh.cells();
    slot.assign(nv, -1);
    std::map<std::pair<double, double>, int> slot_of;
    for (int j = 0; j < nv; ++j) {
      auto key = std::make_pair(vx[j], vy[j]);
      auto it = slot_of.find(key);
      if (it == slot_of.end()) it = slot_of.emplace(key, (int)slot_of.size()).first;
      slot[j] = it->second;
    }
    nslots = (int)slot_of.size();
    inv.assign(slot_of.size(), {});
    if (mesh.geom == 0) {
      trL.resize(2 * nc);
      trR.resize(2 * nc);
      for (int i = 0; i < nc; ++i) {
        const double s = 1.0 / std::sqrt(mesh.width(i));
        trL[2 * i] = s;
        trL[2 * i + 1] = -kS3 * s;
        trR[2 * i] = s;
        trR[2 * i + 1] = kS3 * s;
      }
      for (const auto& kv : slot_of) {
        const double v = kv.first.first;
        auto& flat = inv[kv.second];
        flat.resize(4 * (size_t)nc);
        for (int i = 0; i < nc; ++i) {
          double b[4];
          stream_block(v, mesh.width(i), b);
          for (int e = 0; e < 4; ++e) b[e] += mt[4 * i + e];
          inv2(b, flat.data() + 4 * i);
        }
      }
      return;
    }
    const double hx = mesh.hx(), hy = mesh.hy();
    const double rx = 1.0 / std::sqrt(hx), ry = 1.0 / std::sqrt(hy);
    bxL[0] = rx; bxL[1] = -kS3 * rx;
    bxR[0] = rx; bxR[1] = kS3 * rx;
    byL[0] = ry; byL[1] = -kS3 * ry;
    byR[0] = ry; byR[1] = kS3 * ry;
    gm.assign(slot_of.size(), {});
    for (const auto& kv : slot_of) {
      double bx[4], by[4];
      stream_block(kv.first.first, hx, bx);
      stream_block(kv.first.second, hy, by);
      double* g = gm[kv.second].data();
      for (int e = 0; e < 16; ++e) g[e] = 0.0;
      for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a)
          for (int a2 = 0; a2 < 2; ++a2) g[4 * (a + 2 * b) + (a2 + 2 * b)] += bx[2 * a + a2];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
          for (int b2 = 0; b2 < 2; ++b2) g[4 * (a + 2 * b) + (a + 2 * b2)] += by[2 * b + b2];
    }
    // The reference caches 16 doubles per slot and cell (34 GB per sample at
    // 1024^2 x 256 slots).  Above the budget the oracle computes the same
    // inverse (same operands, same inv4) per cell when it sweeps instead.
    if ((double)nslots * nc * 16 * 8 <= g_cache_budget)
      for (int k = 0; k < nslots; ++k) cache_slot(k);
  }

  // transport_system.cpp:251-259 for one slot: inverse of g + Mt_c per cell
  void cache_slot(int k) {
    const int nc = mesh.cells();
    auto& flat = inv[k];
    flat.resize(16 * (size_t)nc);
    for (int c = 0; c < nc; ++c) cell_inverse(k, c, flat.data() + 16 * c);
  }
  void cell_inverse(int k, int c, double* out) const {
    double bm[16];
    const double* g = gm[k].data();
    for (int e = 0; e < 16; ++e) bm[e] = g[e] + mt[16 * (size_t)c + e];
    inv4(bm, out);
  }

  // transport_system.cpp:276-364
  void sweep(int j, const double* rhs, double* f) const {
    const double* iv = inv[slot[j]].data();
    const bool lazy = inv[slot[j]].empty();
    if (mesh.geom == 0) {
      const int n = mesh.cells();
      const double v = vx[j];
      if (v > 0) {
        for (int i = 0; i < n; ++i) {
          double r0 = rhs[2 * i], r1 = rhs[2 * i + 1];
          if (i > 0) {
            const double u = f[2 * i - 2] * trR[2 * (i - 1)] + f[2 * i - 1] * trR[2 * (i - 1) + 1];
            r0 += v * u * trL[2 * i];
            r1 += v * u * trL[2 * i + 1];
          }
          const double* b = iv + 4 * i;
          f[2 * i] = b[0] * r0 + b[1] * r1;
          f[2 * i + 1] = b[2] * r0 + b[3] * r1;
        }
      } else {
        for (int i = n - 1; i >= 0; --i) {
          double r0 = rhs[2 * i], r1 = rhs[2 * i + 1];
          if (i < n - 1) {
            const double u = f[2 * i + 2] * trL[2 * (i + 1)] + f[2 * i + 3] * trL[2 * (i + 1) + 1];
            r0 -= v * u * trR[2 * i];
            r1 -= v * u * trR[2 * i + 1];
          }
          const double* b = iv + 4 * i;
          f[2 * i] = b[0] * r0 + b[1] * r1;
          f[2 * i + 1] = b[2] * r0 + b[3] * r1;
        }
      }
      return;
    }
    const int nx = mesh.nx, ny = mesh.ny;
    const double ux = vx[j], uy = vy[j];
    const int sx = ux > 0 ? 1 : -1, sy = uy > 0 ? 1 : -1;
    const int ix0 = sx > 0 ? 0 : nx - 1, iy0 = sy > 0 ? 0 : ny - 1;
    for (int ky = 0; ky < ny; ++ky) {
      const int iy = iy0 + sy * ky;
      for (int kx = 0; kx < nx; ++kx) {
        const int ix = ix0 + sx * kx;
        const int cell = ix + nx * iy;
        double r[4] = {rhs[4 * cell], rhs[4 * cell + 1], rhs[4 * cell + 2], rhs[4 * cell + 3]};
        if (kx > 0) {
          const double* cu = f + 4 * (ix - sx + nx * iy);
          for (int b = 0; b < 2; ++b) {
            if (sx > 0) {
              const double u = cu[2 * b] * bxR[0] + cu[2 * b + 1] * bxR[1];
              r[2 * b] += ux * u * bxL[0];
              r[2 * b + 1] += ux * u * bxL[1];
            } else {
              const double u = cu[2 * b] * bxL[0] + cu[2 * b + 1] * bxL[1];
              r[2 * b] -= ux * u * bxR[0];
              r[2 * b + 1] -= ux * u * bxR[1];
            }
          }
        }
        if (ky > 0) {
          const double* cu = f + 4 * (ix + nx * (iy - sy));
          for (int a = 0; a < 2; ++a) {
            if (sy > 0) {
              const double u = cu[a] * byR[0] + cu[a + 2] * byR[1];
              r[a] += uy * u * byL[0];
              r[a + 2] += uy * u * byL[1];
            } else {
              const double u = cu[a] * byL[0] + cu[a + 2] * byL[1];
              r[a] -= uy * u * byR[0];
              r[a + 2] -= uy * u * byR[1];
            }
          }
        }
        double bl[16];
        const double* b = bl;
        if (lazy)
          cell_inverse(slot[j], cell, bl);
        else
          b = iv + 16 * (size_t)cell;
        double* fc = f + 4 * cell;
        for (int k = 0; k < 4; ++k)
          fc[k] = b[4 * k] * r[0] + b[4 * k + 1] * r[1] + b[4 * k + 2] * r[2] + b[4 * k + 3] * r[3];
      }
    }
  }

  // transport_system.cpp:263-268
  void add_bc(int j, double* rhs) const {
    for (const auto& e : bc[j])
      for (int k = 0; k < nl; ++k) rhs[(long)e.cell * nl + k] += e.v[k];
  }

  // transport_system.cpp:373-391 (per-cell block times segment)
  void apply_block(const std::vector<double>& blocks, const double* x, double* o) const {
    const int nc = mesh.cells(), b = nb();
    for (int c = 0; c < nc; ++c) {
      const double* m = blocks.data() + (long)b * c;
      const double* xs = x + (long)nl * c;
      double* os = o + (long)nl * c;
      for (int r = 0; r < nl; ++r) {
        double s = m[nl * r] * xs[0];
        for (int k = 1; k < nl; ++k) s += m[nl * r + k] * xs[k];
        os[r] = s;
      }
    }
  }

  bool cached() const {
    for (const auto& v : inv)
      if (v.empty()) return false;
    return true;
  }

  // Uncached (large) problems: slot-major over threads.  The directions of a
  // slot share (vx, vy), so their sweeps of a common right-hand side are the
  // same arithmetic; each slot is swept once and every direction of it
  // accumulated (w_j f, j ascending within the slot) into the thread's partial
  // sum; the partials are added in thread order.  Differs from the
  // reference's j-ordered sum only in the order of the final additions.
  // rhs_of(j, buf) returns the right-hand side of direction j.
  template <typename Rhs>
  void accumulate_slots(Rhs rhs_of, double* out) const {
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    std::vector<std::vector<double>> part(nt);
#pragma omp parallel num_threads(nt)
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      std::vector<double>& acc = part[t];
      acc.assign(ndof, 0.0);
      std::vector<double> f(ndof), rhs(ndof);
#pragma omp for schedule(static)
      for (int k = 0; k < nslots; ++k) {
        int j0 = -1;
        for (int j = 0; j < nv; ++j)
          if (slot[j] == k) {
            j0 = j;
            break;
          }
        const double* r = rhs_of(j0, rhs);
        sweep(j0, r, f.data());
        for (int j = 0; j < nv; ++j)
          if (slot[j] == k)
            for (long i = 0; i < ndof; ++i) acc[i] += w[j] * f[i];
      }
    }
    std::fill(out, out + ndof, 0.0);
    for (int t = 0; t < nt; ++t)
      for (long i = 0; i < ndof; ++i) out[i] += part[t][i];
  }

  // transport_system.cpp:393-404
  void apply_L(const double* rho, double* out) const {
    std::vector<double> q(ndof), f(ndof);
    apply_block(ms, rho, q.data());
    if (!cached()) {
      accumulate_slots([&](int, std::vector<double>&) { return (const double*)q.data(); }, out);
      return;
    }
    std::fill(out, out + ndof, 0.0);
    for (int j = 0; j < nv; ++j) {
      sweep(j, q.data(), f.data());
      for (long i = 0; i < ndof; ++i) out[i] += w[j] * f[i];
    }
  }

  // transport_system.cpp:406-418
  void assemble_rhs(double* out) const {
    if (!cached()) {
      accumulate_slots(
          [&](int j, std::vector<double>& buf) {
            buf = g;
            add_bc(j, buf.data());
            return (const double*)buf.data();
          },
          out);
      return;
    }
    std::vector<double> rhs(ndof), f(ndof);
    std::fill(out, out + ndof, 0.0);
    for (int j = 0; j < nv; ++j) {
      rhs = g;
      add_bc(j, rhs.data());
      sweep(j, rhs.data(), f.data());
      for (long i = 0; i < ndof; ++i) out[i] += w[j] * f[i];
    }
  }

  // The reference's apply_L restricted to directions [j0, j1) (transport_
  // system.cpp:398-401): out += w_j f_j in j order.  CPU baseline timing of
  // the reference's per-direction sweep cost on a bounded sample.
  void apply_L_dirs(const double* rho, double* out, int j0, int j1) const {
    std::vector<double> q(ndof), f(ndof);
    apply_block(ms, rho, q.data());
    std::fill(out, out + ndof, 0.0);
    for (int j = j0; j < j1; ++j) {
      sweep(j, q.data(), f.data());
      for (long i = 0; i < ndof; ++i) out[i] += w[j] * f[i];
    }
  }

  // transport_system.cpp:420-431
  void kinetic_sweep(const double* rho, double* f) const {
    std::vector<double> q0(ndof), rhs(ndof);
    apply_block(ms, rho, q0.data());
    for (long i = 0; i < ndof; ++i) q0[i] += g[i];
    for (int j = 0; j < nv; ++j) {
      rhs = q0;
      add_bc(j, rhs.data());
      sweep(j, rhs.data(), f + (long)j * ndof);
    }
  }

  // transport_system.cpp:433-441
  void density_of(const double* f, double* rho) const {
    std::fill(rho, rho + ndof, 0.0);
    for (int j = 0; j < nv; ++j)
      for (long i = 0; i < ndof; ++i) rho[i] += w[j] * f[(long)j * ndof + i];
  }

  // transport_system.cpp:446-478 -- D_j f for one slab direction block.
  void apply_dj_1d(double v, const double* f, double* out) const {
    const int n = mesh.cells();
    if (v > 0) {
      for (int i = 0; i < n; ++i) {
        const double h = mesh.width(i);
        const double fr = f[2 * i] * trR[2 * i] + f[2 * i + 1] * trR[2 * i + 1];
        out[2 * i] = v * fr * trR[2 * i];
        out[2 * i + 1] = v * (fr * trR[2 * i + 1] - 2.0 * kS3 / h * f[2 * i]);
        if (i > 0) {
          const double u = f[2 * i - 2] * trR[2 * (i - 1)] + f[2 * i - 1] * trR[2 * (i - 1) + 1];
          out[2 * i] -= v * u * trL[2 * i];
          out[2 * i + 1] -= v * u * trL[2 * i + 1];
        }
      }
    } else {
      for (int i = 0; i < n; ++i) {
        const double h = mesh.width(i);
        const double fl = f[2 * i] * trL[2 * i] + f[2 * i + 1] * trL[2 * i + 1];
        out[2 * i] = -v * fl * trL[2 * i];
        out[2 * i + 1] = -v * (fl * trL[2 * i + 1] + 2.0 * kS3 / h * f[2 * i]);
        if (i < n - 1) {
          const double u = f[2 * i + 2] * trL[2 * (i + 1)] + f[2 * i + 3] * trL[2 * (i + 1) + 1];
          out[2 * i] += v * u * trR[2 * i];
          out[2 * i + 1] += v * u * trR[2 * i + 1];
        }
      }
    }
  }

  // transport_system.cpp:482-558 -- (D_j + Sigma_t) f for one direction.
  void apply_sc(int j, const double* f, double* out) const {
    if (mesh.geom == 0) {
      apply_dj_1d(vx[j], f, out);
    } else {
      const int nx = mesh.nx, ny = mesh.ny;
      const double ux = vx[j], uy = vy[j];
      const double hx = mesh.hx(), hy = mesh.hy();
      for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) {
          const int cell = ix + nx * iy;
          const double* fc = f + 4 * cell;
          double* oc = out + 4 * cell;
          for (int k = 0; k < 4; ++k) oc[k] = 0;
          for (int b = 0; b < 2; ++b) {
            const double c0 = fc[2 * b], c1 = fc[2 * b + 1];
            if (ux > 0) {
              const double fr = c0 * bxR[0] + c1 * bxR[1];
              oc[2 * b] += ux * fr * bxR[0];
              oc[2 * b + 1] += ux * (fr * bxR[1] - 2.0 * kS3 / hx * c0);
              if (ix > 0) {
                const double* cu = f + 4 * (cell - 1);
                const double u = cu[2 * b] * bxR[0] + cu[2 * b + 1] * bxR[1];
                oc[2 * b] -= ux * u * bxL[0];
                oc[2 * b + 1] -= ux * u * bxL[1];
              }
            } else {
              const double fl = c0 * bxL[0] + c1 * bxL[1];
              oc[2 * b] += -ux * fl * bxL[0];
              oc[2 * b + 1] += -ux * (fl * bxL[1] + 2.0 * kS3 / hx * c0);
              if (ix < nx - 1) {
                const double* cu = f + 4 * (cell + 1);
                const double u = cu[2 * b] * bxL[0] + cu[2 * b + 1] * bxL[1];
                oc[2 * b] += ux * u * bxR[0];
                oc[2 * b + 1] += ux * u * bxR[1];
              }
            }
          }
          for (int a = 0; a < 2; ++a) {
            const double c0 = fc[a], c1 = fc[a + 2];
            if (uy > 0) {
              const double fr = c0 * byR[0] + c1 * byR[1];
              oc[a] += uy * fr * byR[0];
              oc[a + 2] += uy * (fr * byR[1] - 2.0 * kS3 / hy * c0);
              if (iy > 0) {
                const double* cu = f + 4 * (cell - nx);
                const double u = cu[a] * byR[0] + cu[a + 2] * byR[1];
                oc[a] -= uy * u * byL[0];
                oc[a + 2] -= uy * u * byL[1];
              }
            } else {
              const double fl = c0 * byL[0] + c1 * byL[1];
              oc[a] += -uy * fl * byL[0];
              oc[a + 2] += -uy * (fl * byL[1] + 2.0 * kS3 / hy * c0);
              if (iy < ny - 1) {
                const double* cu = f + 4 * (cell + nx);
                const double u = cu[a] * byL[0] + cu[a + 2] * byL[1];
                oc[a] += uy * u * byR[0];
                oc[a + 2] += uy * u * byR[1];
              }
            }
          }
        }
    }
    std::vector<double> tmp(ndof);
    apply_block(mt, f, tmp.data());
    for (long i = 0; i < ndof; ++i) out[i] += tmp[i];
  }

  // transport_system.cpp:560-596
  void apply_term_kinetic(int k, const double* u, double* out) const {
    std::vector<double> avg(ndof), dju(ndof), tmp(ndof);
    density_of(u, avg.data());
    const int b = nb();
    for (int j = 0; j < nv; ++j) {
      const double* uj = u + (long)j * ndof;
      double* oj = out + (long)j * ndof;
      if (k == 0) {
        if (mesh.geom == 0) {
          apply_dj_1d(vx[j], uj, dju.data());
          std::copy(dju.begin(), dju.end(), oj);
        } else {
          apply_sc(j, uj, dju.data());
          std::copy(dju.begin(), dju.end(), oj);
          apply_block(mt, uj, tmp.data());
          for (long i = 0; i < ndof; ++i) oj[i] -= tmp[i];
        }
      } else {
        std::fill(oj, oj + ndof, 0.0);
      }
      const int nc = mesh.cells();
      for (int c = 0; c < nc; ++c) {
        const double* mtk = tmt.data() + ((long)k * nc + c) * b;
        const double* msk = tms.data() + ((long)k * nc + c) * b;
        for (int r = 0; r < nl; ++r) {
          double s1 = 0, s2 = 0;
          for (int q = 0; q < nl; ++q) {
            s1 += mtk[nl * r + q] * uj[(long)nl * c + q];
            s2 += msk[nl * r + q] * avg[(long)nl * c + q];
          }
          oj[(long)nl * c + r] += s1;
          oj[(long)nl * c + r] -= s2;
        }
      }
    }
  }

  // transport_system.cpp:598-613
  void apply_kinetic(const double* u, double* out) const {
    std::vector<double> avg(ndof), tmp(ndof), m(ndof);
    density_of(u, avg.data());
    apply_block(ms, avg.data(), m.data());
    for (int j = 0; j < nv; ++j) {
      apply_sc(j, u + (long)j * ndof, tmp.data());
      double* oj = out + (long)j * ndof;
      for (long i = 0; i < ndof; ++i) oj[i] = tmp[i] - m[i];
    }
  }

  // transport_system.cpp:615-624
  void kinetic_rhs(double* b) const {
    for (int j = 0; j < nv; ++j) {
      double* bj = b + (long)j * ndof;
      std::copy(g.begin(), g.end(), bj);
      add_bc(j, bj);
    }
  }
};

// ---------------------------------------------------------------------------
// dsa.cpp -- consistent DSA assembly, as sparse triplet lists.
struct Trip {
  long r, c;
  double v;
};

// Sparse matrix as an ordered map (row, col) -> value; duplicate triplets sum
// like setFromTriplets (dsa.cpp:166-169).
using SpMap = std::map<std::pair<long, long>, double>;

void sp_add(SpMap& m, long r, long c, double v) { m[{r, c}] += v; }

SpMap sp_lin(const SpMap& a, double sa, const SpMap& b, double sb) {
  SpMap o;
  for (const auto& e : a) o[e.first] += sa * e.second;
  for (const auto& e : b) o[e.first] += sb * e.second;
  return o;
}

// dsa.cpp:34-110 -- per-axis upwind (dp) and downwind (dm) streaming
// matrices on the DG space.
void axis_streaming(const Mesh& mesh, int nl, int axis, SpMap& dp, SpMap& dm) {
  auto add_block = [&](SpMap& t, int cr, int cc, const double* m2) {
    if (nl == 2) {
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) sp_add(t, (long)cr * 2 + k, (long)cc * 2 + l, m2[2 * k + l]);
      return;
    }
    for (int other = 0; other < 2; ++other)
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) {
          const int lr = axis == 0 ? k + 2 * other : other + 2 * k;
          const int lc = axis == 0 ? l + 2 * other : other + 2 * l;
          sp_add(t, (long)cr * 4 + lr, (long)cc * 4 + lc, m2[2 * k + l]);
        }
  };
  auto edge = [](double h, double* er, double* el, double* s) {
    er[0] = 1 / h; er[1] = kS3 / h; er[2] = kS3 / h; er[3] = 3 / h;
    el[0] = 1 / h; el[1] = -kS3 / h; el[2] = -kS3 / h; el[3] = 3 / h;
    s[0] = 0; s[1] = 0; s[2] = 2.0 * kS3 / h; s[3] = 0;
  };
  double er[4], el[4], s[4], blk[4];
  if (mesh.geom == 0) {
    const int nc = mesh.cells();
    for (int i = 0; i < nc; ++i) {
      const double h = mesh.width(i);
      edge(h, er, el, s);
      for (int e = 0; e < 4; ++e) blk[e] = er[e] - s[e];
      add_block(dp, i, i, blk);
      for (int e = 0; e < 4; ++e) blk[e] = -el[e] - s[e];
      add_block(dm, i, i, blk);
      if (i > 0) {
        const double si = 1.0 / std::sqrt(h), su = 1.0 / std::sqrt(mesh.width(i - 1));
        const double cpl[4] = {si * su, si * kS3 * su, -kS3 * si * su, -3 * si * su};
        for (int e = 0; e < 4; ++e) blk[e] = -cpl[e];
        add_block(dp, i, i - 1, blk);
      }
      if (i < nc - 1) {
        const double si = 1.0 / std::sqrt(h), su = 1.0 / std::sqrt(mesh.width(i + 1));
        const double cpl[4] = {si * su, -si * kS3 * su, kS3 * si * su, -3 * si * su};
        add_block(dm, i, i + 1, cpl);
      }
    }
    return;
  }
  const int nx = mesh.nx, ny = mesh.ny;
  const double h = axis == 0 ? mesh.hx() : mesh.hy();
  edge(h, er, el, s);
  const double cl[4] = {1 / h, kS3 / h, -kS3 / h, -3 / h};
  const double cr[4] = {1 / h, -kS3 / h, kS3 / h, -3 / h};
  double ncl[4];
  for (int e = 0; e < 4; ++e) ncl[e] = -cl[e];
  double dpb[4], dmb[4];
  for (int e = 0; e < 4; ++e) {
    dpb[e] = er[e] - s[e];
    dmb[e] = -el[e] - s[e];
  }
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix) {
      const int cell = ix + nx * iy;
      add_block(dp, cell, cell, dpb);
      add_block(dm, cell, cell, dmb);
      const int i_ax = axis == 0 ? ix : iy;
      const int n_ax = axis == 0 ? nx : ny;
      const int stride = axis == 0 ? 1 : nx;
      if (i_ax > 0) add_block(dp, cell, cell - stride, ncl);
      if (i_ax < n_ax - 1) add_block(dm, cell, cell + stride, cr);
    }
}

struct Dsa {
  long n = 0;
  int nf = 2;
  // Blocks in the reference's field-major ordering (dsa.cpp:200-212).
  SpMap a_rr;
  std::vector<SpMap> a_rj, a_jr, t_blocks;
};

// dsa.cpp:154-258 (assembly only; the factorization is done by the caller)
Dsa build_dsa(const System& sys) {
  Dsa d;
  d.n = sys.ndof;
  const bool slab = sys.mesh.geom == 0;
  d.nf = slab ? 2 : 3;
  const int nl = sys.nl, nb = sys.nb(), nc = sys.mesh.cells();
  // dsa.cpp:112-127 -- block-diagonal masses; zero entries skipped.
  SpMap ma, mt;
  for (int c = 0; c < nc; ++c)
    for (int k = 0; k < nl; ++k)
      for (int l = 0; l < nl; ++l) {
        const double vt = sys.mt[(long)nb * c + nl * k + l];
        const double va = vt - sys.ms[(long)nb * c + nl * k + l];
        if (va != 0) sp_add(ma, (long)nl * c + k, (long)nl * c + l, va);
        if (vt != 0) sp_add(mt, (long)nl * c + k, (long)nl * c + l, vt);
      }
  // dsa.cpp:167-192 -- angular moments over the transport quadrature.
  auto s1 = [&](const std::vector<double>& cmp) {
    double s = 0;
    for (int j = 0; j < sys.nv; ++j)
      if (cmp[j] > 0) s += sys.w[j] * cmp[j];
    return s;
  };
  auto s2 = [&](const std::vector<double>& cmp) {
    double s = 0;
    for (int j = 0; j < sys.nv; ++j) s += sys.w[j] * cmp[j] * cmp[j];
    return s;
  };
  auto s3 = [&](const std::vector<double>& cmp) {
    double s = 0;
    for (int j = 0; j < sys.nv; ++j)
      if (cmp[j] > 0) s += sys.w[j] * cmp[j] * cmp[j] * cmp[j];
    return s;
  };
  auto s3m = [&](const std::vector<double>& sq, const std::vector<double>& pos) {
    double s = 0;
    for (int j = 0; j < sys.nv; ++j)
      if (pos[j] > 0) s += sys.w[j] * sq[j] * sq[j] * pos[j];
    return s;
  };
  if (slab) {
    SpMap dp, dm;
    axis_streaming(sys.mesh, nl, 0, dp, dm);
    SpMap dj = sp_lin(dm, 1.0, dp, -1.0);
    SpMap dc = sp_lin(dp, 0.5, dm, 0.5);
    const double m1 = s1(sys.vx), m2 = s2(sys.vx), m3 = s3(sys.vx);
    d.a_rr = sp_lin(ma, 1.0, dj, -m1);
    d.a_rj = {sp_lin(dc, 3.0 * m2, SpMap{}, 0)};
    d.a_jr = {sp_lin(dc, m2, SpMap{}, 0)};
    d.t_blocks = {sp_lin(mt, 3.0 * m2, dj, -3.0 * m3)};
  } else {
    SpMap dpx, dmx, dpy, dmy;
    axis_streaming(sys.mesh, nl, 0, dpx, dmx);
    axis_streaming(sys.mesh, nl, 1, dpy, dmy);
    SpMap djx = sp_lin(dmx, 1.0, dpx, -1.0), djy = sp_lin(dmy, 1.0, dpy, -1.0);
    SpMap dcx = sp_lin(dpx, 0.5, dmx, 0.5), dcy = sp_lin(dpy, 0.5, dmy, 0.5);
    const double m1x = s1(sys.vx), m2x = s2(sys.vx), m3x = s3(sys.vx);
    const double m1y = s1(sys.vy), m2y = s2(sys.vy), m3y = s3(sys.vy);
    const double m3yx = s3m(sys.vx, sys.vy), m3xy = s3m(sys.vy, sys.vx);
    d.a_rr = sp_lin(sp_lin(ma, 1.0, djx, -m1x), 1.0, djy, -m1y);
    d.a_rj = {sp_lin(dcx, 3.0 * m2x, SpMap{}, 0), sp_lin(dcy, 3.0 * m2y, SpMap{}, 0)};
    d.a_jr = {sp_lin(dcx, m2x, SpMap{}, 0), sp_lin(dcy, m2y, SpMap{}, 0)};
    d.t_blocks = {sp_lin(sp_lin(mt, 3.0 * m2x, djx, -3.0 * m3x), 1.0, djy, -3.0 * m3yx),
                  sp_lin(sp_lin(mt, 3.0 * m2y, djy, -3.0 * m3y), 1.0, djx, -3.0 * m3xy)};
  }
  return d;
}

struct DsaHandle {
  Dsa d;
  std::vector<Trip> coupled;  // reference ordering (dsa.cpp:272-305)
  std::vector<double> moments;
};

void append(std::vector<Trip>& t, const SpMap& m, long r0, long c0) {
  for (const auto& e : m) t.push_back({r0 + e.first.first, c0 + e.first.second, e.second});
}

}  // namespace

// ===========================================================================
// C API (ctypes).  Status: 0 ok, nonzero error (message via ro_last_error).
extern "C" {

const char* ro_last_error() { return g_err.c_str(); }

void ro_gauss_legendre_nodes(int n, double* x, double* w) { gl_nodes(n, x, w); }

// cases.cpp:11-13 -- unit draws of std::mt19937_64.
void ro_unit_draws(unsigned long long seed, long n, double* out) {
  std::mt19937_64 gen(seed);
  for (long i = 0; i < n; ++i) out[i] = static_cast<double>(gen() >> 11) * 0x1p-53;
}

// Evaluation points of the 6-point cell rules (count = cells * nq^d).
int ro_cell_points(int geom, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                   double y1, int nq, double* px, double* py) {
  Mesh m;
  m.geom = geom;
  m.nx = nx;
  m.ny = geom == 0 ? 1 : ny;
  if (geom == 0) m.b.assign(bounds, bounds + nx + 1);
  m.x0 = x0; m.x1 = x1; m.y0 = y0; m.y1 = y1;
  std::vector<double> gx(nq), gw(nq);
  gl_nodes(nq, gx.data(), gw.data());
  cell_points(m, nq, gx.data(), px, py);
  return 0;
}

// dg_space.cpp:31-71 -- L2 projection from values at the cell points.
int ro_project(int geom, int nx, int ny, const double* bounds, double x0, double x1, double y0,
               double y1, int nq, const double* fvals, double* out) {
  Mesh m;
  m.geom = geom;
  m.nx = nx;
  m.ny = geom == 0 ? 1 : ny;
  if (geom == 0) m.b.assign(bounds, bounds + nx + 1);
  m.x0 = x0; m.x1 = x1; m.y0 = y0; m.y1 = y1;
  std::vector<double> gx(nq), gw(nq);
  gl_nodes(nq, gx.data(), gw.data());
  auto p0 = [](double h) { return 1.0 / std::sqrt(h); };
  auto p1 = [](double h, double rel) { return std::sqrt(12.0 / (h * h * h)) * rel; };
  if (geom == 0) {
    for (int i = 0; i < m.nx; ++i) {
      const double h = m.width(i);
      out[2 * i] = out[2 * i + 1] = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double rel = 0.5 * h * gx[q];
        const double wq = 0.5 * h * gw[q];
        const double fv = fvals[(long)i * nq + q];
        out[2 * i] += wq * fv * p0(h);
        out[2 * i + 1] += wq * fv * p1(h, rel);
      }
    }
    return 0;
  }
  const double hx = m.hx(), hy = m.hy();
  const int npc = nq * nq;
  for (int c = 0; c < m.cells(); ++c) {
    double* o = out + 4L * c;
    o[0] = o[1] = o[2] = o[3] = 0.0;
    for (int qy = 0; qy < nq; ++qy) {
      const double ry = 0.5 * hy * gx[qy];
      for (int qx = 0; qx < nq; ++qx) {
        const double rx = 0.5 * hx * gx[qx];
        const double wq = 0.25 * hx * hy * gw[qx] * gw[qy];
        const double fv = fvals[(long)c * npc + qy * nq + qx];
        const double bx0 = p0(hx), bx1 = p1(hx, rx), by0 = p0(hy), by1 = p1(hy, ry);
        o[0] += wq * fv * bx0 * by0;
        o[1] += wq * fv * bx1 * by0;
        o[2] += wq * fv * bx0 * by1;
        o[3] += wq * fv * bx1 * by1;
      }
    }
  }
  return 0;
}

// TransportSystem ctor (transport_system.cpp:82-109).
//   dirs: [nv][3]; psi: [nterms] (psi[0] must be 1);
//   tot_vals/sct_vals: [nterms][cells*npc] coefficient weights at the cell
//   points (absorption+scattering, scattering alone); src_vals: [cells*npc].
void* ro_system_create(int geom, int nx, int ny, const double* bounds, double x0, double x1,
                       double y0, double y1, int nv, const double* dirs, const double* weights,
                       int nterms, const double* psi, const double* tot_vals,
                       const double* sct_vals, const double* src_vals, const double* inflow) {
  try {
    auto* s = new System();
    Mesh& m = s->mesh;
    m.geom = geom;
    m.nx = nx;
    m.ny = geom == 0 ? 1 : ny;
    if (geom == 0) m.b.assign(bounds, bounds + nx + 1);
    m.x0 = x0; m.x1 = x1; m.y0 = y0; m.y1 = y1;
    s->nl = geom == 0 ? 2 : 4;
    s->ndof = (long)m.cells() * s->nl;
    s->nv = nv;
    for (int j = 0; j < nv; ++j) {
      s->vx.push_back(dirs[3 * j]);
      s->vy.push_back(dirs[3 * j + 1]);
      s->vz.push_back(dirs[3 * j + 2]);
      s->w.push_back(weights[j]);
    }
    if (nterms < 1) throw std::invalid_argument("transport system: no coefficient terms");
    s->nterms = nterms;
    s->psi.assign(psi, psi + nterms);
    if (std::abs(s->psi[0] - 1.0) > 0)
      throw std::invalid_argument("transport system: term 0 must be parameter independent (psi == 1)");
    for (int k = 0; k < 4; ++k) s->inflow[k] = inflow[k];
    // build_masses (transport_system.cpp:111-140) with weighted_mass (:17-55)
    const int nq = 6;
    std::vector<double> gx(nq), gw(nq);
    gl_nodes(nq, gx.data(), gw.data());
    const int nc = m.cells(), nl = s->nl, nb = s->nb();
    const int npc = geom == 0 ? nq : nq * nq;
    s->tmt.assign((size_t)nterms * nc * nb, 0.0);
    s->tms.assign((size_t)nterms * nc * nb, 0.0);
    s->mt.assign((size_t)nc * nb, 0.0);
    s->ms.assign((size_t)nc * nb, 0.0);
    std::vector<double> phi;
    for (int k = 0; k < nterms; ++k)
      for (int c = 0; c < nc; ++c) {
        basis_at(m, c, nq, gx.data(), phi);
        double* bt = s->tmt.data() + ((size_t)k * nc + c) * nb;
        double* bs = s->tms.data() + ((size_t)k * nc + c) * nb;
        for (int p = 0; p < npc; ++p) {
          const double pw = point_weight(m, c, nq, gw.data(), p);
          const double wt = pw * tot_vals[((size_t)k * nc + c) * npc + p];
          const double ws = pw * sct_vals[((size_t)k * nc + c) * npc + p];
          for (int r = 0; r < nl; ++r)
            for (int q = 0; q < nl; ++q) {
              bt[nl * r + q] += (wt * phi[nl * p + r]) * phi[nl * p + q];
              bs[nl * r + q] += (ws * phi[nl * p + r]) * phi[nl * p + q];
            }
        }
        for (int e = 0; e < nb; ++e) {
          s->mt[(size_t)c * nb + e] += s->psi[k] * bt[e];
          s->ms[(size_t)c * nb + e] += s->psi[k] * bs[e];
        }
      }
    s->g.assign(s->ndof, 0.0);
    if (src_vals) {
      ro_project(geom, nx, m.ny, bounds, x0, x1, y0, y1, nq, src_vals, s->g.data());
    }
    s->build_bc();
    s->build_cache();
    return s;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ro_system_destroy(void* h) { delete static_cast<System*>(h); }
long ro_n_dof(void* h) { return static_cast<System*>(h)->ndof; }
int ro_n_slots(void* h) { return (int)static_cast<System*>(h)->inv.size(); }
// bytes of per-slot inverse cache built by later ro_system_create calls
void ro_set_cache_budget(double bytes) { g_cache_budget = bytes; }
int ro_is_cached(void* h) { return static_cast<System*>(h)->cached() ? 1 : 0; }
// build the cache of slots [k0, k1) (xy) -- the reference's build_sweep_cache for those slots
void ro_cache_slots(void* h, int k0, int k1) {
  auto* s = static_cast<System*>(h);
  if (s->mesh.geom == 0) return;
  for (int k = k0; k < k1 && k < s->nslots; ++k)
    if (s->inv[k].empty()) s->cache_slot(k);
}
int ro_dir_slot(void* h, int j) { return static_cast<System*>(h)->slot[j]; }
void ro_apply_L_dirs(void* h, const double* rho, double* out, int j0, int j1) {
  static_cast<System*>(h)->apply_L_dirs(rho, out, j0, j1);
}
// CPU baseline timing (bench.py): `nthreads` concurrent copies of the
// reference's per-direction apply_L work (transport_system.cpp:393-404: one
// sweep with the cached per-slot inverse, then out += w_j f), thread t
// sweeping directions dirs[t], dirs[t + nthreads], ... into its own buffers,
// as independent single-threaded reference solves on separate cores would.
// The caches of the slots involved must be built (ro_cache_slots).  Returns
// the wall seconds of the timed region.
double ro_time_sweeps(void* h, const double* rho, const int* dirs, int ndirs, int nthreads) {
  auto* s = static_cast<System*>(h);
  const long nd = s->ndof;
  std::vector<double> q(nd);
  s->apply_block(s->ms, rho, q.data());
  std::vector<std::vector<double>> f(nthreads, std::vector<double>(nd)), out(nthreads, std::vector<double>(nd, 0.0));
  double t0 = 0, t1 = 0;
#ifdef _OPENMP
  t0 = omp_get_wtime();
#pragma omp parallel num_threads(nthreads)
  {
    const int t = omp_get_thread_num();
    for (int k = t; k < ndirs; k += nthreads) {
      const int j = dirs[k];
      s->sweep(j, q.data(), f[t].data());
      for (long i = 0; i < nd; ++i) out[t][i] += s->w[j] * f[t][i];
    }
  }
  t1 = omp_get_wtime();
#else
  (void)nthreads;
  const auto c0 = std::chrono::steady_clock::now();
  for (int k = 0; k < ndirs; ++k) {
    const int j = dirs[k];
    s->sweep(j, q.data(), f[0].data());
    for (long i = 0; i < nd; ++i) out[0][i] += s->w[j] * f[0][i];
  }
  t1 = std::chrono::duration<double>(std::chrono::steady_clock::now() - c0).count();
#endif
  return t1 - t0;
}

void ro_mass_blocks(void* h, double* mt, double* ms) {
  auto* s = static_cast<System*>(h);
  std::copy(s->mt.begin(), s->mt.end(), mt);
  std::copy(s->ms.begin(), s->ms.end(), ms);
}
void ro_term_mass_blocks(void* h, double* tmt, double* tms) {
  auto* s = static_cast<System*>(h);
  std::copy(s->tmt.begin(), s->tmt.end(), tmt);
  std::copy(s->tms.begin(), s->tms.end(), tms);
}
void ro_volumetric_source(void* h, double* g) {
  auto* s = static_cast<System*>(h);
  std::copy(s->g.begin(), s->g.end(), g);
}
void ro_boundary_source(void* h, int j, double* out) {
  auto* s = static_cast<System*>(h);
  std::fill(out, out + s->ndof, 0.0);
  s->add_bc(j, out);
}
void ro_sweep_direction(void* h, int j, const double* rhs, double* f) {
  static_cast<System*>(h)->sweep(j, rhs, f);
}
void ro_apply_sc(void* h, int j, const double* f, double* out) {
  static_cast<System*>(h)->apply_sc(j, f, out);
}
void ro_apply_Ms(void* h, const double* x, double* o) {
  auto* s = static_cast<System*>(h);
  s->apply_block(s->ms, x, o);
}
void ro_apply_Mt(void* h, const double* x, double* o) {
  auto* s = static_cast<System*>(h);
  s->apply_block(s->mt, x, o);
}
void ro_apply_L(void* h, const double* rho, double* out) { static_cast<System*>(h)->apply_L(rho, out); }
void ro_assemble_rhs(void* h, double* out) { static_cast<System*>(h)->assemble_rhs(out); }
void ro_kinetic_sweep(void* h, const double* rho, double* f) {
  static_cast<System*>(h)->kinetic_sweep(rho, f);
}
void ro_density_of(void* h, const double* f, double* rho) { static_cast<System*>(h)->density_of(f, rho); }
void ro_apply_term_kinetic(void* h, int k, const double* u, double* out) {
  static_cast<System*>(h)->apply_term_kinetic(k, u, out);
}
void ro_apply_kinetic(void* h, const double* u, double* out) {
  static_cast<System*>(h)->apply_kinetic(u, out);
}
void ro_kinetic_rhs(void* h, double* b) { static_cast<System*>(h)->kinetic_rhs(b); }

// ---- DSA assembly (dsa.cpp:154-258) ----------------------------------------
void* ro_dsa_create(void* h) {
  try {
    auto* s = static_cast<System*>(h);
    auto* d = new DsaHandle();
    d->d = build_dsa(*s);
    const long n = d->d.n;
    append(d->coupled, d->d.a_rr, 0, 0);
    if (d->d.nf == 2) {
      append(d->coupled, d->d.a_rj[0], 0, n);
      append(d->coupled, d->d.a_jr[0], n, 0);
      append(d->coupled, d->d.t_blocks[0], n, n);
    } else {
      append(d->coupled, d->d.a_rj[0], 0, n);
      append(d->coupled, d->d.a_rj[1], 0, 2 * n);
      append(d->coupled, d->d.a_jr[0], n, 0);
      append(d->coupled, d->d.t_blocks[0], n, n);
      append(d->coupled, d->d.a_jr[1], 2 * n, 0);
      append(d->coupled, d->d.t_blocks[1], 2 * n, 2 * n);
    }
    return d;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ro_dsa_destroy(void* d) { delete static_cast<DsaHandle*>(d); }
long ro_dsa_nnz(void* d) { return (long)static_cast<DsaHandle*>(d)->coupled.size(); }
int ro_dsa_fields(void* d) { return static_cast<DsaHandle*>(d)->d.nf; }
void ro_dsa_triplets(void* d, long* rows, long* cols, double* vals) {
  const auto& t = static_cast<DsaHandle*>(d)->coupled;
  for (size_t i = 0; i < t.size(); ++i) {
    rows[i] = t[i].r;
    cols[i] = t[i].c;
    vals[i] = t[i].v;
  }
}
// Individual blocks for apply_eliminated (dsa.cpp:279-293):
// which: 0 = A_rr, 1 = A_rJ[i], 2 = A_Jr[i], 3 = T[i].
long ro_dsa_block_nnz(void* d, int which, int i) {
  auto& D = static_cast<DsaHandle*>(d)->d;
  const SpMap& m = which == 0 ? D.a_rr : which == 1 ? D.a_rj[i] : which == 2 ? D.a_jr[i] : D.t_blocks[i];
  return (long)m.size();
}
void ro_dsa_block(void* d, int which, int i, long* rows, long* cols, double* vals) {
  auto& D = static_cast<DsaHandle*>(d)->d;
  const SpMap& m = which == 0 ? D.a_rr : which == 1 ? D.a_rj[i] : which == 2 ? D.a_jr[i] : D.t_blocks[i];
  long k = 0;
  for (const auto& e : m) {
    rows[k] = e.first.first;
    cols[k] = e.first.second;
    vals[k] = e.second;
    ++k;
  }
}

}  // extern "C"
