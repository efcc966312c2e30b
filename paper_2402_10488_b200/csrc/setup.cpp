// setup.cpp -- host-side discretization helpers of the C-ABI (problem
// setup): Gauss-Legendre nodes (quadrature.cpp:8-39), cell evaluation points,
// weighted per-cell mass blocks (transport_system.cpp:17-55) and the DG L2
// projection (dg_space.cpp:31-71).  They turn ProblemDefinition-style
// coefficient closures, evaluated by the caller at the returned points, into
// the per-cell blocks and load vectors rte_create consumes.
#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/rte_b200.h"

namespace {

void gl(int n, double* x, double* w) {
  const long double pi = 3.141592653589793238462643383279502884L;
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    long double z = std::cos(pi * (i + 0.75L) / (n + 0.5L)), d = 0.0L;
    for (int it = 0; it < 100; ++it) {
      long double a = 1.0L, b = z;
      for (int k = 2; k <= n; ++k) {
        const long double c = ((2.0L * k - 1.0L) * z * b - (k - 1.0L) * a) / k;
        a = b;
        b = c;
      }
      d = n * (z * b - a) / (z * z - 1.0L);
      const long double dz = b / d;
      z -= dz;
      if (std::fabs(dz) < 1e-19L) break;
    }
    const long double wt = 2.0L / ((1.0L - z * z) * d * d);
    x[i] = (double)(-z);
    x[n - 1 - i] = (double)z;
    w[i] = w[n - 1 - i] = (double)wt;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

struct Geo {
  int geom, nx, ny;
  const double* b;
  double x0, x1, y0, y1;
  int cells() const { return geom == RTE_SLAB1D ? nx : nx * ny; }
};

}  // namespace

extern "C" {

int rte_gauss_legendre_nodes(int n, double* x, double* w) {
  if (n < 1 || !x || !w) return RTE_ERR_INVALID;
  gl(n, x, w);
  return RTE_OK;
}

int rte_cell_points(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0, double y1,
                    int nq, double* px, double* py) {
  if (nq < 1 || nq > 32 || !px || !py) return RTE_ERR_INVALID;
  std::vector<double> g(nq), gw(nq);
  gl(nq, g.data(), gw.data());
  long k = 0;
  if (geometry == RTE_SLAB1D) {
    if (!bounds) return RTE_ERR_INVALID;
    for (int i = 0; i < nx; ++i) {
      const double h = bounds[i + 1] - bounds[i], xc = 0.5 * (bounds[i] + bounds[i + 1]);
      for (int q = 0; q < nq; ++q, ++k) {
        px[k] = xc + 0.5 * h * g[q];
        py[k] = 0.0;
      }
    }
    return RTE_OK;
  }
  const double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  const long nc = (long)nx * ny;
  // cells are independent: one thread per cell range, same per-cell arithmetic
#pragma omp parallel for schedule(static)
  for (long cell = 0; cell < nc; ++cell) {
    const int iy = (int)(cell / nx), ix = (int)(cell - (long)iy * nx);
    const double xc = x0 + ix * hx + 0.5 * hx, yc = y0 + iy * hy + 0.5 * hy;
    long kk = cell * nq * nq;
    for (int qy = 0; qy < nq; ++qy)
      for (int qx = 0; qx < nq; ++qx, ++kk) {
        px[kk] = xc + 0.5 * hx * g[qx];
        py[kk] = yc + 0.5 * hy * g[qy];
      }
  }
  (void)k;
  return RTE_OK;
}

// ws: point stride of the values (1: one value per point, 0: one constant)
static int weighted_mass_impl(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                              double y1, int nq, const double* wv, long ws, double* out) {
  if (nq < 1 || nq > 32 || !wv || !out) return RTE_ERR_INVALID;
  std::vector<double> g(nq), gw(nq);
  gl(nq, g.data(), gw.data());
  if (geometry == RTE_SLAB1D) {
    if (!bounds) return RTE_ERR_INVALID;
    for (int i = 0; i < nx; ++i) {
      const double h = bounds[i + 1] - bounds[i], xc = 0.5 * (bounds[i] + bounds[i + 1]);
      double m[4] = {0, 0, 0, 0};
      for (int q = 0; q < nq; ++q) {
        const double x = xc + 0.5 * h * g[q];
        const double ww = 0.5 * h * gw[q] * wv[((long)i * nq + q) * ws];
        const double p[2] = {1.0 / std::sqrt(h), std::sqrt(12.0 / (h * h * h)) * (x - xc)};
        for (int r = 0; r < 2; ++r)
          for (int c = 0; c < 2; ++c) m[2 * r + c] += (ww * p[r]) * p[c];
      }
      for (int e = 0; e < 4; ++e) out[4L * i + e] = m[e];
    }
    return RTE_OK;
  }
  const double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  const long ncells = (long)nx * ny;
#pragma omp parallel for schedule(static)
  for (long cell = 0; cell < ncells; ++cell) {
      const int iy = (int)(cell / nx), ix = (int)(cell - (long)iy * nx);
      const double xc = x0 + ix * hx + 0.5 * hx, yc = y0 + iy * hy + 0.5 * hy;
      double m[16] = {0};
      for (int qy = 0; qy < nq; ++qy) {
        const double y = yc + 0.5 * hy * g[qy];
        const double py0 = 1.0 / std::sqrt(hy), py1 = std::sqrt(12.0 / (hy * hy * hy)) * (y - yc);
        for (int qx = 0; qx < nq; ++qx) {
          const double x = xc + 0.5 * hx * g[qx];
          const double px0 = 1.0 / std::sqrt(hx), px1 = std::sqrt(12.0 / (hx * hx * hx)) * (x - xc);
          const double ww = 0.25 * hx * hy * gw[qx] * gw[qy] * wv[(cell * nq * nq + qy * nq + qx) * ws];
          const double p[4] = {px0 * py0, px1 * py0, px0 * py1, px1 * py1};
          for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) m[4 * r + c] += (ww * p[r]) * p[c];
        }
      }
      for (int e = 0; e < 16; ++e) out[16 * cell + e] = m[e];
    }
  return RTE_OK;
}

static int project_impl(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0, double y1,
                        int nq, const double* fv, long ws, double* out) {
  if (nq < 1 || nq > 32 || !fv || !out) return RTE_ERR_INVALID;
  std::vector<double> g(nq), gw(nq);
  gl(nq, g.data(), gw.data());
  auto p0 = [](double h) { return 1.0 / std::sqrt(h); };
  auto p1 = [](double h, double rel) { return std::sqrt(12.0 / (h * h * h)) * rel; };
  if (geometry == RTE_SLAB1D) {
    if (!bounds) return RTE_ERR_INVALID;
    for (int i = 0; i < nx; ++i) {
      const double h = bounds[i + 1] - bounds[i];
      double o0 = 0, o1 = 0;
      for (int q = 0; q < nq; ++q) {
        const double rel = 0.5 * h * g[q], wq = 0.5 * h * gw[q], f = fv[((long)i * nq + q) * ws];
        o0 += wq * f * p0(h);
        o1 += wq * f * p1(h, rel);
      }
      out[2L * i] = o0;
      out[2L * i + 1] = o1;
    }
    return RTE_OK;
  }
  const double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  const long nc = (long)nx * ny;
#pragma omp parallel for schedule(static)
  for (long c = 0; c < nc; ++c) {
    double o[4] = {0, 0, 0, 0};
    for (int qy = 0; qy < nq; ++qy) {
      const double ry = 0.5 * hy * g[qy];
      for (int qx = 0; qx < nq; ++qx) {
        const double rx = 0.5 * hx * g[qx];
        const double wq = 0.25 * hx * hy * gw[qx] * gw[qy], f = fv[(c * nq * nq + qy * nq + qx) * ws];
        const double bx0 = p0(hx), bx1 = p1(hx, rx), by0 = p0(hy), by1 = p1(hy, ry);
        o[0] += wq * f * bx0 * by0;
        o[1] += wq * f * bx1 * by0;
        o[2] += wq * f * bx0 * by1;
        o[3] += wq * f * bx1 * by1;
      }
    }
    for (int e = 0; e < 4; ++e) out[4 * c + e] = o[e];
  }
  return RTE_OK;
}

int rte_weighted_mass(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0, double y1,
                      int nq, const double* wv, double* out) {
  return weighted_mass_impl(geometry, nx, ny, bounds, x0, x1, y0, y1, nq, wv, 1, out);
}
int rte_weighted_mass_const(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                            double y1, int nq, double w, double* out) {
  return weighted_mass_impl(geometry, nx, ny, bounds, x0, x1, y0, y1, nq, &w, 0, out);
}
int rte_project(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0, double y1, int nq,
                const double* fv, double* out) {
  return project_impl(geometry, nx, ny, bounds, x0, x1, y0, y1, nq, fv, 1, out);
}
int rte_project_const(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0, double y1,
                      int nq, double f, double* out) {
  return project_impl(geometry, nx, ny, bounds, x0, x1, y0, y1, nq, &f, 0, out);
}

}  // extern "C"

// ---- per-parameter system assembly helpers (the host side of the
// TransportSystem constructor for a batch, transport_system.cpp:82-140) ----

// Per-cell blocks [n][nl*nl] -> scalars d0 when every block is d0 I to 1e-12
// relative (the closed-form XY cell solve needs sigma I blocks).
int rte_scalar_blocks(long n, int nl, const double* m, double* out) {
  if (n < 0 || nl < 1 || (n && (!m || !out))) return RTE_ERR_INVALID;
  const long nb = (long)nl * nl;
  int bad = 0;
  for (long c = 0; c < n; ++c) {
    const double* f = m + c * nb;
    const double d0 = f[0];
    double err = 0.0, scale = 1e-300;
    for (int i = 0; i < nl; ++i)
      for (int j = 0; j < nl; ++j) {
        err = std::max(err, std::fabs(f[i * nl + j] - (i == j ? d0 : 0.0)));
        if (i == j) scale = std::max(scale, std::fabs(f[i * nl + j]));
      }
    if (err > 1e-12 * scale) bad |= 1;
    out[c] = d0;
  }
  return bad ? RTE_ERR_UNSUPPORTED : RTE_OK;
}

// build_masses accumulation order (transport_system.cpp:133-138) for a batch:
// out[s][e] = sum_k psi[s][k] * terms[k][e], k ascending, each product rounded
// before the add (no contraction).
// products and sums rounded separately, as numpy does (setup.cpp is built with -ffp-contract=off)
int rte_combine_terms(int S, int K, long n, const double* psi, const double* terms, double* out) {
  if (S < 1 || K < 1 || n < 0 || !psi || !terms || !out) return RTE_ERR_INVALID;
  for (int s = 0; s < S; ++s) {
    double* o = out + (long)s * n;
    for (long e = 0; e < n; ++e) o[e] = 0.0;
    for (int k = 0; k < K; ++k) {
      const double p = psi[(long)s * K + k];
      const double* t = terms + (long)k * n;
      for (long e = 0; e < n; ++e) o[e] = o[e] + p * t[e];
    }
  }
  return RTE_OK;
}
