// Host-side 1D tables in long double: Gauss rule, GLL nodes, Lagrange value
// and derivative tables.  Same definitions as the reference
// (quadrature.py:48-105, basis.py:15-84); long double Newton iterations give
// values within 1 ulp of the reference's double results.
#include <cmath>
#include <vector>

#include "tables.h"

namespace dg {

typedef long double ld;

static void legendre(int n, ld x, ld &p, ld &dp) {
  ld p0 = 1.0L, p1 = x;
  if (n == 0) {
    p = 1.0L;
    dp = 0.0L;
    return;
  }
  for (int j = 1; j < n; ++j) {
    ld p2 = ((2 * j + 1) * x * p1 - j * p0) / (j + 1);
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  if (std::fabs(std::fabs(x) - 1.0L) < 1e-300L)
    dp = (x > 0 ? 1.0L : ((n - 1) % 2 ? -1.0L : 1.0L)) * n * (n + 1) / 2.0L;
  else
    dp = n * (x * p1 - p0) / (x * x - 1.0L);
}

void gauss_rule(int n, std::vector<double> &pts, std::vector<double> &wts) {
  pts.assign(n, 0.0);
  wts.assign(n, 0.0);
  if (n == 1) {
    pts[0] = 0.0;
    wts[0] = 2.0;
    return;
  }
  const ld pi = 3.141592653589793238462643383279502884L;
  std::vector<ld> x(n);
  for (int i = 0; i < n; ++i) {
    x[i] = -std::cos(pi * (i + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 200; ++it) {
      ld p, dp;
      legendre(n, x[i], p, dp);
      ld dx = p / dp;
      x[i] -= dx;
      if (std::fabs(dx) < 1e-19L) break;
    }
  }
  for (int i = 0; i < n; ++i) {  // symmetrise
    ld s = 0.5L * (x[i] - x[n - 1 - i]);
    pts[i] = (double)s;
  }
  for (int i = 0; i < n; ++i) {
    ld xi = 0.5L * (x[i] - x[n - 1 - i]);
    ld p, dp;
    legendre(n, xi, p, dp);
    wts[i] = (double)(2.0L / ((1.0L - xi * xi) * dp * dp));
  }
}

void gll_nodes(int k, std::vector<double> &nodes) {
  nodes.assign(k + 1, 0.0);
  nodes[0] = -1.0;
  nodes[k] = 1.0;
  if (k == 1) return;
  const ld pi = 3.141592653589793238462643383279502884L;
  std::vector<ld> x(k - 1);
  for (int i = 0; i < k - 1; ++i) {
    x[i] = -std::cos(pi * (i + 1 + 0.26L) / k);
    for (int it = 0; it < 200; ++it) {
      ld p, dp;
      legendre(k, x[i], p, dp);
      ld ddp = (2 * x[i] * dp - k * (k + 1) * p) / (1.0L - x[i] * x[i]);
      ld dx = dp / ddp;
      x[i] -= dx;
      if (std::fabs(dx) < 1e-19L) break;
    }
  }
  for (int i = 0; i < k - 1; ++i) nodes[i + 1] = (double)(0.5L * (x[i] - x[k - 2 - i]));
}

// V[q][i] = l_i(x_q), Dv[q][i] = l_i'(x_q) (long double, exact at nodes)
void lagrange_tables(const std::vector<double> &nodes, const std::vector<double> &x,
                     std::vector<double> &V, std::vector<double> &Dv) {
  const int n = (int)nodes.size(), m = (int)x.size();
  V.assign((size_t)m * n, 0.0);
  Dv.assign((size_t)m * n, 0.0);
  std::vector<ld> bw(n);
  for (int i = 0; i < n; ++i) {
    ld p = 1.0L;
    for (int j = 0; j < n; ++j)
      if (j != i) p *= ((ld)nodes[i] - (ld)nodes[j]);
    bw[i] = 1.0L / p;
  }
  for (int q = 0; q < m; ++q) {
    const ld xq = x[q];
    // values: l_i(x) = prod_{j!=i} (x - x_j)/(x_i - x_j)
    // derivatives: l_i'(x) = sum_{j!=i} 1/(x_i-x_j) prod_{l!=i,j} (x-x_l)/(x_i-x_l)
    for (int i = 0; i < n; ++i) {
      ld val = 1.0L;
      for (int j = 0; j < n; ++j)
        if (j != i) val *= (xq - (ld)nodes[j]) / ((ld)nodes[i] - (ld)nodes[j]);
      ld der = 0.0L;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        ld t = 1.0L / ((ld)nodes[i] - (ld)nodes[j]);
        for (int l = 0; l < n; ++l)
          if (l != i && l != j) t *= (xq - (ld)nodes[l]) / ((ld)nodes[i] - (ld)nodes[l]);
        der += t;
      }
      V[(size_t)q * n + i] = (double)val;
      Dv[(size_t)q * n + i] = (double)der;
    }
  }
}

void basis_tables(int k, int nq, Basis1D &b) {
  b.k = k;
  b.n = k + 1;
  b.nq = nq;
  gll_nodes(k, b.nodes);
  gauss_rule(nq, b.pts, b.wts);
  lagrange_tables(b.nodes, b.pts, b.S, b.D);
  std::vector<double> e{-1.0, 1.0}, Ve, De;
  lagrange_tables(b.nodes, e, Ve, De);
  b.ld.assign(De.begin(), De.begin() + b.n);
  b.rd.assign(De.begin() + b.n, De.end());
  const int n = b.n;
  // M = S^T W S, K = D^T W D, integrals of l_i: wint = S^T w
  b.M.assign((size_t)n * n, 0.0);
  b.K.assign((size_t)n * n, 0.0);
  b.wint.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    ld wi = 0.0L;
    for (int q = 0; q < nq; ++q) wi += (ld)b.S[(size_t)q * n + i] * (ld)b.wts[q];
    b.wint[i] = (double)wi;
    for (int j = 0; j < n; ++j) {
      ld m = 0.0L, kk = 0.0L;
      for (int q = 0; q < nq; ++q) {
        m += (ld)b.S[(size_t)q * n + i] * (ld)b.wts[q] * (ld)b.S[(size_t)q * n + j];
        kk += (ld)b.D[(size_t)q * n + i] * (ld)b.wts[q] * (ld)b.D[(size_t)q * n + j];
      }
      b.M[(size_t)i * n + j] = (double)m;
      b.K[(size_t)i * n + j] = (double)kk;
    }
  }
  // inverse of the 1D mass matrix (Gauss-Jordan in long double)
  std::vector<ld> A((size_t)n * 2 * n, 0.0L);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      ld m = 0.0L;
      for (int q = 0; q < nq; ++q)
        m += (ld)b.S[(size_t)q * n + i] * (ld)b.wts[q] * (ld)b.S[(size_t)q * n + j];
      A[(size_t)i * 2 * n + j] = m;
    }
    A[(size_t)i * 2 * n + n + i] = 1.0L;
  }
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[(size_t)r * 2 * n + c]) > std::fabs(A[(size_t)piv * 2 * n + c])) piv = r;
    if (piv != c)
      for (int j = 0; j < 2 * n; ++j) std::swap(A[(size_t)c * 2 * n + j], A[(size_t)piv * 2 * n + j]);
    ld d = A[(size_t)c * 2 * n + c];
    for (int j = 0; j < 2 * n; ++j) A[(size_t)c * 2 * n + j] /= d;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      ld f = A[(size_t)r * 2 * n + c];
      if (f == 0.0L) continue;
      for (int j = 0; j < 2 * n; ++j) A[(size_t)r * 2 * n + j] -= f * A[(size_t)c * 2 * n + j];
    }
  }
  b.Minv.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) b.Minv[(size_t)i * n + j] = (double)A[(size_t)i * 2 * n + n + j];
}

}  // namespace dg
