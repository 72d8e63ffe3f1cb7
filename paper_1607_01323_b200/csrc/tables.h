#pragma once
#include <vector>

namespace dg {

struct Basis1D {
  int k = 0, n = 0, nq = 0;
  std::vector<double> nodes, pts, wts;  // GLL nodes; Gauss points/weights
  std::vector<double> S, D;             // (nq x n) row-major
  std::vector<double> ld, rd;           // endpoint derivative rows (n)
  std::vector<double> M, K, Minv;       // (n x n) 1D reference mass/stiffness
  std::vector<double> wint;             // integrals of l_i on [-1,1]
};

void gauss_rule(int n, std::vector<double> &pts, std::vector<double> &wts);
void gll_nodes(int k, std::vector<double> &nodes);
void basis_tables(int k, int nq, Basis1D &b);
// V[q][i] = l_i(x_q), Dv[q][i] = l_i'(x_q) for the Lagrange basis on nodes
void lagrange_tables(const std::vector<double> &nodes, const std::vector<double> &x,
                     std::vector<double> &V, std::vector<double> &Dv);

}  // namespace dg
