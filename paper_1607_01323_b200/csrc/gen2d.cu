// Host side of the general-geometry 2D operators (gen2d.cuh): the context
// holds the caller's device geometry / connectivity arrays (not owned) and
// the 1D tables; the C-ABI entry points are declared in include/dgmf.h.
#include <algorithm>
#include <string>
#include <vector>

#include "ctx.h"
#include "gen2d.cuh"
#include "tables.h"

using namespace dg;

struct dg_g2 {
  G2Geo geo;
  G2Tab tab;
};

namespace {

template <int N, int NQ>
int g2_launch_nq(dg_g2 *g, const G2Params &prm, const double *src, double *dst, cudaStream_t st) {
  using C = G2Cfg<N, NQ>;
  if (g->geo.ncells == 0) return DG_OK;
  const unsigned grid = (unsigned)((g->geo.ncells + C::CPB - 1) / C::CPB);
  g2_kernel<N, NQ><<<grid, C::THREADS, 0, st>>>(src, dst, g->geo, g->tab, prm);
  DG_LAUNCH_CHECK("g2_kernel");
  return DG_OK;
}

// (n, n_q) pairs: the linear rule n_q = n and the convective over-integration
// rule n_q = floor(3k/2) + 1 (basis.py:103-105)
int g2_launch(dg_g2 *g, const G2Params &prm, const double *src, double *dst, cudaStream_t st) {
  const int n = g->geo.n, nq = g->geo.nq;
#define DG_G(NN, QQ) \
  if (n == NN && nq == QQ) return g2_launch_nq<NN, QQ>(g, prm, src, dst, st);
  DG_G(2, 2) DG_G(3, 3) DG_G(4, 4) DG_G(5, 5) DG_G(6, 6) DG_G(7, 7) DG_G(8, 8)
  DG_G(3, 4) DG_G(4, 5) DG_G(5, 7) DG_G(6, 8) DG_G(7, 10) DG_G(8, 11)
#undef DG_G
  return inval("general 2D: unsupported (n, n_q) = (" + std::to_string(n) + ", " +
               std::to_string(nq) + ")");
}

}  // namespace

extern "C" {

int dg_g2_create(const dg_g2_desc *d, dg_g2 **out) {
  if (!d || !out) return inval("null argument");
  *out = nullptr;
  if (d->n < 2 || d->n > kG2MaxN) return inval("general 2D path: 1 <= k <= 7");
  if (d->nq < 1 || d->nq > kG2MaxQ) return inval("general 2D path: n_q <= 11");
  if (d->ncells < 0) return inval("negative cell count");
  if (!d->jxw || !d->jit || !d->fsj || !d->fnrm || !d->fjit || !d->nbr || !d->nslot ||
      !d->nflip || !d->tau || !d->S || !d->D || !d->ld || !d->rd)
    return inval("null geometry / table array");
  dg_g2 *g = new dg_g2();
  g->geo = G2Geo{d->n, d->nq, d->ncells, d->jxw, d->jit, d->fsj, d->fnrm, d->fjit,
                 d->nbr, d->nslot, d->nflip, d->tau};
  for (int i = 0; i < d->nq * d->n; ++i) {
    g->tab.S[i] = d->S[i];
    g->tab.D[i] = d->D[i];
  }
  for (int i = 0; i < d->n * d->n; ++i) g->tab.Si[i] = d->Si ? d->Si[i] : 0.0;
  for (int i = 0; i < d->n; ++i) {
    g->tab.ld[i] = d->ld[i];
    g->tab.rd[i] = d->rd[i];
  }
  *out = g;
  return DG_OK;
}

int dg_g2_destroy(dg_g2 *g) {
  delete g;
  return DG_OK;
}

int dg_g2_apply(dg_g2 *g, int op, double tau_scale, const int *kind, const double *src,
                double *dst, int ncomp, void *stream) {
  if (!g || !src || !dst) return inval("null argument");
  if (op < kG2Mass || op > kG2Laplace) return inval("general 2D: unknown operator");
  if (op == kG2Laplace && !kind) return inval("general 2D Laplace needs the boundary kinds");
  if (op == kG2InvMass && g->geo.nq != g->geo.n)
    return inval("inverse mass requires the n_q = k + 1 Gauss rule");
  if (op == kG2Laplace && ncomp != 1) return inval("the Laplacian acts on one scalar field");
  if (src == dst) return inval("general 2D: src and dst must not alias");
  G2Params prm{};
  prm.op = op;
  prm.tau_scale = tau_scale;
  prm.kind = kind;
  prm.local_node = -1;
  const int64_t per = g->geo.ncells * g->geo.n * g->geo.n;
  for (int c = 0; c < ncomp; ++c)  // one component at a time
    if (int rc = g2_launch(g, prm, src + c * per, dst + c * per, (cudaStream_t)stream)) return rc;
  return DG_OK;
}

int dg_g2_operator(dg_g2 *g, const dg_g2_params *p, const double *src, double *dst,
                   void *stream) {
  if (!g || !p || !dst) return inval("null argument");
  const int op = p->op;
  if (op < kG2Laplace || op > kG2PressureNeumann || op == kG2LaplaceLocal)
    return inval("general 2D: unknown operator");
  if (!p->kind) return inval("general 2D: boundary kinds required");
  G2Params prm{};
  prm.op = op;
  prm.tau_scale = p->tau_scale;
  prm.kind = p->kind;
  prm.local_node = -1;
  prm.gamma0_dt = p->gamma0_dt;
  prm.nu = p->nu;
  prm.tau_d = p->tau_d;
  prm.tau_c = p->tau_c;
  prm.scale = p->scale;
  prm.form = p->form;
  prm.fdata = p->fdata;
  if (op == kG2Convective || op == kG2PressureNeumann) {
    if (p->n_hist < 1 || p->n_hist > kG2MaxHist) return inval("need 1..4 history levels");
    prm.n_hist = p->n_hist;
    for (int j = 0; j < p->n_hist; ++j) {
      if (!p->hist[j]) return inval("null history level");
      if (op == kG2PressureNeumann && !p->vort[j]) return inval("null vorticity level");
      if (p->hist[j] == dst || p->vort[j] == dst)
        return inval("dst must not alias a history level");
      prm.hist[j] = p->hist[j];
      prm.beta[j] = p->beta[j];
      prm.gdata[j] = p->gdata[j];
      prm.vort[j] = p->vort[j];
    }
    prm.body = p->body;
  } else if (op != kG2GpDirichlet && op != kG2ViscousBc) {
    if (!src) return inval("null argument");
    if (src == dst) return inval("general 2D: src and dst must not alias");
  }
  if ((op == kG2Divergence && (p->form < 0 || p->form > 2)) ||
      (op == kG2Gradient && (p->form < 0 || p->form > 1)))
    return inval("unknown form");
  return g2_launch(g, prm, src, dst, (cudaStream_t)stream);
}

int dg_g2_laplace_diagonal(dg_g2 *g, double tau_scale, const int *kind, double *diag,
                           void *stream) {
  if (!g || !kind || !diag) return inval("null argument");
  const int np = g->geo.n * g->geo.n;
  for (int l = 0; l < np; ++l) {
    G2Params prm{};
    prm.op = kG2LaplaceLocal;
    prm.tau_scale = tau_scale;
    prm.kind = kind;
    prm.local_node = l;
    if (int rc = g2_launch(g, prm, nullptr, diag, (cudaStream_t)stream)) return rc;
  }
  return DG_OK;
}

int dg_g2_transfer(int k, int prolong, int64_t n_fine, const int64_t *parent, const int *quadrant,
                   int64_t n_coarse, const int64_t *children, const double *in, double *out,
                   int add, void *stream) {
  if (k < 1 || k + 1 > kG2MaxN) return inval("general 2D transfer: 1 <= k <= 7");
  if (!in || !out || (prolong && (!parent || !quadrant)) || (!prolong && !children))
    return inval("null argument");
  if (in == out) return inval("transfer: in and out must not alias");
  const int N = k + 1;
  G2Emb T;
  std::vector<double> nodes, V, Dv, pts(N);
  gll_nodes(k, nodes);
  for (int c = 0; c < 2; ++c) {
    for (int q = 0; q < N; ++q) pts[q] = 0.5 * (nodes[q] + (c ? 1.0 : -1.0));
    lagrange_tables(nodes, pts, V, Dv);
    for (int i = 0; i < N * N; ++i) T.E[c][i] = V[i];
  }
  const int64_t n = (prolong ? n_fine : n_coarse) * N * N;
  if (n == 0) return DG_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (prolong)
    g2_prolong_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(in, out, N, n_fine, parent,
                                                              quadrant, T, add);
  else
    g2_restrict_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(in, out, N, n_coarse, children, T);
  DG_LAUNCH_CHECK(prolong ? "g2_prolong_kernel" : "g2_restrict_kernel");
  return DG_OK;
}

}  // extern "C"

