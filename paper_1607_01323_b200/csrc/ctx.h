// The library context (opaque dg_ctx of include/dgmf.h), shared by the
// translation units of libdgmf (dgmf.cu: Laplacian, mass, solvers, halos;
// vecops.cu: quadrature-point operators and right-hand sides).
#pragma once
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "tables.h"

namespace dg {
int inval(const std::string &m);  // sets the error text, returns DG_EINVAL
}  // namespace dg

struct dg_ctx {
  int dim = 3, k = 1, n = 2, nq_over = 2;
  int gcounts[3] = {1, 1, 1};
  int counts[3] = {1, 1, 1};
  int slab_begin = 0, slab_end = 0;
  int periodic[3] = {0, 0, 0};
  int bc[6] = {0, 0, 0, 0, 0, 0};
  int mode[6] = {0, 0, 0, 0, 0, 0};
  dg::Basis1D basis, over;
  std::vector<double> gvert[3];
  std::vector<double> hx, hy, hz, tau;  // host, owned
  double ghost_h[2] = {1.0, 1.0};
  std::vector<double> ghost_tau_h[2];
  double *d_hx = nullptr, *d_hy = nullptr, *d_hz = nullptr, *d_tau = nullptr;
  double *d_hinv = nullptr;  // [1/hx | 1/hy | 1/hz]
  double *d_axis = nullptr;  // per-axis [h, 1/h, tau part, 0] incl. one neighbour per side
  int64_t axis_off[3] = {0, 0, 0};
  double *d_ghost_tau[2] = {nullptr, nullptr};
  const double *d_recv[2] = {nullptr, nullptr};  // caller-owned ghost layers
  int64_t halo_count = 0;
  int64_t n_cells = 0, n_dofs = 0, np = 0;
  double volume = 0.0;  // |Omega| of the GLOBAL mesh
  double *d_red = nullptr;     // reduction partials (kRedBlocks) + scalars
  double *d_red3 = nullptr;    // 3 x kRedBlocks partials (sharded CG dots)
  double *d_hcell = nullptr;   // per-cell dual-weight factor hx hy hz / 8 (3D)
  unsigned *d_counter = nullptr;  // work counter of the persistent warp-column kernel
  int halo_traces = 0;         // ghost layers carry face traces (column kernel)
  double *d_zero_ghost = nullptr;  // zero ghost layer (dg_laplace_vmult_split phase 1)
  double *d_scal = nullptr;    // 16 device scalars
  double *h_scal = nullptr;    // pinned mirror
  std::vector<double *> work;  // solver work vectors (n_dofs each)
  double *d_partials = nullptr;  // per-brick partial sums of the fused vmult epilogue
  int64_t partials_n = 0;
  int64_t epi_nparts = 0;  // partial-sum slots written by the last fused-dot vmult
  double *d_hin = nullptr, *d_hout = nullptr;   // device staging of dg_laplace_vmult_host
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  double *d_ctab = nullptr;  // Laplace cell table (laplace6.cuh), built on first use
  double *d_trc = nullptr;  // face traces of the Cartesian vector operators (vcart.cu)
  int64_t trc_n = 0;
  std::vector<double *> vwork;  // vector-PCG work vectors (vwork_n doubles each)
  int64_t vwork_n = 0;
  double *d_vpart = nullptr;    // per-CTA partial sums of the vector-PCG update
  int64_t vpart_n = 0;
  double *d_apdot = nullptr;    // per-CTA p.Ap partials of the vector-PCG operator
  int64_t apdot_n = 0;
  std::mutex mu;

  dg::Geo geo() const {
    dg::Geo g;
    g.nx = counts[0];
    g.ny = counts[1];
    g.nz = counts[2];
    g.hx = d_hx;
    g.hy = d_hy;
    g.hz = d_hz;
    g.tau = d_tau;
    g.hxi = d_hinv;
    g.hyi = d_hinv ? d_hinv + counts[0] : nullptr;
    g.hzi = d_hinv ? d_hinv + counts[0] + counts[1] : nullptr;
    for (int i = 0; i < 6; ++i) g.mode[i] = mode[i];
    for (int s = 0; s < 2; ++s) {
      g.ghost[s] = d_recv[s];
      g.ghost_tau[s] = d_ghost_tau[s];
      g.ghost_h[s] = ghost_h[s];
      g.ghost_hi[s] = 1.0 / ghost_h[s];
    }
    static const int exp_flags = [] {
      const char *v = getenv("DG_EXP");
      return v ? atoi(v) : 0;
    }();
    g.exp_flags = exp_flags;
    g.bz0 = 0;
    g.ghost_traces = halo_traces;
    g.ctab = d_ctab;
    for (int d = 0; d < 3; ++d) g.ax[d] = d_axis ? d_axis + axis_off[d] : nullptr;
    return g;
  }
};
