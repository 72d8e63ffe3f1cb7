// Shared device-side definitions of the matrix-free DG library (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/dgmf.h"

namespace dg {

void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *where);

#define DG_CUDA_CHECK(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::dg::cuda_fail(_e, #expr); \
  } while (0)

#define DG_LAUNCH_CHECK(where)                                \
  do {                                                        \
    cudaError_t _e = cudaGetLastError();                      \
    if (_e != cudaSuccess) return ::dg::cuda_fail(_e, where); \
  } while (0)

constexpr int kMaxN = 8;  // k <= 7

// Edge handling of the owned block of cells, per side
// (xlo, xhi, ylo, yhi, zlo, zhi).
enum SideMode : int {
  kWrap = 0,         // periodic, neighbour is the local cell at the other end
  kGhost = 1,        // neighbour lives on another rank (x-slabs), ghost layer
  kBndNone = 2,      // velocity-Dirichlet: pressure-Neumann, no operator term
  kBndNeumann = 3,   // velocity-Neumann: pressure-Dirichlet term with 2 tau
};

// Cartesian geometry of the owned cells. All pointers are device pointers.
struct Geo {
  int nx, ny, nz;            // owned cells per axis (nz = 1 in 2D)
  const double *hx, *hy, *hz;  // cell sizes per axis index (owned)
  const double *hxi, *hyi, *hzi;  // their inverses (host-computed: no divisions in kernels)
  const double *tau;         // tau_e per owned cell (Eq. 18)
  int mode[6];
  const double *ghost[2];    // x-ghost layers (ny*nz cells each) or null
  const double *ghost_tau[2];
  double ghost_h[2];
  double ghost_hi[2];
  int exp_flags;             // timing experiments (DG_EXP env); 0 in production
  int bz0;                   // first brick z index of a chunked (z-range) launch, else 0
  const double *ctab;        // per-cell SIP face coefficients + scales (kCellTab each) or null
  const double *ax[3];
  int ghost_traces;          // ghost layers hold face traces [cell][z][y][v|g], not cells       // per-axis [h, 1/h, tau part, 0] at local index i (i = -1..n: neighbours)
};

// doubles per cell of the Laplace cell table (laplace6.cuh): 6 sides x (A /
// tau_scale, B, Dn), 3 s_d Kh scales, |cell|/8, one pad (odd stride)
constexpr int kCellTab = 23;

// 1D reference matrices on [-1,1] for n = k+1 GLL nodes, Gauss rule n_q = n:
// M = S^T W S, K = D^T W D, endpoint derivative rows.  Passed by value
// (kernel parameter space -> constant bank operands of DFMA).
template <int N, class R = double>
struct LapTab {  // R: the arithmetic type (double; float for the fp32 V-cycle)
  static constexpr int H = N / 2, NE = (N + 1) / 2;
  R M[N * N];
  R K[N * N];
  R dL[N];
  R dR[N];
  // even-odd (centro-symmetric) splits: A v = merge(Ae e, Ao o) with
  // e_j = v_j + v_{N-1-j}, o_j = v_j - v_{N-1-j} (e_H = v_H for odd N)
  R Me[NE * NE], Mo[H * H > 0 ? H * H : 1];
  R Ke[NE * NE], Ko[H * H > 0 ? H * H : 1];
  R dLe[NE], dLo[H > 0 ? H : 1];
};

// non-deduced context for scalar arguments of templated helpers
template <class X>
struct Ident {
  using type = X;
};

template <int N>
struct TensorTab {  // a single 1D matrix A (N x N) for tensor-product apply
  double A[N * N];
};

}  // namespace dg
