// Instantiations of the convective term on the over-integration rule:
// (n, n_q) pairs floor(3k/2)+1 (reference, basis.py:103-105) and 3(k+1)/2
// (BASELINE literal).  See vecops_impl.cuh.
#include <algorithm>
#include <cstdint>
#include <string>

#include <cstdlib>

#include "vconv2.cuh"
#include "vecops_impl.cuh"

namespace dg {

template <int N, int NQ>
static CvEo<N, NQ> cv_eo(const QuadTab<N, NQ> &q) {
  double st[N * NQ], dt[N * NQ];
  for (int a = 0; a < NQ; ++a)
    for (int n = 0; n < N; ++n) {
      st[n * NQ + a] = q.S[a * N + n];
      dt[n * NQ + a] = q.D[a * N + n];
    }
  CvEo<N, NQ> t;
  t.S = eo_tab<NQ, N>(q.S);
  t.D = eo_tab<NQ, N>(q.D);
  t.St = eo_tab<N, NQ>(st);
  t.Dt = eo_tab<N, NQ>(dt);
  return t;
}

template <int N, int NQ, int TV = 0, int MB = 0>
static int launch_vconv(dg_ctx *c, double *dst, const VecParams &prm, cudaStream_t st) {
  using C = CvCfg<N, NQ, TV, MB>;
  auto kern = vconv_kernel<N, NQ, TV, MB>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr = true;
  }
  if (c->n_cells == 0) return DG_OK;
  const QuadTab<N, NQ> q = quad_tab<N, NQ>(c->over);
  kern<<<(unsigned)c->n_cells, C::T, C::SMEM, st>>>(dst, c->geo(), q, cv_eo<N, NQ>(q), prm,
                                                    c->n_cells);
  DG_LAUNCH_CHECK("vconv_kernel");
  return DG_OK;
}

// persistent pipelined kernel (vconv2.cuh): as many CTAs as fit on the GPU
template <int N, int NQ, int TV = 0, int MB = 0>
static int launch_vconv2(dg_ctx *c, double *dst, const VecParams &prm, cudaStream_t st) {
  using C = Cv2Cfg<N, NQ, TV, MB>;
  auto kern = vconv2_kernel<N, NQ, TV, MB>;
  static int grid_max = 0;
  if (!grid_max) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_sm = 0, dev = 0, sms = 0;
    DG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::T, C::SMEM));
    DG_CUDA_CHECK(cudaGetDevice(&dev));
    DG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid_max = std::max(1, per_sm) * sms;
  }
  if (c->n_cells == 0) return DG_OK;
  const QuadTab<N, NQ> q = quad_tab<N, NQ>(c->over);
  const unsigned grid = (unsigned)std::min<int64_t>(c->n_cells, grid_max);
  kern<<<grid, C::T, C::SMEM, st>>>(dst, c->geo(), q, cv_eo<N, NQ>(q), prm, c->n_cells);
  DG_LAUNCH_CHECK("vconv2_kernel");
  return DG_OK;
}

int vecop_over(dg_ctx *c, const double *src, double *dst, const VecParams &prm, cudaStream_t st) {
  static const bool generic = [] {
    const char *v = getenv("DG_VEC_GENERIC");
    return v && atoi(v) != 0;
  }();
  if (c->dim == 3 && !generic) {
    for (int j = 0; j < prm.n_hist; ++j)
      if (prm.hist[j] == dst) return inval("convective term: dst must not alias a history level");
    // DG_VCONV_CFG=1 (per call): the one-CTA-per-cell kernel (vconv.cuh), A/B
    const char *v = getenv("DG_VCONV_CFG");
    const bool old = v && atoi(v) == 1;
    bool aligned = prm.n_hist >= 1;
    for (int j = 0; j < prm.n_hist; ++j)
      aligned = aligned && (reinterpret_cast<uintptr_t>(prm.hist[j]) & 15) == 0;
    if (!old && aligned) {
      // (measured at Q5: 128 threads x 3 CTAs/SM best; 256 x 2: 0.866 ms,
      // 192 x 2: 0.848, 128 x 4 (spills): 0.830 vs 0.804 ms)
#define DG_V2(NN, QQ) \
  if (c->n == NN && c->nq_over == QQ) return launch_vconv2<NN, QQ>(c, dst, prm, st);
      // even N only: the cell and its TMA copies are whole 16 B units
      DG_V2(2, 2) DG_V2(2, 3) DG_V2(4, 5) DG_V2(4, 6) DG_V2(6, 8) DG_V2(6, 9)
#undef DG_V2
    }
#define DG_V(NN, QQ) \
  if (c->n == NN && c->nq_over == QQ) return launch_vconv<NN, QQ>(c, dst, prm, st);
    DG_V(2, 2) DG_V(2, 3) DG_V(3, 4) DG_V(4, 5) DG_V(4, 6) DG_V(5, 7) DG_V(6, 8) DG_V(6, 9)
#undef DG_V
  }
#define DG_O(D, NN, QQ) \
  if (c->n == NN && c->nq_over == QQ) return launch_vecop<D, NN, QQ, D, D>(c, src, dst, prm, c->over, st);
  if (c->dim == 3) {
    DG_O(3, 2, 2) DG_O(3, 2, 3) DG_O(3, 3, 4) DG_O(3, 4, 5) DG_O(3, 4, 6)
    DG_O(3, 5, 7) DG_O(3, 6, 8) DG_O(3, 6, 9)
  } else {
    DG_O(2, 2, 2) DG_O(2, 2, 3) DG_O(2, 3, 4) DG_O(2, 4, 5) DG_O(2, 4, 6)
    DG_O(2, 5, 7) DG_O(2, 6, 8) DG_O(2, 6, 9)
  }
#undef DG_O
  return inval("convective term: unsupported (k, n_q) = (" + std::to_string(c->k) + ", " +
               std::to_string(c->nq_over) + "); supported k <= 5 with n_q in "
               "{floor(3k/2)+1, 3(k+1)/2}");
}

}  // namespace dg
