// search.cu -- wq_search: the whole search module of WindowQuant in ONE launch
// ("a single fused scorer -> assign kernel"): Eq.8 window scores
// (P:307-311), the rank order (Q7), Alg.1's bands / pin / vote / budget and Alg.2's
// stable partition for every layer.
//
// A cooperative persistent grid (128-thread CTAs, as many as are co-resident) runs four
// phases separated by grid-wide barriers:
//   1. pooled text rows tbar[b]                       (one task per request)
//   2. window scores scores[b][w]                     (one task per window)
//   3. the rank order of each request -- ONE bitonic sort per request (plus the batch-mean
//      order under the vote), where the 3-launch chain re-sorts in every (request, layer)
//      CTA of k_assign when a budget is set
//   4. the assignment of every (layer, request) from that order (assign_body)
// The same device code as the unfused kernels (scores.cuh, assign.cuh): identical scores,
// ranks, bits and permutations.
#include <cooperative_groups.h>

#include "assign.cuh"
#include "scores.cuh"

namespace cg = cooperative_groups;

namespace wq {

struct SearchArgs {
  const __half *vis;
  int64_t vrs, vbs;
  const __half *txt;
  int64_t trs, tbs;
  int B, M, N, D, S;
  double *tbar, *scores;
  int32_t *order;            // [B + 1][W]: rank order of each request (+ batch means)
  AssignParams p;
  uint8_t *bits;
  int32_t *rank, *perm, *seg;
};

template <int NC, bool CENTER>
__global__ void __launch_bounds__(ST, WQ_SC_MINB) k_search(SearchArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ double red[4 * WQ_SC_RB];
  __shared__ uint64_t warp_tot[32];
  __shared__ int s_rstar;
  cg::grid_group grid = cg::this_grid();
  const int W = a.M / a.S;
  // 1. pooled text rows
  for (int b = blockIdx.x; b < a.B; b += gridDim.x)
    text_pool_body<NC, CENTER>(a.txt, a.trs, a.tbs, a.N, a.D, a.tbar, b, reinterpret_cast<double *>(sm), red);
  grid.sync();
  // 2. window scores
  for (int t = blockIdx.x; t < a.B * W; t += gridDim.x)
    window_score_body<NC, CENTER>(a.vis, a.vrs, a.vbs, a.M, a.N, a.D, a.S, a.tbar, a.scores, a.D, 0, t % W, t / W,
                                  W, red);
  grid.sync();
  // 3. rank order: one sort per request, plus the batch-mean order under the vote (Q14)
  const int np = pow2_at_least(W);
  const int nsort = a.B + (a.p.vote && a.p.budget > 0.0 ? 1 : 0);
  for (int j = blockIdx.x; j < nsort; j += gridDim.x) {
    double *key = reinterpret_cast<double *>(sm);
    int *idx = reinterpret_cast<int *>(key + np);
    for (int i = threadIdx.x; i < np; i += ST) {
      double kv = -INFINITY;
      if (i < W) {
        if (j < a.B) {
          kv = a.scores[(int64_t)j * W + i];
        } else {
          double s = 0.0;
          for (int bb = 0; bb < a.B; bb++) s += a.scores[(int64_t)bb * W + i];
          kv = s / (double)a.B;
        }
      }
      key[i] = kv;
      idx[i] = i < W ? i : 0x7fffffff;
    }
    __syncthreads();
    bitonic(key, idx, np);
    for (int r = threadIdx.x; r < W; r += ST) {
      a.order[(int64_t)j * W + r] = idx[r];
      if (j < a.B && a.rank) a.rank[(int64_t)j * W + idx[r]] = r;
    }
    __syncthreads();
  }
  grid.sync();
  // 4. the assignment of every (layer, request) from the precomputed order
  const int nreq = a.p.vote ? 1 : a.B;
  for (int t = blockIdx.x; t < a.p.L * nreq; t += gridDim.x) {
    const int l = t / nreq, b = t - l * nreq;
    const int32_t *ord = a.order + (int64_t)(a.p.vote ? a.B : b) * W;
    assign_body<ST>(a.scores, a.p, a.bits, a.perm, a.seg, b, l, ord, sm, warp_tot, &s_rstar);
    __syncthreads();
  }
}

size_t search_smem(int W, int D) {
  int np = 1;
  while (np < W) np <<= 1;
  const size_t as = (size_t)np * (sizeof(double) + sizeof(int)) + (size_t)W * sizeof(int);
  const size_t tp = (size_t)D * sizeof(double);
  return as > tp ? as : tp;
}

template <int NC, bool CENTER>
static cudaError_t launch_search_t(const SearchArgs &a, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_search<NC, CENTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search<NC, CENTER>, ST, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  const int W = a.M / a.S;
  int grid = per_sm * device_sm_count();
  const int most = a.B * W > a.p.L * a.B ? a.B * W : a.p.L * a.B;
  if (grid > most) grid = most;
  SearchArgs args = a;
  void *params[] = {&args};
  return cudaLaunchCooperativeKernel((void *)k_search<NC, CENTER>, dim3(grid), dim3(ST), params, smem, st);
}

cudaError_t launch_search(const __half *vis, int64_t vrs, int64_t vbs, const __half *txt, int64_t trs, int64_t tbs,
                          int B, int M, int N, int D, int S, int metric, const AssignParams &p, double *tbar,
                          double *scores, int32_t *order, uint8_t *bits, int32_t *rank, int32_t *perm, int32_t *seg,
                          cudaStream_t st) {
  SearchArgs a{vis, vrs, vbs, txt, trs, tbs, B, M, N, D, S, tbar, scores, order, p, bits, rank, perm, seg};
  const size_t smem = search_smem(M / S, D);
  const int nc = (D / 8 + ST - 1) / ST;
#define WQ_SE(NCV)                                                                              \
  case NCV:                                                                                     \
    return metric == 1 ? launch_search_t<NCV, true>(a, smem, st) : launch_search_t<NCV, false>(a, smem, st);
  switch (nc) {
    WQ_SE(1) WQ_SE(2) WQ_SE(3) WQ_SE(4)
    default: return cudaErrorInvalidValue;
  }
#undef WQ_SE
}

}  // namespace wq
