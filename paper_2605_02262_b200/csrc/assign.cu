// assign.cu -- wq_assign_bits (Alg.1 lines 8-16, P:313 bands, P:322 pin, P:395 vote,
// reading Q13 budget; Alg.2 P:420-444 stable partition -> perm, seg_off).
//
//   k_rank:   one CTA per request: bitonic sort of (score, index) in shared memory,
//             rank[b][w] = position in (-score, w) order (Q7).
//   k_assign: one CTA per (request, layer) (per layer under the batch vote):
//             band -> pin -> vote -> budget -> stable partition.
// The budget rule "demote the lowest-ranked eligible window one width step while
// over budget" is evaluated in closed form: windows are demoted completely in
// ascending-score order, so a suffix scan over the rank order finds the window
// at which the budget is met, and that one window is stepped down one width at a
// time.  All decisions are taken on the same fp64 scores and integer sums as the
// definition; everything is integer/comparison work (latency-bound, tiny).
#include "assign.cuh"

namespace wq {

__global__ void __launch_bounds__(AT) k_rank(const double *__restrict__ scores, int W,
                                             int32_t *__restrict__ rank) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int np = pow2_at_least(W);
  double *key = reinterpret_cast<double *>(sm);
  int *idx = reinterpret_cast<int *>(key + np);
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < np; i += AT) {
    key[i] = i < W ? scores[(int64_t)b * W + i] : -INFINITY;
    idx[i] = i < W ? i : 0x7fffffff;
  }
  __syncthreads();
  bitonic(key, idx, np);
  for (int r = threadIdx.x; r < W; r += AT) rank[(int64_t)b * W + idx[r]] = r;
}

__global__ void __launch_bounds__(AT) k_assign(const double *__restrict__ scores, AssignParams p,
                                               uint8_t *__restrict__ bits_out,
                                               int32_t *__restrict__ perm_out,
                                               int32_t *__restrict__ seg_out) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t warp_tot[32];
  __shared__ int s_rstar;
  assign_body<AT>(scores, p, bits_out, perm_out, seg_out, blockIdx.x, blockIdx.y, nullptr, sm, warp_tot, &s_rstar);
}

static size_t assign_smem(int W) {
  int np = 1;
  while (np < W) np <<= 1;
  return (size_t)np * (sizeof(double) + sizeof(int)) + (size_t)W * sizeof(int);
}

cudaError_t launch_rank(const double *scores, int B, int W, int32_t *rank, cudaStream_t st) {
  size_t smem = assign_smem(W);
  cudaError_t e = cudaFuncSetAttribute(k_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_rank<<<B, AT, smem, st>>>(scores, W, rank);
  return cudaGetLastError();
}

cudaError_t launch_assign(const double *scores, const AssignParams &p, uint8_t *bits, int32_t *perm,
                          int32_t *seg_off, cudaStream_t st) {
  size_t smem = assign_smem(p.W);
  cudaError_t e = cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(p.vote ? 1 : p.B, p.L);
  k_assign<<<grid, AT, smem, st>>>(scores, p, bits, perm, seg_off);
  return cudaGetLastError();
}

}  // namespace wq
