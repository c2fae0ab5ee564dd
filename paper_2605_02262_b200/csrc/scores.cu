// scores.cu -- wq_window_scores: Eq.8, Alg.1 lines 9-12.
//
// sim(T, W_w) = 1/(S N) sum_j sum_k cos(t_j, v_k) is evaluated through the exact
// identity sum_j sum_k t^_j . v^_k = (sum_k v^_k) . (sum_j t^_j), x^ = x/||x||
// (reading Q3): one pass over the visual tokens (HBM-bound), fp64 accumulation
// (Q6), fixed reduction trees (bit-reproducible), zero-norm rows contribute 0 (Q5).
//   k_text_pool:     tbar[b][c] = sum_j t_j[c] / ||t_j||           (tiny)
//   k_window_scores: one CTA per (window, request): row norms in chunks of 4 rows,
//                    pooled window vector in shared memory, dot with tbar.
#include "scores.cuh"

namespace wq {

// Per-layer scorer text side (reading Q36): text row j of request b is the concatenation
// over kv heads h of the mean of its GQA group's queries, (1/g) sum_{g'} Q[b][h g + g'][j][:]
// (D = H d, fp64); tbar[b][:] = sum_j row_j / ||row_j|| (a zero row contributes 0).
__global__ void __launch_bounds__(ST) k_text_pool_q(const __half *__restrict__ qt, int64_t qsb, int64_t qsh,
                                                    int64_t qsj, int N, int H, int grp, int d,
                                                    double *__restrict__ tbar) {
  extern __shared__ double sh[];                 // pooled [D], row [D]
  __shared__ double red[4];
  const int b = blockIdx.x, D = H * d;
  double *pooled = sh, *row = sh + D;
  for (int c = threadIdx.x; c < D; c += ST) pooled[c] = 0.0;
  for (int j = 0; j < N; j++) {
    double ss[1] = {0.0};
    for (int c = threadIdx.x; c < D; c += ST) {
      const int h = c / d, cc = c - h * d;
      double acc = 0.0;
      for (int gq = 0; gq < grp; gq++)
        acc += (double)__half2float(qt[b * qsb + (int64_t)(h * grp + gq) * qsh + (int64_t)j * qsj + cc]);
      const double x = acc / (double)grp;
      row[c] = x;
      ss[0] = fma(x, x, ss[0]);
    }
    block_sum<1>(ss, red);
    const double inv = ss[0] > 0.0 ? 1.0 / sqrt(ss[0]) : 0.0;
    for (int c = threadIdx.x; c < D; c += ST) pooled[c] = fma(row[c], inv, pooled[c]);
    __syncthreads();
  }
  for (int c = threadIdx.x; c < D; c += ST) tbar[(int64_t)b * D + c] = pooled[c];
}

cudaError_t launch_text_pool_q(const __half *qt, int64_t qsb, int64_t qsh, int64_t qsj, int B, int N, int H,
                               int grp, int d, double *tbar, cudaStream_t st) {
  const size_t smem = (size_t)2 * H * d * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_text_pool_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_text_pool_q<<<B, ST, smem, st>>>(qt, qsb, qsh, qsj, N, H, grp, d, tbar);
  return cudaGetLastError();
}

cudaError_t launch_text_pool(const __half *txt, int64_t trs, int64_t tbs, int B, int N, int D,
                             double *tbar, int metric, cudaStream_t st) {
  size_t smem = (size_t)D * sizeof(double);
  auto kern = metric == 1 ? k_text_pool<true> : k_text_pool<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<B, ST, smem, st>>>(txt, trs, tbs, N, D, tbar);
  return cudaGetLastError();
}

cudaError_t launch_window_scores(const __half *vis, int64_t vrs, int64_t vbs, int B, int M, int N,
                                 int D, int S, const double *tbar, double *scores, int metric, cudaStream_t st,
                                 int dh, int64_t hs) {
  int W = M / S;
  int nc = (D / 8 + ST - 1) / ST;
  dim3 grid(W, B);
  if (dh <= 0) { dh = D; hs = 0; }
#define WQ_WS(NCV)                                                                                   \
  case NCV:                                                                                          \
    if (metric == 1) k_window_scores<NCV, true><<<grid, ST, 0, st>>>(vis, vrs, vbs, M, N, D, S, tbar, scores, dh, hs); \
    else k_window_scores<NCV, false><<<grid, ST, 0, st>>>(vis, vrs, vbs, M, N, D, S, tbar, scores, dh, hs);          \
    break;
  switch (nc) {
    WQ_WS(1) WQ_WS(2) WQ_WS(3) WQ_WS(4)
    default: return cudaErrorInvalidValue;
  }
#undef WQ_WS
  return cudaGetLastError();
}

}  // namespace wq
