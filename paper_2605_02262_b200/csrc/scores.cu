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
// A warp per text row (8 warps, rows j = warp, warp + 8, ...): lane l owns channels
// l + 32 i of the row; the row's norm is a warp-shuffle tree; the 8 warps' pooled
// vectors are summed in fixed order at the end (sh: [8][D] doubles).
constexpr int TPQ = 256;
template <int NCH>                               // 8-channel chunks per lane: ceil(D / 256)
__global__ void __launch_bounds__(TPQ) k_text_pool_q(const __half *__restrict__ qt, int64_t qsb, int64_t qsh,
                                                     int64_t qsj, int N, int H, int grp, int d,
                                                     double *__restrict__ tbar) {
  extern __shared__ double sh[];                 // [8][D] per-warp pooled vectors
  const int b = blockIdx.x, D = H * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *mine = sh + (size_t)warp * D;
  for (int c = lane; c < D; c += 32) mine[c] = 0.0;
  __syncwarp();
  const double ginv = 1.0 / (double)grp;
  for (int j = warp; j < N; j += TPQ / 32) {
    double x[NCH][8];
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < NCH; i++) {
      const int c0 = 8 * (lane + 32 * i);
#pragma unroll
      for (int e = 0; e < 8; e++) x[i][e] = 0.0;
      if (c0 < D) {
        const int h = c0 / d, cc = c0 - h * d;
        const __half *row = qt + b * qsb + (int64_t)h * grp * qsh + (int64_t)j * qsj + cc;
        // the group's query rows: independent 16-byte loads, summed in fp64 in head order
        uint4 u[8];
#pragma unroll
        for (int gq = 0; gq < 8; gq++)
          if (gq < grp) u[gq] = __ldg(reinterpret_cast<const uint4 *>(row + gq * qsh));
#pragma unroll
        for (int gq = 0; gq < 8; gq++) {
          if (gq >= grp) break;
          const __half2 *hh = reinterpret_cast<const __half2 *>(&u[gq]);
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const float2 f = __half22float2(hh[e]);
            x[i][2 * e] += (double)f.x;
            x[i][2 * e + 1] += (double)f.y;
          }
        }
#pragma unroll
        for (int e = 0; e < 8; e++) {
          x[i][e] *= ginv;
          ss = fma(x[i][e], x[i][e], ss);
        }
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double inv = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
#pragma unroll
    for (int i = 0; i < NCH; i++) {
      const int c0 = 8 * (lane + 32 * i);
      if (c0 < D)
#pragma unroll
        for (int e = 0; e < 8; e++) mine[c0 + e] = fma(x[i][e], inv, mine[c0 + e]);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += TPQ) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < TPQ / 32; w++) v += sh[(size_t)w * D + c];
    tbar[(int64_t)b * D + c] = v;
  }
}

// Per-layer scorer visual side for short head-split rows (D = H d <= 1024): one CTA of
// 4 warps per (window, request), a WARP per token row -- lane l owns the 16-byte chunks
// l + 32 i (i < NCW) of every row, the row's sum of squares is a warp-shuffle tree (no
// block barrier per row), RB rows per warp in flight; the 4 warps' pooled vectors are
// summed in fixed order through shared memory and dotted with tbar.  Same arithmetic as
// window_score_body (fp64, zero-norm rows contribute 0), another fixed summation order.
template <int NCW>
__global__ void __launch_bounds__(ST) k_window_scores_rows(const __half *__restrict__ vis, int64_t vrs,
                                                           int64_t vbs, int N, int D, int S,
                                                           const double *__restrict__ tbar,
                                                           double *__restrict__ scores, int dh, int64_t hs) {
  constexpr int RB = 4;
  extern __shared__ double wpool[];              // [4][D]
  __shared__ double red[4];
  const int w = blockIdx.x, b = blockIdx.y, W = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunk = D / 8;
  int coff[NCW];
#pragma unroll
  for (int i = 0; i < NCW; i++) {
    const int c = 8 * (lane + 32 * i);
    coff[i] = (int)((int64_t)(c / dh) * hs + c % dh);
  }
  double pool[NCW][8];
#pragma unroll
  for (int i = 0; i < NCW; i++)
#pragma unroll
    for (int e = 0; e < 8; e++) pool[i][e] = 0.0;
  const __half *base = vis + b * vbs + (int64_t)w * S * vrs;
  for (int r0 = warp * RB; r0 < S; r0 += 4 * RB) {
    uint4 raw[RB][NCW];
#pragma unroll
    for (int r = 0; r < RB; r++)
#pragma unroll
      for (int i = 0; i < NCW; i++)
        raw[r][i] = (r0 + r < S && lane + 32 * i < nchunk)
                        ? __ldcs(reinterpret_cast<const uint4 *>(base + (int64_t)(r0 + r) * vrs + coff[i]))
                        : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < RB; r++) {
      double ss = 0.0;
#pragma unroll
      for (int i = 0; i < NCW; i++) {
        const __half2 *h = reinterpret_cast<const __half2 *>(&raw[r][i]);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const float2 f = __half22float2(h[e]);
          ss = fma((double)f.x, (double)f.x, ss);
          ss = fma((double)f.y, (double)f.y, ss);
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const double inv = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
#pragma unroll
      for (int i = 0; i < NCW; i++) {
        const __half2 *h = reinterpret_cast<const __half2 *>(&raw[r][i]);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const float2 f = __half22float2(h[e]);
          pool[i][2 * e] = fma((double)f.x, inv, pool[i][2 * e]);
          pool[i][2 * e + 1] = fma((double)f.y, inv, pool[i][2 * e + 1]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NCW; i++) {
    const int k = lane + 32 * i;
    if (k < nchunk)
#pragma unroll
      for (int e = 0; e < 8; e++) wpool[warp * D + 8 * k + e] = pool[i][e];
  }
  __syncthreads();
  double dot[1] = {0.0};
  const double *tb = tbar + (int64_t)b * D;
  for (int c = threadIdx.x; c < D; c += ST) {
    const double v = ((wpool[c] + wpool[D + c]) + wpool[2 * D + c]) + wpool[3 * D + c];
    dot[0] = fma(v, tb[c], dot[0]);
  }
  block_sum<1>(dot, red);
  if (threadIdx.x == 0) scores[(int64_t)b * W + w] = dot[0] / ((double)S * (double)N);
}

cudaError_t launch_text_pool_q(const __half *qt, int64_t qsb, int64_t qsh, int64_t qsj, int B, int N, int H,
                               int grp, int d, double *tbar, cudaStream_t st) {
  const size_t smem = (size_t)(TPQ / 32) * H * d * sizeof(double);
  if (grp > 8 || (d % 8) || (qsb % 8) || (qsh % 8) || (qsj % 8) || (reinterpret_cast<uintptr_t>(qt) & 15))
    return cudaErrorInvalidValue;                // (16-byte loads: the ABI checks these first)
  const int nch = (H * d / 8 + 31) / 32;
  auto kern = nch <= 1 ? k_text_pool_q<1> : nch <= 2 ? k_text_pool_q<2> : k_text_pool_q<4>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<B, TPQ, smem, st>>>(qt, qsb, qsh, qsj, N, H, grp, d, tbar);
  return cudaGetLastError();
}

cudaError_t launch_text_pool(const __half *txt, int64_t trs, int64_t tbs, int B, int N, int D,
                             double *tbar, int metric, cudaStream_t st) {
  size_t smem = (size_t)D * sizeof(double);
  const int nc = (D / 8 + ST - 1) / ST;
  auto kern = metric == 1 ? (nc <= 1 ? k_text_pool<1, true> : nc <= 2 ? k_text_pool<2, true>
                             : nc <= 3 ? k_text_pool<3, true> : k_text_pool<4, true>)
                          : (nc <= 1 ? k_text_pool<1, false> : nc <= 2 ? k_text_pool<2, false>
                             : nc <= 3 ? k_text_pool<3, false> : k_text_pool<4, false>);
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
  if ((int64_t)(D / dh - 1) * hs + dh >= (1LL << 31)) return cudaErrorInvalidValue;
  const bool split = dh != D;
  if (split && metric == 0 && D <= 1024 && D % 8 == 0) {
    // short head-split rows (the per-layer scorer): warp per row
    const size_t smem = (size_t)4 * D * sizeof(double);
    const int ncw = (D / 8 + 31) / 32;
    auto kern = ncw <= 1 ? k_window_scores_rows<1> : ncw <= 2 ? k_window_scores_rows<2>
                         : k_window_scores_rows<4>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, ST, smem, st>>>(vis, vrs, vbs, N, D, S, tbar, scores, dh, hs);
    return cudaGetLastError();
  }
#define WQ_WS(NCV)                                                                                      \
  case NCV:                                                                                             \
    if (split)                                                                                          \
      (metric == 1 ? k_window_scores<NCV, true, true> : k_window_scores<NCV, false, true>)              \
          <<<grid, ST, 0, st>>>(vis, vrs, vbs, M, N, D, S, tbar, scores, dh, hs);                       \
    else                                                                                                \
      (metric == 1 ? k_window_scores<NCV, true, false> : k_window_scores<NCV, false, false>)            \
          <<<grid, ST, 0, st>>>(vis, vrs, vbs, M, N, D, S, tbar, scores, dh, hs);                       \
    break;
  switch (nc) {
    WQ_WS(1) WQ_WS(2) WQ_WS(3) WQ_WS(4)
    default: return cudaErrorInvalidValue;
  }
#undef WQ_WS
  return cudaGetLastError();
}

}  // namespace wq
