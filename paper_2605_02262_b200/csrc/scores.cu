// scores.cu -- wq_window_scores: Eq.8, Alg.1 lines 9-12.
//
// sim(T, W_w) = 1/(S N) sum_j sum_k cos(t_j, v_k) is evaluated through the exact
// identity sum_j sum_k t^_j . v^_k = (sum_k v^_k) . (sum_j t^_j), x^ = x/||x||
// (reading Q3): one pass over the visual tokens (HBM-bound), fp64 accumulation
// (Q6), fixed reduction trees (bit-reproducible), zero-norm rows contribute 0 (Q5).
//   k_text_pool:     tbar[b][c] = sum_j t_j[c] / ||t_j||           (tiny)
//   k_window_scores: one CTA per (window, request): row norms in chunks of 4 rows,
//                    pooled window vector in shared memory, dot with tbar.
#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {

constexpr int ST = 128;  // threads per CTA
#ifndef WQ_SC_RB
#define WQ_SC_RB 2        // visual rows per block reduction (2 with 3 CTAs/SM: C5 702 -> 560 us)
#endif
#ifndef WQ_SC_MINB
#define WQ_SC_MINB 3      // CTAs per SM the register budget must allow
#endif

// Deterministic block sum of NV doubles per thread (fixed tree).
template <int NV>
WQ_DEV void block_sum(double (&v)[NV], double *red /* [4][NV] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; i++)
    for (int o = 16; o >= 1; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; i++) red[warp * NV + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; i++) v[i] = ((red[i] + red[NV + i]) + red[2 * NV + i]) + red[3 * NV + i];
  __syncthreads();
}

WQ_DEV void load8(const __half *p, double (&x)[8]) {
  uint4 u = *reinterpret_cast<const uint4 *>(p);
  const __half2 *h = reinterpret_cast<const __half2 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) {
    float2 f = __half22float2(h[i]);
    x[2 * i] = (double)f.x;
    x[2 * i + 1] = (double)f.y;
  }
}

template <bool CENTER>
__global__ void __launch_bounds__(ST) k_text_pool(const __half *__restrict__ txt, int64_t trs,
                                                  int64_t tbs, int N, int D, double *__restrict__ tbar) {
  extern __shared__ double pooled[];  // [D]
  __shared__ double red[4];
  const int b = blockIdx.x, nchunk = D / 8;
  for (int c = threadIdx.x; c < D; c += ST) pooled[c] = 0.0;
  for (int j = 0; j < N; j++) {
    const __half *row = txt + b * tbs + (int64_t)j * trs;
    double mu = 0.0;
    if (CENTER) {                                  // Pearson: centre the row first (T11)
      double sm[1] = {0.0};
      for (int k = threadIdx.x; k < nchunk; k += ST) {
        double x[8];
        load8(row + 8 * k, x);
#pragma unroll
        for (int i = 0; i < 8; i++) sm[0] += x[i];
      }
      block_sum<1>(sm, red);
      mu = sm[0] / (double)D;
    }
    double ss[1] = {0.0};
    for (int k = threadIdx.x; k < nchunk; k += ST) {
      double x[8];
      load8(row + 8 * k, x);
#pragma unroll
      for (int i = 0; i < 8; i++) ss[0] = fma(x[i] - mu, x[i] - mu, ss[0]);
    }
    block_sum<1>(ss, red);
    double inv = ss[0] > 0.0 ? 1.0 / sqrt(ss[0]) : 0.0;
    for (int k = threadIdx.x; k < nchunk; k += ST) {
      double x[8];
      load8(row + 8 * k, x);
#pragma unroll
      for (int i = 0; i < 8; i++) pooled[8 * k + i] = fma(x[i] - mu, inv, pooled[8 * k + i]);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += ST) tbar[(int64_t)b * D + c] = pooled[c];
}

// A visual "row" is D elements; with head-split rows (the per-layer scorer) element c lives
// at row + (c / dh) * hs + c % dh (dh = head dim, hs = head stride); dh = D, hs = 0 otherwise.
template <int NC, bool CENTER>  // 16-byte chunks per thread per row: ceil(D / 8 / ST); CENTER: Pearson
__global__ void __launch_bounds__(ST, WQ_SC_MINB) k_window_scores(const __half *__restrict__ vis, int64_t vrs,
                                                      int64_t vbs, int M, int N, int D, int S,
                                                      const double *__restrict__ tbar,
                                                      double *__restrict__ scores, int dh, int64_t hs) {
  constexpr int RB = WQ_SC_RB;  // rows per batch
  __shared__ double red[4 * RB];
  const int w = blockIdx.x, b = blockIdx.y, W = gridDim.x, tid = threadIdx.x;
  const int nchunk = D / 8;
  double pool[NC][8];
#pragma unroll
  for (int i = 0; i < NC; i++)
#pragma unroll
    for (int e = 0; e < 8; e++) pool[i][e] = 0.0;
  const __half *base = vis + b * vbs + (int64_t)w * S * vrs;
  for (int r0 = 0; r0 < S; r0 += RB) {
    uint4 raw[RB][NC];
#pragma unroll
    for (int r = 0; r < RB; r++)
#pragma unroll
      for (int i = 0; i < NC; i++) {
        int k = tid + ST * i;
        const int c = 8 * k;                                // first element of the chunk
        raw[r][i] = k < nchunk ? __ldcs(reinterpret_cast<const uint4 *>(base + (int64_t)(r0 + r) * vrs +
                                                                      (int64_t)(c / dh) * hs + c % dh))
                               : make_uint4(0, 0, 0, 0);
      }
    double mu[RB];
#pragma unroll
    for (int r = 0; r < RB; r++) mu[r] = 0.0;
    if constexpr (CENTER) {                        // Pearson: row means first (T11)
#pragma unroll
      for (int r = 0; r < RB; r++) {
#pragma unroll
        for (int i = 0; i < NC; i++) {
          const __half2 *h = reinterpret_cast<const __half2 *>(&raw[r][i]);
#pragma unroll
          for (int e = 0; e < 4; e++) {
            float2 f = __half22float2(h[e]);
            mu[r] += (double)f.x;
            mu[r] += (double)f.y;
          }
        }
      }
      block_sum<RB>(mu, red);
#pragma unroll
      for (int r = 0; r < RB; r++) mu[r] /= (double)D;
    }
    double ss[RB];
#pragma unroll
    for (int r = 0; r < RB; r++) {
      ss[r] = 0.0;
#pragma unroll
      for (int i = 0; i < NC; i++) {
        const __half2 *h = reinterpret_cast<const __half2 *>(&raw[r][i]);
        const bool in = tid + ST * i < nchunk;     // padding chunks are zeros, not (0 - mu)
#pragma unroll
        for (int e = 0; e < 4; e++) {
          float2 f = __half22float2(h[e]);
          const double x0 = in ? (double)f.x - mu[r] : 0.0, x1 = in ? (double)f.y - mu[r] : 0.0;
          ss[r] = fma(x0, x0, ss[r]);
          ss[r] = fma(x1, x1, ss[r]);
        }
      }
    }
    block_sum<RB>(ss, red);
#pragma unroll
    for (int r = 0; r < RB; r++) {
      double inv = ss[r] > 0.0 ? 1.0 / sqrt(ss[r]) : 0.0;
#pragma unroll
      for (int i = 0; i < NC; i++) {
        const __half2 *h = reinterpret_cast<const __half2 *>(&raw[r][i]);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          float2 f = __half22float2(h[e]);
          pool[i][2 * e] = fma((double)f.x - mu[r], inv, pool[i][2 * e]);
          pool[i][2 * e + 1] = fma((double)f.y - mu[r], inv, pool[i][2 * e + 1]);
        }
      }
    }
  }
  double dot[1] = {0.0};
  const double *tb = tbar + (int64_t)b * D;
#pragma unroll
  for (int i = 0; i < NC; i++) {
    int k = tid + ST * i;
    if (k < nchunk)
#pragma unroll
      for (int e = 0; e < 8; e++) dot[0] = fma(pool[i][e], tb[8 * k + e], dot[0]);
  }
  block_sum<1>(dot, red);
  if (tid == 0) scores[(int64_t)b * W + w] = dot[0] / ((double)S * (double)N);
}

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
