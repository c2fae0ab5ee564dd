// scores.cuh -- device side of wq_window_scores (scores.cu) shared with the fused search
// kernel (search.cu): deterministic block sums, the text pool and the window-score
// kernels' bodies.
#pragma once
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

// tbar[b] of request b by one CTA of ST threads; pooled: shared [D] doubles (>= 8), red:
// shared [4].  Rows are taken in batches of NB: (A) a warp per row computes its mean
// (Pearson) and inverse norm with lane-strided 16-byte loads and a shuffle tree into
// pooled; (B) each thread accumulates its NC channel chunks over the batch's rows in row
// order (independent loads, no barrier per row).  tbar[b][c] = sum_j (x_j[c] - mu_j) /
// ||x_j - mu_j|| in ascending j for every c (a zero row contributes 0).
template <int NC, bool CENTER>
WQ_DEV void text_pool_body(const __half *__restrict__ txt, int64_t trs, int64_t tbs, int N, int D,
                           double *__restrict__ tbar, int b, double *pooled, double *red) {
  (void)red;
  const int nchunk = D / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NB = D / 2 < 32 ? D / 2 : 32;        // rows per batch ((mu, inv) pairs in pooled)
  double acc[NC][8];
#pragma unroll
  for (int i = 0; i < NC; i++)
#pragma unroll
    for (int e = 0; e < 8; e++) acc[i][e] = 0.0;
  const __half *base = txt + b * tbs;
  for (int j0 = 0; j0 < N; j0 += NB) {
    const int nb = N - j0 < NB ? N - j0 : NB;
    for (int jj = warp; jj < nb; jj += ST / 32) {
      const __half *row = base + (int64_t)(j0 + jj) * trs;
      double mu = 0.0;
      if (CENTER) {
        double sm = 0.0;
        for (int k = lane; k < nchunk; k += 32) {
          double x[8];
          load8(row + 8 * k, x);
#pragma unroll
          for (int e = 0; e < 8; e++) sm += x[e];
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
        mu = sm / (double)D;
      }
      double ss = 0.0;
      for (int k = lane; k < nchunk; k += 32) {
        double x[8];
        load8(row + 8 * k, x);
#pragma unroll
        for (int e = 0; e < 8; e++) ss = fma(x[e] - mu, x[e] - mu, ss);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) {
        pooled[2 * jj] = mu;
        pooled[2 * jj + 1] = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NC; i++) {
      const int k = threadIdx.x + ST * i;
      if (k < nchunk) {
#pragma unroll 4
        for (int jj = 0; jj < nb; jj++) {
          double x[8];
          load8(base + (int64_t)(j0 + jj) * trs + 8 * k, x);
          const double m = pooled[2 * jj], inv = pooled[2 * jj + 1];
#pragma unroll
          for (int e = 0; e < 8; e++) acc[i][e] = fma(x[e] - m, inv, acc[i][e]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < NC; i++) {
    const int k = threadIdx.x + ST * i;
    if (k < nchunk)
#pragma unroll
      for (int e = 0; e < 8; e++) tbar[(int64_t)b * D + 8 * k + e] = acc[i][e];
  }
  __syncthreads();
}

// A visual "row" is D elements; with head-split rows (the per-layer scorer) element c lives
// at row + (c / dh) * hs + c % dh (dh = head dim, hs = head stride); dh = D, hs = 0 otherwise.
// score of window w of request b by one CTA of ST threads; red: shared [4 * WQ_SC_RB]
// NC: 16-byte chunks per thread per row, ceil(D / 8 / ST); CENTER: Pearson; HS: head-split rows
template <int NC, bool CENTER, bool HS = false>
WQ_DEV void window_score_body(const __half *__restrict__ vis, int64_t vrs, int64_t vbs, int M, int N, int D, int S,
                              const double *__restrict__ tbar, double *__restrict__ scores, int dh, int64_t hs,
                              int w, int b, int W, double *red) {
  constexpr int RB = WQ_SC_RB;  // rows per batch
  const int tid = threadIdx.x;
  const int nchunk = D / 8;
  double pool[NC][8];
#pragma unroll
  for (int i = 0; i < NC; i++)
#pragma unroll
    for (int e = 0; e < 8; e++) pool[i][e] = 0.0;
  const __half *base = vis + b * vbs + (int64_t)w * S * vrs;
  // element offset of each of the thread's chunks inside a row (the same for every row;
  // computed once: a division per load cost 560 -> 760 us on C5)
  // (32-bit: the launcher checks (D / dh - 1) * hs + dh < 2^31; without head split the
  // offset is the element index itself)
  int coff[NC];
#pragma unroll
  for (int i = 0; i < NC; i++) {
    const int c = 8 * (tid + ST * i);                       // first element of the chunk
    coff[i] = HS ? (int)((int64_t)(c / dh) * hs + c % dh) : 0;
  }
  for (int r0 = 0; r0 < S; r0 += RB) {
    uint4 raw[RB][NC];
#pragma unroll
    for (int r = 0; r < RB; r++)
#pragma unroll
      for (int i = 0; i < NC; i++) {
        const int k = tid + ST * i;
        raw[r][i] = k < nchunk ? __ldcs(reinterpret_cast<const uint4 *>(base + (int64_t)(r0 + r) * vrs +
                                                                      (HS ? coff[i] : 8 * k)))
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

}  // namespace wq

namespace wq {
template <int NC, bool CENTER>
__global__ void __launch_bounds__(ST) k_text_pool(const __half *__restrict__ txt, int64_t trs,
                                                  int64_t tbs, int N, int D, double *__restrict__ tbar) {
  extern __shared__ double pooled[];  // [D]
  __shared__ double red[4];
  text_pool_body<NC, CENTER>(txt, trs, tbs, N, D, tbar, blockIdx.x, pooled, red);
}

template <int NC, bool CENTER, bool HS>
__global__ void __launch_bounds__(ST, CENTER ? 2 : WQ_SC_MINB) k_window_scores(const __half *__restrict__ vis, int64_t vrs,
                                                      int64_t vbs, int M, int N, int D, int S,
                                                      const double *__restrict__ tbar,
                                                      double *__restrict__ scores, int dh, int64_t hs) {
  __shared__ double red[4 * WQ_SC_RB];
  window_score_body<NC, CENTER, HS>(vis, vrs, vbs, M, N, D, S, tbar, scores, dh, hs, blockIdx.x, blockIdx.y, gridDim.x,
                                red);
}
}  // namespace wq
