// assign.cuh -- device side of wq_assign_bits (assign.cu) shared with the fused search
// kernel (search.cu): the (-key, index) bitonic sort, Q8 bands and the per-(request, layer)
// assignment body (band -> pin -> vote -> budget -> stable partition).
#pragma once
#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {


constexpr int AT = 1024;       // threads
constexpr int MAXW = 4096;     // windows per request supported

WQ_DEV bool before(double ka, int ia, double kb, int ib) {  // (-key, index) order
  return ka > kb || (ka == kb && ia < ib);
}

// Bitonic sort of n (power of two) pairs, descending key, ascending index on ties.
WQ_DEV void bitonic(double *key, int *idx, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          bool up = (i & k) == 0;
          double a = key[i], c = key[ixj];
          int ia = idx[i], ic = idx[ixj];
          bool sw = up ? before(c, ic, a, ia) : before(a, ia, c, ic);
          if (sw) {
            key[i] = c; key[ixj] = a;
            idx[i] = ic; idx[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
}

WQ_DEV int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Q8: level = [x >= T1] + sum_{interior} [x >= Tj] + [x > T_top]  (n >= 3)
WQ_DEV int band_level(double x, const double *T, int n) {
  if (n == 1) return 0;
  if (n == 2) return x > T[0] ? 1 : 0;
  int lv = x >= T[0] ? 1 : 0;
  for (int j = 1; j < n - 2; j++) lv += x >= T[j] ? 1 : 0;
  lv += x > T[n - 2] ? 1 : 0;
  return lv;
}

WQ_DEV int cls_of(int bits) { return bits == 2 ? 0 : bits == 4 ? 1 : bits == 8 ? 2 : 3; }

// Block-wide exclusive scan of one uint64 per thread (fixed order).
WQ_DEV uint64_t block_exscan_u64(uint64_t v, uint64_t *warp_tot /* [32] */, uint64_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t t = lane < nw ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;  // inclusive
  }
  __syncthreads();
  uint64_t before_w = warp == 0 ? 0 : warp_tot[warp - 1];
  *total = warp_tot[nw - 1];
  uint64_t r = before_w + x - v;
  __syncthreads();
  return r;
}

// The assignment of (request b, layer l) by one CTA of NT threads (k_assign: NT = AT; the
// fused search kernel: NT = 128).  order: NULL, or the precomputed (-key, index) order of
// the budget ranking (idx[r] = window at rank r; the batch-mean order under the vote),
// which then replaces the in-CTA sort.
template <int NT>
WQ_DEV void assign_body(const double *__restrict__ scores, const AssignParams &p, uint8_t *__restrict__ bits_out,
                        int32_t *__restrict__ perm_out, int32_t *__restrict__ seg_out, int b, int l,
                        const int32_t *__restrict__ order, uint8_t *sm, uint64_t *warp_tot, int *s_rstar_p) {
  constexpr int PER = MAXW / NT; // windows per thread (contiguous)
  const int W = p.W, B = p.B, n = p.n_widths;
  const int np = pow2_at_least(W);
  double *key = reinterpret_cast<double *>(sm);               // [np]
  int *idx = reinterpret_cast<int *>(key + np);               // [np]
  int *bits = idx + np;                                       // [W]
  int &s_rstar = *s_rstar_p;
  const int tid = threadIdx.x;
  const double *T = p.thr + l * 3;
  const int wmin = p.widths[0];

  // ---- band, vote, pin ----
  for (int w = tid; w < W; w += NT) {
    int bw;
    if (p.vote) {
      int cnt[4] = {0, 0, 0, 0};
      for (int bb = 0; bb < B; bb++) {
        int x = (p.pin && w == 0) ? 16 : p.widths[band_level(scores[(int64_t)bb * W + w], T, n)];
        cnt[cls_of(x)]++;
      }
      int best = 0;
      for (int k = 1; k < 4; k++)
        if (cnt[k] >= cnt[best]) best = k;
      bw = 2 << best;  // class k -> 2,4,8,16
    } else {
      bw = p.widths[band_level(scores[(int64_t)b * W + w], T, n)];
      if (p.pin && w == 0) bw = 16;
    }
    bits[w] = bw;
  }
  __syncthreads();

  // ---- budget (Q13) ----
  if (p.budget > 0.0) {
    if (order) {
      for (int r = tid; r < W; r += NT) idx[r] = order[r];   // the precomputed rank order
    } else {
      for (int i = tid; i < np; i += NT) {
        double kv = -INFINITY;
        if (i < W) {
          if (p.vote) {
            double s = 0.0;
            for (int bb = 0; bb < B; bb++) s += scores[(int64_t)bb * W + i];
            kv = s / (double)B;
          } else {
            kv = scores[(int64_t)b * W + i];
          }
        }
        key[i] = kv;
        idx[i] = i < W ? i : 0x7fffffff;
      }
      __syncthreads();
      bitonic(key, idx, np);  // idx[r] = window at rank r
    }
    __syncthreads();
    // reduction available at rank position r (demote fully to wmin)
    long long red_local[PER];
    long long tot_local = 0;
    uint64_t sum_red = 0;
    for (int e = 0; e < PER; e++) {
      int r = tid * PER + e;
      long long rv = 0;
      if (r < W) {
        int w = idx[r];
        tot_local += bits[w];
        if (!(p.pin && w == 0)) rv = bits[w] - wmin;
      }
      red_local[e] = rv;
      sum_red += (uint64_t)rv;
    }
    uint64_t tot_all;
    block_exscan_u64((uint64_t)tot_local, warp_tot, &tot_all);
    const long long total = (long long)tot_all;
    const double limit = p.budget * (double)W;
    // suffix sums from the bottom: Suf(r) = sum_{r' >= r} red[r'] = R_all - prefix(r)
    uint64_t red_all;
    uint64_t pre = block_exscan_u64(sum_red, warp_tot, &red_all);
    if (tid == 0) s_rstar = -1;
    __syncthreads();
    if ((double)total > limit) {
      long long acc = (long long)pre;  // sum of red over ranks < tid*PER
      for (int e = 0; e < PER; e++) {
        int r = tid * PER + e;
        if (r >= W) break;
        long long suf_r = (long long)red_all - acc;           // Suf(r)
        long long suf_r1 = suf_r - red_local[e];              // Suf(r+1)
        bool ok_r = (double)(total - suf_r) <= limit;
        bool ok_r1 = (double)(total - suf_r1) <= limit;
        if (ok_r && !ok_r1) s_rstar = r;                      // unique
        acc += red_local[e];
      }
      __syncthreads();
      const int rstar = s_rstar;
      if (rstar >= 0) {
        // fully demote ranks > rstar (non-pinned), then step rank rstar
        for (int e = 0; e < PER; e++) {
          int r = tid * PER + e;
          if (r < W && r > rstar) {
            int w = idx[r];
            if (!(p.pin && w == 0)) bits[w] = wmin;
          }
        }
        __syncthreads();
        if (tid == 0) {
          long long t = 0;
          for (int w = 0; w < W; w++) t += bits[w];
          // bits of rstar not yet touched: t already includes the full demotions
          int w = idx[rstar];
          while ((double)t > limit && bits[w] > wmin) {
            int k = 0;
            while (p.widths[k] != bits[w]) k++;
            t -= bits[w] - p.widths[k - 1];
            bits[w] = p.widths[k - 1];
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- stable partition by width class (Alg.2) ----
  uint64_t cnt = 0;  // 4 x 16-bit class counters of this thread's windows
  for (int e = 0; e < PER; e++) {
    int w = tid * PER + e;
    if (w < W) cnt += 1ull << (16 * cls_of(bits[w]));
  }
  uint64_t all;
  uint64_t pre = block_exscan_u64(cnt, warp_tot, &all);
  int seg[5];
  seg[0] = 0;
  for (int k = 0; k < 4; k++) seg[k + 1] = seg[k] + (int)((all >> (16 * k)) & 0xffff);
  int run[4];
  for (int k = 0; k < 4; k++) run[k] = seg[k] + (int)((pre >> (16 * k)) & 0xffff);
  const int nb_out = p.vote ? B : 1;
  for (int e = 0; e < PER; e++) {
    int w = tid * PER + e;
    if (w >= W) break;
    int k = cls_of(bits[w]);
    int slot = run[k]++;
    WQ_CHECK(slot >= seg[k] && slot < seg[k + 1]);
    for (int bo = 0; bo < nb_out; bo++) {
      int bb = p.vote ? bo : b;
      int64_t row = (int64_t)l * B + bb;
      perm_out[row * W + slot] = w;
      bits_out[row * W + w] = (uint8_t)bits[w];
    }
  }
  if (tid < 5)
    for (int bo = 0; bo < nb_out; bo++) {
      int bb = p.vote ? bo : b;
      seg_out[((int64_t)l * B + bb) * 5 + tid] = seg[tid];
    }
}

}  // namespace wq
