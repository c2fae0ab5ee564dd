// quant.cu -- wq_layer_layout and wq_reorder_quantize_pack (Alg.2 prefill
// branch P:420-446, Eq.14-16, group = window P:508, readings Q17-Q22).
//
// One CTA per (slot, kv-head, request).  The window's fp16 K and V rows are pulled
// into shared memory by the TMA bulk-copy engine (one cp.async.bulk per tensor when
// rows are contiguous), per-channel K and per-token V (min, max) are reduced with
// fp16x2 min/max, the fp32 quantizer contract (Q17) runs per element with explicit
// round-to-nearest intrinsics (no FMA contraction), and the record is written in
// D-1 fragment order with 16-byte stores at the window's REORDERED slot (so the
// reorder of Alg.2 is an address remap, not a copy).
#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {

// offs[b*H + h] of one layer from seg_off_l[B][5]; one thread per request, then a
// serial prefix (B <= 4096) by thread 0 -- tiny.
__global__ void k_layer_layout(const int32_t *__restrict__ seg_off, int B, int H, int d, int S,
                               int64_t *__restrict__ offs) {
  extern __shared__ int64_t img[];
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int32_t *so = seg_off + 5 * b;
    int64_t t = 0;
    for (int k = 0; k < 4; k++) t += (int64_t)(so[k + 1] - so[k]) * record_bytes(class_bits(k), d, S);
    img[b] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t off = 0;
    for (int b = 0; b < B; b++)
      for (int h = 0; h < H; h++) {
        offs[(int64_t)b * H + h] = off;
        off += img[b];
      }
    offs[(int64_t)B * H] = off;
  }
}

constexpr int QT = 256;  // threads per quantize CTA

struct QuantArgs {
  const __half *k, *v;
  int64_t sb, sh, st;     // strides in elements (b, h, t); channel stride 1
  int vis_off;
  int B, H, d, S;
  const int32_t *perm;
  int perm_stride;
  const int32_t *seg_off;
  const int64_t *offs;
  uint8_t *packed;
};

// 16-byte unit ui of a code tile, word e -> (lane, word in the lane's chunk) (D-1:
// chunks of >= 16 bytes are interleaved in 16-byte groups, 8-byte chunks are linear)
WQ_DEV void unit_lane_word(int ui, int e, int chunk_words, int &L, int &wl) {
  if (chunk_words >= 4) {
    L = ui & 31;
    wl = 4 * (ui >> 5) + e;
  } else {
    L = 2 * ui + (e >> 1);
    wl = e & 1;
  }
}

// Q17 on one element: clamp(rint(fl(fl(x - mn) * r)), 0, qmax).  prod >= +0 (x >= mn,
// r > 0); clamping the float to qmax before rounding gives the same integer as
// clamping after it, and adding 1.5*2^23 rounds to nearest-even exactly like
// cvt.rni for |prod| < 2^22 -- the code is then the low mantissa bits.
WQ_DEV uint32_t q17_code(float x, float mn, float r, float qmaxf) {
  float prod = __fmul_rn(__fsub_rn(x, mn), r);
  prod = fminf(prod, qmaxf);
  const float big = __fadd_rn(prod, 12582912.0f);
  return __float_as_uint(big) & 0xFFu;
}

// Codes of one window in D-1 fragment order: 16-byte units, thread-strided.  For
// each unit the lane L and its chunk words follow D-1 (unit_lane_word); every pair
// is two Q17 codes of adjacent columns (K) / adjacent tokens (V).
template <int D, int S, int BITS>
WQ_DEV void pack_codes(const __half *Ks, const __half *Vs, const float2 *kp2, const float2 *vp2,
                       uint4 *dst, int tid) {
  constexpr int PPW = 16 / BITS;
  constexpr int CW = D * BITS / 64;           // chunk words per lane
  constexpr int UPT = 2 * D * BITS / 16;      // 16-byte units per tile
  constexpr int UNITS = (S / 16) * UPT;       // per tensor
  constexpr float QMAX = (float)((1 << BITS) - 1);
  constexpr uint32_t MASK = (1u << BITS) - 1u;
  // K: rows = tokens, cols = channels
  for (int u = tid; u < UNITS; u += QT) {
    const int tile = u / UPT, ui = u % UPT;
    uint32_t wv[4];
#pragma unroll
    for (int e = 0; e < 4; e++) {
      int L, wl;
      unit_lane_word(ui, e, CW, L, wl);
      const int g = L >> 2, q = L & 3;
      const __half *kb = Ks + (tile * 16 + g) * D + 2 * q;
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < PPW; j++) {
        const int P = wl * PPW + j, m = P >> 2, r = P & 3;
        const int col = 16 * m + 8 * (r >> 1);
        const float2 x = __half22float2(*reinterpret_cast<const __half2 *>(kb + 8 * (r & 1) * D + col));
        const float4 pr = *reinterpret_cast<const float4 *>(kp2 + col + 2 * q);
        const uint32_t c0 = q17_code(x.x, pr.x, pr.y, QMAX) & MASK;
        const uint32_t c1 = q17_code(x.y, pr.z, pr.w, QMAX) & MASK;
        acc |= (c0 << (BITS * j)) | (c1 << (16 + BITS * j));
      }
      wv[e] = acc;
    }
    dst[u] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  // V: rows = channels, cols = tokens
  uint4 *vdst = dst + UNITS;
  for (int u = tid; u < UNITS; u += QT) {
    const int tile = u / UPT, ui = u % UPT;
    uint32_t wv[4];
#pragma unroll
    for (int e = 0; e < 4; e++) {
      int L, wl;
      unit_lane_word(ui, e, CW, L, wl);
      const int g = L >> 2, q = L & 3;
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < PPW; j++) {
        const int P = wl * PPW + j, m = P >> 2, r = P & 3;
        const int ch = 16 * m + g + 8 * (r & 1), t = tile * 16 + 2 * q + 8 * (r >> 1);
        const float4 pr = *reinterpret_cast<const float4 *>(vp2 + t);     // {mn, r} of t, t+1
        const uint32_t c0 = q17_code(__half2float(Vs[t * D + ch]), pr.x, pr.y, QMAX) & MASK;
        const uint32_t c1 = q17_code(__half2float(Vs[(t + 1) * D + ch]), pr.z, pr.w, QMAX) & MASK;
        acc |= (c0 << (BITS * j)) | (c1 << (16 + BITS * j));
      }
      wv[e] = acc;
    }
    vdst[u] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

// Quantize + pack one staged window (K, V rows in shared memory) into rec.
template <int D, int S>
WQ_DEV void quant_window(const __half *Ks, const __half *Vs, float2 *kp2, float2 *vp2, __half2 *red,
                         uint8_t *params, uint8_t *rec, int bits, int tid) {

  const int64_t code_bytes = (int64_t)S * D * bits / 8;      // one of K or V
  if (bits == 16) {
    // FP16 window: values re-laid in fragment order (pairs of adjacent columns).
    // word index u over K tiles then V tiles: tile i, lane L, pair P = word in lane chunk
    constexpr int UPT = 32 * D / 16;                         // 16-byte units per tile
    constexpr int UNITS = (S / 16) * UPT;                    // per tensor
    uint4 *dst = reinterpret_cast<uint4 *>(rec);
    for (int u4 = tid; u4 < 2 * UNITS; u4 += QT) {
      const int isv = u4 >= UNITS;
      const int uu = isv ? u4 - UNITS : u4;
      const int tile = uu / UPT, ui = uu % UPT;
      uint32_t wv[4];
#pragma unroll
      for (int e = 0; e < 4; e++) {
        int L, P;
        unit_lane_word(ui, e, D / 4, L, P);
        int g = L >> 2, q = L & 3, m = P >> 2, r = P & 3;
        if (!isv) {
          int row = tile * 16 + g + 8 * (r & 1), col = 16 * m + 2 * q + 8 * (r >> 1);
          wv[e] = *reinterpret_cast<const uint32_t *>(Ks + row * D + col);
        } else {
          int ch = 16 * m + g + 8 * (r & 1), t = tile * 16 + 2 * q + 8 * (r >> 1);
          uint32_t lo = __half_as_ushort(Vs[t * D + ch]);
          uint32_t hi = __half_as_ushort(Vs[(t + 1) * D + ch]);
          wv[e] = lo | (hi << 16);
        }
      }
      dst[u4] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    return;
  }

  const int qmax = (1 << bits) - 1;
  const float qmaxf = (float)qmax;

  // ---- K: per-channel (min, max) over the S tokens ----
  {
    constexpr int CP = D / 2;                 // channel pairs
    constexpr int TG = QT / CP;               // token groups
    const int cp = tid % CP, tg = tid / CP;
    __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
    for (int t = tg; t < S; t += TG) {
      __half2 x = *reinterpret_cast<const __half2 *>(Ks + t * D + 2 * cp);
      mn2 = __hmin2(mn2, x);
      mx2 = __hmax2(mx2, x);
    }
    red[2 * tid] = mn2;
    red[2 * tid + 1] = mx2;
    __syncthreads();
    if (tid < CP) {
      for (int g2 = 1; g2 < TG; g2++) {
        mn2 = __hmin2(mn2, red[2 * (g2 * CP + cp)]);
        mx2 = __hmax2(mx2, red[2 * (g2 * CP + cp) + 1]);
      }
#pragma unroll
      for (int e = 0; e < 2; e++) {
        int c = 2 * cp + e;
        float mn = __half2float(e ? __high2half(mn2) : __low2half(mn2));
        float mx = __half2float(e ? __high2half(mx2) : __low2half(mx2));
        __half s16 = __float2half_ru(__fdiv_rn(__fsub_rn(mx, mn), qmaxf));
        if (__half2float(s16) < 5.9604644775390625e-08f) s16 = __ushort_as_half(0x0001);
        kp2[c] = make_float2(mn, __frcp_rn(__half2float(s16)));
        int m = c / 16, q = (c % 8) / 2, hh = (c % 16) / 8;
        __half *grp = reinterpret_cast<__half *>(params + (q * (D / 16) + m) * 16);
        grp[4 * hh + e] = __float2half_rn(mn);      // D-1 K group {mn01, s01, mn89, s89}
        grp[4 * hh + 2 + e] = s16;
      }
    }
  }
  // ---- V: per-token (min, max) over the D channels ----
  {
    constexpr int TPT = QT / S;               // threads per token
    constexpr int CH = D / TPT;               // channels per thread (multiple of 2)
    const int t = tid / TPT, part = tid % TPT;
    __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
#pragma unroll
    for (int c = 0; c < CH; c += 2) {
      __half2 x = *reinterpret_cast<const __half2 *>(Vs + t * D + part * CH + c);
      mn2 = __hmin2(mn2, x);
      mx2 = __hmax2(mx2, x);
    }
    __half mn = __hmin(__low2half(mn2), __high2half(mn2));
    __half mx = __hmax(__low2half(mx2), __high2half(mx2));
#pragma unroll
    for (int o = TPT / 2; o >= 1; o >>= 1) {
      mn = __hmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = __hmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (part == 0) {
      float mnf = __half2float(mn), mxf = __half2float(mx);
      __half s16 = __float2half_ru(__fdiv_rn(__fsub_rn(mxf, mnf), qmaxf));
      if (__half2float(s16) < 5.9604644775390625e-08f) s16 = __ushort_as_half(0x0001);
      vp2[t] = make_float2(mnf, __frcp_rn(__half2float(s16)));
      int i = t / 16, col = t % 16, q = (col % 8) / 2, hh = col / 8, e = col % 2;
      __half *grp = reinterpret_cast<__half *>(params + 4 * D + (4 * i + q) * 16);
      grp[2 * hh + e] = s16;
      grp[4 + 2 * hh + e] = mn;
    }
  }
  __syncthreads();

  // ---- codes in fragment order (templated per width: unrolled, constant shifts) ----
  uint4 *dst = reinterpret_cast<uint4 *>(rec);
  switch (bits) {
    case 2: pack_codes<D, S, 2>(Ks, Vs, kp2, vp2, dst, tid); break;
    case 4: pack_codes<D, S, 4>(Ks, Vs, kp2, vp2, dst, tid); break;
    default: pack_codes<D, S, 8>(Ks, Vs, kp2, vp2, dst, tid); break;
  }
  // ---- params (K then V) after the codes ----
  uint4 *pdst = reinterpret_cast<uint4 *>(rec + 2 * code_bytes);
  const uint4 *psrc = reinterpret_cast<const uint4 *>(params);
  for (int i = tid; i < (4 * D + 4 * S) / 16; i += QT) pdst[i] = psrc[i];
}

// Persistent kernel: each CTA walks windows blockIdx.x, +gridDim.x, ... of the
// flattened (request, kv head, slot) space with an NSTG-deep TMA ring, so the
// next windows stream in while the current one is quantized.
template <int D, int S>
struct QuantSmem {
  static constexpr int WIN = 4 * S * D;                     // K + V bytes of one window
  static constexpr int NSTG = WIN >= 65536 ? 2 : 3;
  static constexpr size_t ring = (size_t)NSTG * WIN;
  static constexpr size_t total = ring + (2 * D + 2 * S) * 8 + 2 * QT * 4 + 4 * D + 4 * S + 64;
};

template <int D, int S>
__global__ void __launch_bounds__(QT) k_quant(QuantArgs a) {
  using QS = QuantSmem<D, S>;
  constexpr int NSTG = QS::NSTG;
  extern __shared__ __align__(128) uint8_t sm[];
  float2 *kp2 = reinterpret_cast<float2 *>(sm + QS::ring);  // [D] {mn, 1/s} per channel
  float2 *vp2 = kp2 + D;                                     // [S] {mn, 1/s} per token
  __half2 *red = reinterpret_cast<__half2 *>(vp2 + S);       // [QT] x (min2, max2)
  uint8_t *params = reinterpret_cast<uint8_t *>(red + 2 * QT);  // [4D + 4S]
  __shared__ uint64_t bar[NSTG];
  const int tid = threadIdx.x;
  const int total = a.B * a.H * a.perm_stride;

  // window k of this CTA -> (b, h, slot); valid if slot < seg_off[b][4]
  auto locate = [&](int k, int &b, int &h, int &slot) -> bool {
    const int idx = blockIdx.x + k * gridDim.x;
    if (idx >= total) return false;
    slot = idx % a.perm_stride;
    const int bh = idx / a.perm_stride;
    h = bh % a.H;
    b = bh / a.H;
    return true;
  };
  auto issue = [&](int k) {                       // thread 0: TMA of window k into its stage
    int b, h, slot;
    if (!locate(k, b, h, slot)) return;
    if (slot >= a.seg_off[5 * b + 4]) {           // no window: complete the phase anyway
      mbar_arrive(&bar[k % NSTG]);
      return;
    }
    const int w = a.perm[(int64_t)b * a.perm_stride + slot];
    const __half *K0 = a.k + b * a.sb + h * a.sh + (int64_t)(a.vis_off + w * S) * a.st;
    const __half *V0 = a.v + b * a.sb + h * a.sh + (int64_t)(a.vis_off + w * S) * a.st;
    __half *Ks = reinterpret_cast<__half *>(sm + (size_t)(k % NSTG) * QS::WIN);
    __half *Vs = Ks + S * D;
    uint64_t *bb = &bar[k % NSTG];
    constexpr uint32_t ROW = D * 2;
    mbar_arrive_expect_tx(bb, 2u * S * ROW);
    const uint64_t pol = policy_evict_first();
    if (a.st == D) {
      bulk_g2s_evict_first(Ks, K0, S * ROW, bb, pol);
      bulk_g2s_evict_first(Vs, V0, S * ROW, bb, pol);
    } else {
      for (int t = 0; t < S; t++) {
        bulk_g2s_evict_first(Ks + t * D, K0 + t * a.st, ROW, bb, pol);
        bulk_g2s_evict_first(Vs + t * D, V0 + t * a.st, ROW, bb, pol);
      }
    }
  };
  if (tid == 0) {
    for (int i = 0; i < NSTG; i++) mbar_init(&bar[i], 1);
    fence_mbar_init();
    for (int k = 0; k < NSTG - 1; k++) issue(k);
  }
  __syncthreads();
  for (int k = 0;; k++) {
    int b, h, slot;
    if (!locate(k, b, h, slot)) break;
    if (tid == 0) issue(k + NSTG - 1);            // its stage was released by the last barrier
    const int32_t *so = a.seg_off + 5 * b;
    if (slot < so[4]) {
      int cls = 0;
      while (slot >= so[cls + 1]) cls++;
      const int bits = class_bits(cls);
      int64_t roff = a.offs[(int64_t)b * a.H + h];
      for (int kk = 0; kk < cls; kk++) roff += (int64_t)(so[kk + 1] - so[kk]) * record_bytes(class_bits(kk), D, S);
      roff += (int64_t)(slot - so[cls]) * record_bytes(bits, D, S);
      mbar_wait(&bar[k % NSTG], (uint32_t)(k / NSTG) & 1u);
      const __half *Ks = reinterpret_cast<const __half *>(sm + (size_t)(k % NSTG) * QS::WIN);
      quant_window<D, S>(Ks, Ks + S * D, kp2, vp2, red, params, a.packed + roff, bits, tid);
    }
    __syncthreads();
  }
}

template <int D, int S>
static cudaError_t launch_quant_t(const QuantArgs &a, cudaStream_t st) {
  using QS = QuantSmem<D, S>;
  const size_t smem = QS::total;
  cudaError_t e = cudaFuncSetAttribute(k_quant<D, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_quant<D, S>, QT, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t total = (int64_t)a.B * a.H * a.perm_stride;
  int64_t grid = (int64_t)device_sm_count() * per_sm;
  if (grid > total) grid = total;
  if (grid < 1) grid = 1;
  k_quant<D, S><<<(unsigned)grid, QT, smem, st>>>(a);
  return cudaGetLastError();
}

// wq_shard_slots: one CTA per request; rank r keeps chunk r of every segment.
__global__ void k_shard_slots(const int32_t *__restrict__ perm, const int32_t *__restrict__ seg, int W,
                              int G, int r, int32_t *__restrict__ perm_r, int32_t *__restrict__ seg_r) {
  const int b = blockIdx.x;
  const int32_t *so = seg + 5 * b;
  int lo[4], cnt[4], start[5];
  start[0] = 0;
  for (int k = 0; k < 4; k++) {
    const int n = so[k + 1] - so[k];
    lo[k] = so[k] + (int)((int64_t)n * r / G);
    cnt[k] = so[k] + (int)((int64_t)n * (r + 1) / G) - lo[k];
    start[k + 1] = start[k] + cnt[k];
  }
  for (int k = 0; k < 4; k++)
    for (int i = threadIdx.x; i < cnt[k]; i += blockDim.x)
      perm_r[(int64_t)b * W + start[k] + i] = perm[(int64_t)b * W + lo[k] + i];
  if (threadIdx.x < 5) seg_r[5 * b + threadIdx.x] = start[threadIdx.x];
}


cudaError_t launch_shard_slots(const int32_t *perm, const int32_t *seg, int B, int W, int G, int r,
                               int32_t *perm_r, int32_t *seg_r, cudaStream_t st) {
  k_shard_slots<<<B, 256, 0, st>>>(perm, seg, W, G, r, perm_r, seg_r);
  return cudaGetLastError();
}

cudaError_t launch_layer_layout(const int32_t *seg_off, int B, int H, int d, int S, int64_t *offs,
                                cudaStream_t st) {
  k_layer_layout<<<1, 256, (size_t)B * sizeof(int64_t), st>>>(seg_off, B, H, d, S, offs);
  return cudaGetLastError();
}

cudaError_t launch_quant(const __half *k, const __half *v, const int64_t strides[3], int vis_off,
                         int B, int H, int d, int S, const int32_t *perm, int perm_stride,
                         const int32_t *seg_off, const int64_t *offs, uint8_t *packed,
                         cudaStream_t st) {
  QuantArgs a{k, v, strides[0], strides[1], strides[2], vis_off, B, H, d, S, perm, perm_stride,
              seg_off, offs, packed};
#define WQ_Q(DD, SS) \
  if (d == DD && S == SS) return launch_quant_t<DD, SS>(a, st);
  WQ_Q(64, 16) WQ_Q(64, 32) WQ_Q(64, 64) WQ_Q(64, 128)
  WQ_Q(128, 16) WQ_Q(128, 32) WQ_Q(128, 64) WQ_Q(128, 128)
#undef WQ_Q
  return cudaErrorInvalidValue;
}

}  // namespace wq
