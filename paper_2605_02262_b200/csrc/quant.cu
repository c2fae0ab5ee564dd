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

// Q17 on one element: clamp(rint(fl(fl(x - mn) * r)), 0, qmax)
WQ_DEV uint32_t q17_code(float x, float mn, float r, int qmax) {
  float prod = __fmul_rn(__fsub_rn(x, mn), r);
  int c = __float2int_rn(prod);
  c = c < 0 ? 0 : c;
  c = c > qmax ? qmax : c;
  return (uint32_t)c;
}

template <int D, int S>
__global__ void __launch_bounds__(QT) k_quant(QuantArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __half *Ks = reinterpret_cast<__half *>(sm);              // [S][D]
  __half *Vs = Ks + S * D;                                   // [S][D]
  float *kmn = reinterpret_cast<float *>(Vs + S * D);        // [D]
  float *kr = kmn + D;                                       // [D]
  float *vmn = kr + D;                                       // [S]
  float *vr = vmn + S;                                       // [S]
  __half2 *red = reinterpret_cast<__half2 *>(vr + S);        // [QT] x (min2, max2)
  uint8_t *params = reinterpret_cast<uint8_t *>(red + 2 * QT);  // [4D + 4S]
  __shared__ uint64_t bar;

  const int slot = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int32_t *so = a.seg_off + 5 * b;
  if (slot >= so[4]) return;
  int cls = 0;
  while (slot >= so[cls + 1]) cls++;
  const int bits = class_bits(cls);
  int64_t roff = a.offs[(int64_t)b * a.H + h];
  for (int k = 0; k < cls; k++) roff += (int64_t)(so[k + 1] - so[k]) * record_bytes(class_bits(k), D, S);
  roff += (int64_t)(slot - so[cls]) * record_bytes(bits, D, S);
  uint8_t *rec = a.packed + roff;
  const int w = a.perm[(int64_t)b * a.perm_stride + slot];
  const __half *K0 = a.k + b * a.sb + h * a.sh + (int64_t)(a.vis_off + w * S) * a.st;
  const __half *V0 = a.v + b * a.sb + h * a.sh + (int64_t)(a.vis_off + w * S) * a.st;
  const int tid = threadIdx.x;

  // ---- stage the window (TMA bulk copies) ----
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    constexpr uint32_t ROW = D * 2;
    mbar_arrive_expect_tx(&bar, 2u * S * ROW);
    uint64_t pol = policy_evict_first();
    if (a.st == D) {
      bulk_g2s_evict_first(Ks, K0, S * ROW, &bar, pol);
      bulk_g2s_evict_first(Vs, V0, S * ROW, &bar, pol);
    } else {
      for (int t = 0; t < S; t++) {
        bulk_g2s_evict_first(Ks + t * D, K0 + t * a.st, ROW, &bar, pol);
        bulk_g2s_evict_first(Vs + t * D, V0 + t * a.st, ROW, &bar, pol);
      }
    }
  }
  mbar_wait(&bar, 0);

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
        kmn[c] = mn;
        kr[c] = __frcp_rn(__half2float(s16));
        int m = c / 16, q = (c % 8) / 2, hh = (c % 16) / 8;
        __half *grp = reinterpret_cast<__half *>(params + (q * (D / 16) + m) * 16);
        grp[2 * hh + e] = s16;
        grp[4 + 2 * hh + e] = __float2half_rn(mn);
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
      vmn[t] = mnf;
      vr[t] = __frcp_rn(__half2float(s16));
      int i = t / 16, col = t % 16, q = (col % 8) / 2, hh = col / 8, e = col % 2;
      __half *grp = reinterpret_cast<__half *>(params + 4 * D + (4 * i + q) * 16);
      grp[2 * hh + e] = s16;
      grp[4 + 2 * hh + e] = mn;
    }
  }
  __syncthreads();

  // ---- codes in fragment order, 16 bytes (4 words) per thread-iteration ----
  const int ppw = 16 / bits;                  // pairs per word
  const int chunk_words = D * bits / 64;      // (D/4 pairs) / ppw
  const int upt = 2 * D * bits / 16;          // 16-byte units per tile
  const int units = (S / 16) * upt;           // per tensor
  uint4 *dst = reinterpret_cast<uint4 *>(rec);
  for (int u4 = tid; u4 < 2 * units; u4 += QT) {
    const int isv = u4 >= units;
    const int uu = isv ? u4 - units : u4;
    const int tile = uu / upt, ui = uu % upt;
    uint32_t wv[4];
#pragma unroll
    for (int e4 = 0; e4 < 4; e4++) {
      int L, wl;
      unit_lane_word(ui, e4, chunk_words, L, wl);
      int g = L >> 2, q = L & 3;
      uint32_t acc = 0;
      for (int j = 0; j < ppw; j++) {
        int P = wl * ppw + j, m = P >> 2, r = P & 3;
        uint32_t c0, c1;
        if (!isv) {
          int row = tile * 16 + g + 8 * (r & 1), col = 16 * m + 2 * q + 8 * (r >> 1);
          __half2 x = *reinterpret_cast<const __half2 *>(Ks + row * D + col);
          c0 = q17_code(__low2float(x), kmn[col], kr[col], qmax);
          c1 = q17_code(__high2float(x), kmn[col + 1], kr[col + 1], qmax);
        } else {
          int ch = 16 * m + g + 8 * (r & 1), t = tile * 16 + 2 * q + 8 * (r >> 1);
          c0 = q17_code(__half2float(Vs[t * D + ch]), vmn[t], vr[t], qmax);
          c1 = q17_code(__half2float(Vs[(t + 1) * D + ch]), vmn[t + 1], vr[t + 1], qmax);
        }
        acc |= (c0 << (bits * j)) | (c1 << (16 + bits * j));
      }
      wv[e4] = acc;
    }
    dst[u4] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  // ---- params (K then V) after the codes ----
  uint4 *pdst = reinterpret_cast<uint4 *>(rec + 2 * code_bytes);
  const uint4 *psrc = reinterpret_cast<const uint4 *>(params);
  for (int i = tid; i < (4 * D + 4 * S) / 16; i += QT) pdst[i] = psrc[i];
}

template <int D, int S>
static size_t quant_smem() {
  return (size_t)2 * S * D * 2 + (2 * D + 2 * S) * 4 + 2 * QT * 4 + 4 * D + 4 * S;
}

template <int D, int S>
static cudaError_t launch_quant_t(const QuantArgs &a, int max_slots, cudaStream_t st) {
  size_t smem = quant_smem<D, S>();
  cudaError_t e = cudaFuncSetAttribute(k_quant<D, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(max_slots, a.H, a.B);
  k_quant<D, S><<<grid, QT, smem, st>>>(a);
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
  int ms = perm_stride;
#define WQ_Q(DD, SS) \
  if (d == DD && S == SS) return launch_quant_t<DD, SS>(a, ms, st);
  WQ_Q(64, 16) WQ_Q(64, 32) WQ_Q(64, 64) WQ_Q(64, 128)
  WQ_Q(128, 16) WQ_Q(128, 32) WQ_Q(128, 64) WQ_Q(128, 128)
#undef WQ_Q
  return cudaErrorInvalidValue;
}

}  // namespace wq
