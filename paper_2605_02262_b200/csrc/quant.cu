// quant.cu -- wq_layer_layout and wq_reorder_quantize_pack (Alg.2 prefill
// branch P:420-446, Eq.14-16, group = window P:508, readings Q17-Q22).
//
// Persistent teams of 4 warps.  A window's fp16 K and V rows are pulled into shared
// memory by tensor-map TMA copies (128-byte swizzled boxes), per-channel K and per-token
// V (min, max) are reduced with
// fp16x2 min/max, the fp32 quantizer contract (Q17) runs per element with explicit
// round-to-nearest intrinsics (no FMA contraction), and the record is written in
// D-1 fragment order with 16-byte stores at the window's REORDERED slot (so the
// reorder of Alg.2 is an address remap, not a copy).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {

// offs[b*H + h] of one layer from seg_off_l[B][5]; one thread per request, then a
// serial prefix (B <= 4096) by thread 0 -- tiny.
__global__ void k_layer_layout(const int32_t *__restrict__ seg_off, int B, int H, int d, int S, int gran,
                               int64_t *__restrict__ offs) {
  extern __shared__ int64_t img[];
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int32_t *so = seg_off + 5 * b;
    int64_t t = 0;
    for (int k = 0; k < 4; k++) t += (int64_t)(so[k + 1] - so[k]) * record_bytes(class_bits(k), d, S, gran);
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

struct QuantArgs {
  const __half *k, *v;
  int64_t sb, sh, st;     // strides in elements (b, h, t); channel stride 1
  int vis_off;
  int B, H, d, S, M;
  const int32_t *perm;
  int perm_stride;
  const int32_t *seg_off;
  const int64_t *offs;
  uint8_t *packed;
};

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
// Q17 code via the float magic, left as big = 0x4B400000 + code: fl(fl(x - mn) * r) lies
// in [0, q_max + 2^-21] (s = RoundUp(range / q_max) >= range / q_max), so the clamp of
// Q17 never binds and adding 1.5*2^23 rounds it to nearest-even into the low bits.
WQ_DEV uint32_t q17_big(float x, float mn, float r) {
  return __float_as_uint(__fadd_rn(__fmul_rn(__fsub_rn(x, mn), r), 12582912.0f));
}
// Packing word = sum_j big_j * 2^(sh_j) + BIAS (mod 2^32): the BIAS cancels the
// 0x4B400000 of every big, one IMAD per code.
template <int BITS>
struct PackBias {
  static constexpr uint32_t value() {
    uint32_t b = 0;
    for (int j = 0; j < 16 / BITS; j++) b += (0x4B400000u << (BITS * j)) + (0x4B400000u << (16 + BITS * j));
    return 0u - b;
  }
};

// Q17 scale of a group: s = max(RoundUp_fp16(fl(mx - mn) / qmax), 2^-24)
WQ_DEV __half q17_scale(float mn, float mx, float qmaxf) {
  __half s16 = __float2half_ru(__fdiv_rn(__fsub_rn(mx, mn), qmaxf));
  if (__half2float(s16) < 5.9604644775390625e-08f) s16 = __ushort_as_half(0x0001);
  return s16;
}

#ifndef WQ_Q_SLEEP
#define WQ_Q_SLEEP 0           // ns of back-off between mbarrier polls (0: spin)
#endif
// waiting warps back off so the warps that compute get the issue slots
WQ_DEV void qwait(uint64_t *b, uint32_t parity) {
  if (WQ_Q_SLEEP > 0) mbar_wait_sleep(b, parity, WQ_Q_SLEEP);
  else mbar_wait(b, parity);
}

// ---------------------------------------------------------------------------------
// k_quant: persistent.  A CTA runs TEAMS teams of 4 warps; a team owns NSL window slots
// in shared memory and quantizes windows gt, gt + nteams, ... of the flattened (request,
// kv head, slot) space.  A window's K and V rows land by tensor-map TMA copies
// (cp.async.bulk.tensor, one box of S tokens x 64 channels per 128-byte row, 128-byte
// swizzle: 16-byte chunk j of token row r sits at chunk j ^ (r mod 8)), so the fragment-
// order reads below are bank-conflict free straight from the landed tile -- no re-layout
// buffer.  A window's work splits into independent warp tasks -- the two channel halves of
// K (per-channel parameters need only their channels) and the 16-token tiles of V
// (per-token parameters) -- so no CTA barrier is ever needed: the slot is released
// through an mbarrier once the team's 4 warps are done with it.
// ---------------------------------------------------------------------------------
// what a team slot holds, written by the issuing lane with the copy (so the consumer
// warps never wait on the metadata loads): record offset and width, bits = 0 if empty
struct WinDesc {
  int64_t roff;
  int bits, pad;
};

template <int D, int S>
struct QuantGeo {
  static constexpr int KH = D / 64;                     // 64-channel boxes per K (and V) window
  static constexpr int BOX = S * 128;                   // bytes of one box: S token rows x 128 B
  static constexpr int WIN = 2 * KH * BOX;              // K boxes, then V boxes (= 4*S*D)
  static constexpr int SCR = (D > S ? D : S) * 8;       // float2 params scratch per warp
#ifndef WQ_Q_NSL
#define WQ_Q_NSL 0                                      // 0: by window size (below)
#endif
  // window slots per team: two for S <= 32, one for S >= 64 (32-64 KB windows), and up to
  // five teams: more warps to hide the latencies of an issue-bound kernel beat deeper
  // per-team buffering (A/B round 2, tools/quant_ab.py, vs 3-4 slots x 4 teams: C5 117.4 ->
  // 110.8 us, C4 S=32 418 -> 379, S=16 639 -> 538, S=64 509 -> 467, S=128 unchanged)
  static constexpr int NSL0 = S >= 64 ? 1 : 2;
  static constexpr int NSL = WQ_Q_NSL > 0 ? WQ_Q_NSL : NSL0;
  static constexpr int PER_TEAM = ((NSL * WIN + 4 * SCR) + 1023) / 1024 * 1024;   // slots 1024-B aligned
  static constexpr int T0 = (216 * 1024) / PER_TEAM;
#ifndef WQ_Q_TMAX
#define WQ_Q_TMAX 5                                     // most teams (4 warps each) per CTA
#endif
  static constexpr int TEAMS = T0 > WQ_Q_TMAX ? WQ_Q_TMAX : (T0 < 1 ? 1 : T0);
  static constexpr int NT = S / 16 + 2;                 // tasks per window: 2 K halves + S/16 V tiles
  static constexpr size_t bar_off = (size_t)TEAMS * PER_TEAM;
  static constexpr size_t desc_off = bar_off + TEAMS * 2 * NSL * 8;   // [TEAMS][NSL] WinDesc
  static constexpr size_t total = desc_off + TEAMS * NSL * 16;
};

// byte offset of (token row, byte b of the 64-channel box row) in a 128-byte-swizzled box
WQ_DEV uint32_t swz(int row, int b) { return (uint32_t)(row * 128 + ((((b >> 4) ^ row) & 7) << 4) + (b & 15)); }
// the 4 bytes of channels (c, c+1) of token row t of a window (boxes of 64 channels)
WQ_DEV uint32_t pair_at(const uint8_t *boxes, int t, int c, int box_bytes) {
  return lds32(boxes + (c >> 6) * box_bytes + swz(t, 2 * (c & 63)));
}
WQ_DEV uint32_t half_at(const uint8_t *boxes, int t, int c, int box_bytes) {
  return *reinterpret_cast<const uint16_t *>(boxes + (c >> 6) * box_bytes + swz(t, 2 * (c & 63)));
}

// K channel half hf (channels [hf*D/2, (hf+1)*D/2)) of a window: per-channel min/max
// over the S rows, parameters, then codes tile by tile (the fragment lane's words whose
// channels fall in this half).
template <int D, int S, int BITS>
WQ_DEV void quant_k_half(const uint8_t *kbox, float2 *kp, uint8_t *rec, int hf, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr float QMAX = (float)((1 << BITS) - 1);
  constexpr int PPW = 16 / BITS;
  constexpr int CW = D * BITS / 64;                     // chunk words per lane per tile
  constexpr int TILE = 2 * D * BITS;                    // bytes per 16-token tile
  constexpr int KBYTES = S * D * BITS / 8;
  constexpr int HP = D / 4;                             // channel pairs per half
  // (1) min/max (IEEE minimum/maximum, Q17): lane = channel pair, rows from the landed box
  if (lane < HP) {
    const int cp = hf * HP + lane;
    __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
    // channel pair cp: box cp/32, byte 4*(cp%32) = chunk c0, word cp%4; row t at t*128 with
    // chunk c0 ^ (t mod 8) (the XOR term is a constant of each unrolled row)
    const uint8_t *cb = kbox + (cp >> 5) * QG::BOX + 4 * (cp & 3);
    const int c0 = (cp & 31) >> 2;
    int xo[8];
#pragma unroll
    for (int u = 0; u < 8; u++) xo[u] = u * 128 + ((c0 ^ u) << 4);
#pragma unroll 1
    for (int t0 = 0; t0 < S; t0 += 8) {
      const uint8_t *rb = cb + t0 * 128;
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const __half2 x = u2h(lds32(rb + xo[u]));
        mn2 = __hmin2(mn2, x);
        mx2 = __hmax2(mx2, x);
      }
    }
    const float mn0 = __low2float(mn2), mn1 = __high2float(mn2);
    const __half s0 = q17_scale(mn0, __low2float(mx2), QMAX), s1 = q17_scale(mn1, __high2float(mx2), QMAX);
    kp[2 * cp] = make_float2(mn0, __frcp_rn(__half2float(s0)));
    kp[2 * cp + 1] = make_float2(mn1, __frcp_rn(__half2float(s1)));
    // D-1 K group (q, m) = {mn01, s01, mn89, s89}: this pair fills one half of it
    const int m = cp >> 3, j = cp & 7, q = j & 3, hh = j >> 2;
    uint2 pv;
    pv.x = (uint32_t)__half_as_ushort(__low2half(mn2)) | ((uint32_t)__half_as_ushort(__high2half(mn2)) << 16);
    pv.y = (uint32_t)__half_as_ushort(s0) | ((uint32_t)__half_as_ushort(s1) << 16);
    *reinterpret_cast<uint2 *>(rec + 2 * KBYTES + (4 * m + q) * 16 + hh * 8) = pv;
  }
  __syncwarp();
  // (2) codes: words of fragment lane L = lane whose pairs lie in this channel half
  //     (pair P -> m = P/4; m < D/32 is half 0).  WH words per tile per half.
  constexpr int WH = CW / 2 > 0 ? CW / 2 : 1;          // CW >= 2 always (d >= 64, b >= 2)
  const int g = lane >> 2, q = lane & 3;
  // row mod 8 = g for every code word of the lane: the swizzle term of chunk cc is gx[cc]
  int gx[8];
#pragma unroll
  for (int cc = 0; cc < 8; cc++) gx[cc] = (cc ^ g) << 4;
  const uint8_t *lb = kbox + g * 128 + 4 * q;
#pragma unroll 1
  for (int tile = 0; tile < S / 16; tile++) {
    const uint8_t *tb0 = lb + tile * 16 * 128;
    uint32_t wv[WH];
#pragma unroll
    for (int e = 0; e < WH; e++) {
      const int wl = hf * WH + e;
      uint32_t acc = PackBias<BITS>::value();
#pragma unroll
      for (int j = 0; j < PPW; j++) {
        const int P = wl * PPW + j, m = P >> 2, r = P & 3;
        const int col = 16 * m + 8 * (r >> 1) + 2 * q;
        // row = tile*16 + g + 8(r&1) (row mod 8 = g); byte 2*(col%64) = chunk cc, word q
        const int cc = (2 * m + (r >> 1)) & 7;
        const float2 x = __half22float2(u2h(lds32(tb0 + (m >> 2) * QG::BOX + 8 * (r & 1) * 128 + gx[cc])));
        const float4 pr = *reinterpret_cast<const float4 *>(kp + col);
        acc += q17_big(x.x, pr.x, pr.y) * (1u << (BITS * j));
        acc += q17_big(x.y, pr.z, pr.w) * (1u << (16 + BITS * j));
      }
      wv[e] = acc;
    }
    // D-1 chunk of lane L: words 4*gi + e at byte gi*512 + L*16 + 4e (chunks >= 16 B) or
    // L*8 + 4e (8-byte chunks); this half owns words [hf*WH, (hf+1)*WH)
    uint8_t *tb = rec + tile * TILE;
    if constexpr (CW >= 4) {
#pragma unroll
      for (int e0 = 0; e0 < WH; e0 += (WH >= 4 ? 4 : 2)) {
        const int wl = hf * WH + e0;
        uint8_t *dst = tb + (wl >> 2) * 512 + lane * 16 + 4 * (wl & 3);
        if constexpr (WH >= 4) *reinterpret_cast<uint4 *>(dst) = make_uint4(wv[e0], wv[e0 + 1], wv[e0 + 2], wv[e0 + 3]);
        else *reinterpret_cast<uint2 *>(dst) = make_uint2(wv[e0], wv[e0 + 1]);
      }
    } else {
      *reinterpret_cast<uint32_t *>(tb + lane * 8 + 4 * hf) = wv[0];
    }
  }
}

// V tile vt (tokens [16vt, 16vt+16)): per-token min/max over D channels, parameters,
// codes of the fragment lane L = lane for this tile.
template <int D, int S, int BITS>
WQ_DEV void quant_v_tile(const uint8_t *vbox, float2 *vp, uint8_t *rec, int vt, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr float QMAX = (float)((1 << BITS) - 1);
  constexpr int PPW = 16 / BITS;
  constexpr int CW = D * BITS / 64;
  constexpr int TILE = 2 * D * BITS;
  constexpr int KBYTES = S * D * BITS / 8;
  // (1) min/max: two lanes per token (each half of the channels), combined by a shuffle;
  // the pair order is rotated per lane so rows t and t + 8 and the two halves hit
  // different bank groups
  {
    const int t = lane >> 1, hc = lane & 1;
    // the lane's half of token row t, 16-byte chunk by chunk; the second half starts 4
    // chunks later so a phase's 8 lanes read 8 different bank groups
    constexpr int NC = D / 16;                          // 16-byte chunks per half (8 channels each)
    __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
    const int row = vt * 16 + t;
#pragma unroll
    for (int i = 0; i < NC; i++) {
      const int c = hc * (D / 2) / 8 + ((i + 4 * hc) % NC);          // chunk of 8 channels
      const uint4 v = lds128(vbox + (c >> 3) * QG::BOX + row * 128 + ((((c & 7) ^ row) & 7) << 4));
      const __half2 x0 = u2h(v.x), x1 = u2h(v.y), x2 = u2h(v.z), x3 = u2h(v.w);
      mn2 = __hmin2(mn2, __hmin2(__hmin2(x0, x1), __hmin2(x2, x3)));
      mx2 = __hmax2(mx2, __hmax2(__hmax2(x0, x1), __hmax2(x2, x3)));
    }
    __half mn = __hmin(__low2half(mn2), __high2half(mn2));
    __half mx = __hmax(__low2half(mx2), __high2half(mx2));
    mn = __hmin(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
    mx = __hmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    if (hc == 0) {
      const float mnf = __half2float(mn);
      const __half s16 = q17_scale(mnf, __half2float(mx), QMAX);
      vp[t] = make_float2(mnf, __frcp_rn(__half2float(s16)));
      // D-1 V group (i, q) = {s(t0), s(t0+1), s(t0+8), s(t0+9), mn(...)}, t0 = 16i + 2q
      const int qq = (t & 7) >> 1, hh = t >> 3, e = t & 1;
      __half *grp = reinterpret_cast<__half *>(rec + 2 * KBYTES + 4 * D + (4 * vt + qq) * 16);
      grp[2 * hh + e] = s16;
      grp[4 + 2 * hh + e] = mn;
    }
  }
  __syncwarp();
  const int g = lane >> 2, q = lane & 3;
  uint8_t *tb = rec + KBYTES + vt * TILE;
  constexpr int NG = CW >= 4 ? CW / 4 : 1;
  // tokens 2q + 8(r>>1) (+1): row mod 8 = 2q (2q + 1); swizzle terms of chunk cc
  int qx0[8], qx1[8];
#pragma unroll
  for (int cc = 0; cc < 8; cc++) { qx0[cc] = (cc ^ (2 * q)) << 4; qx1[cc] = 128 + ((cc ^ (2 * q + 1)) << 4); }
  const uint8_t *lb = vbox + (vt * 16 + 2 * q) * 128 + 2 * g;
#pragma unroll
  for (int gi = 0; gi < NG; gi++) {
    uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int e = 0; e < (CW >= 4 ? 4 : CW); e++) {
      const int wl = 4 * gi + e;
      uint32_t acc = PackBias<BITS>::value();
#pragma unroll
      for (int j = 0; j < PPW; j++) {
        const int P = wl * PPW + j, m = P >> 2, r = P & 3;
        const int t = 2 * q + 8 * (r >> 1);
        const float4 pr = *reinterpret_cast<const float4 *>(vp + t);      // {mn, r} of t, t+1
        // channel 16m + g + 8(r&1): box m/4, chunk cc, byte 2g; tokens t, t+1 (row mod 8 = 2q, 2q+1)
        const int cc = (2 * m + (r & 1)) & 7;
        const uint8_t *rb = lb + (m >> 2) * QG::BOX + 8 * (r >> 1) * 128;
        const float x0 = __half2float(*reinterpret_cast<const __half *>(rb + qx0[cc]));
        const float x1 = __half2float(*reinterpret_cast<const __half *>(rb + qx1[cc]));
        acc += q17_big(x0, pr.x, pr.y) * (1u << (BITS * j));
        acc += q17_big(x1, pr.z, pr.w) * (1u << (16 + BITS * j));
      }
      wv[e] = acc;
    }
    if constexpr (CW >= 4)
      *reinterpret_cast<uint4 *>(tb + gi * 512 + lane * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    else
      *reinterpret_cast<uint2 *>(tb + lane * 8) = make_uint2(wv[0], wv[1]);
  }
}

// Paper-literal groups (reading Q37): the IEEE minimum / maximum of ALL S x d values
// of one tensor of the window (its d/64 boxes, any order: the set of values is the window),
// by one warp: 16-byte chunks lane-strided (conflict-free), then a shuffle reduction.
template <int D, int S>
WQ_DEV void group_minmax(const uint8_t *boxes, int lane, __half &mn, __half &mx) {
  using QG = QuantGeo<D, S>;
  constexpr int NCH = QG::KH * QG::BOX / 16;
  __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
#pragma unroll 4
  for (int i = lane; i < NCH; i += 32) {
    const uint4 v = lds128(boxes + 16 * i);
    const __half2 x0 = u2h(v.x), x1 = u2h(v.y), x2 = u2h(v.z), x3 = u2h(v.w);
    mn2 = __hmin2(mn2, __hmin2(__hmin2(x0, x1), __hmin2(x2, x3)));
    mx2 = __hmax2(mx2, __hmax2(__hmax2(x0, x1), __hmax2(x2, x3)));
  }
  mn = __hmin(__low2half(mn2), __high2half(mn2));
  mx = __hmax(__low2half(mx2), __high2half(mx2));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    mn = __hmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = __hmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
}

// K channel half hf of a window under group granularity: the window's single (s, mn)
// (computed by every K task from the whole window), codes of this half
template <int D, int S, int BITS>
WQ_DEV void quant_k_half_grp(const uint8_t *kbox, uint8_t *rec, int hf, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr float QMAX = (float)((1 << BITS) - 1);
  constexpr int PPW = 16 / BITS;
  constexpr int CW = D * BITS / 64;
  constexpr int TILE = 2 * D * BITS;
  constexpr int KBYTES = S * D * BITS / 8;
  __half mnh, mxh;
  group_minmax<D, S>(kbox, lane, mnh, mxh);
  const float mn = __half2float(mnh);
  const __half s16 = q17_scale(mn, __half2float(mxh), QMAX);
  const float r = __frcp_rn(__half2float(s16));
  if (hf == 0 && lane == 0) {
    // the 16-byte block {mn_K, s_K, mn_V, s_V, 0, 0, 0, 0}: K half 0 writes K's pair and the zeros
    const uint32_t kp = (uint32_t)__half_as_ushort(mnh) | ((uint32_t)__half_as_ushort(s16) << 16);
    *reinterpret_cast<uint32_t *>(rec + 2 * KBYTES) = kp;
    *reinterpret_cast<uint2 *>(rec + 2 * KBYTES + 8) = make_uint2(0u, 0u);
  }
  constexpr int WH = CW / 2 > 0 ? CW / 2 : 1;
  const int g = lane >> 2, q = lane & 3;
  int gx[8];
#pragma unroll
  for (int cc = 0; cc < 8; cc++) gx[cc] = (cc ^ g) << 4;
  const uint8_t *lb = kbox + g * 128 + 4 * q;
#pragma unroll 1
  for (int tile = 0; tile < S / 16; tile++) {
    const uint8_t *tb0 = lb + tile * 16 * 128;
    uint32_t wv[WH];
#pragma unroll
    for (int e = 0; e < WH; e++) {
      const int wl = hf * WH + e;
      uint32_t acc = PackBias<BITS>::value();
#pragma unroll
      for (int j = 0; j < PPW; j++) {
        const int P = wl * PPW + j, m = P >> 2, rr = P & 3;
        const int cc = (2 * m + (rr >> 1)) & 7;
        const float2 x = __half22float2(u2h(lds32(tb0 + (m >> 2) * QG::BOX + 8 * (rr & 1) * 128 + gx[cc])));
        acc += q17_big(x.x, mn, r) * (1u << (BITS * j));
        acc += q17_big(x.y, mn, r) * (1u << (16 + BITS * j));
      }
      wv[e] = acc;
    }
    uint8_t *tb = rec + tile * TILE;
    if constexpr (CW >= 4) {
#pragma unroll
      for (int e0 = 0; e0 < WH; e0 += (WH >= 4 ? 4 : 2)) {
        const int wl = hf * WH + e0;
        uint8_t *dst = tb + (wl >> 2) * 512 + lane * 16 + 4 * (wl & 3);
        if constexpr (WH >= 4) *reinterpret_cast<uint4 *>(dst) = make_uint4(wv[e0], wv[e0 + 1], wv[e0 + 2], wv[e0 + 3]);
        else *reinterpret_cast<uint2 *>(dst) = make_uint2(wv[e0], wv[e0 + 1]);
      }
    } else {
      *reinterpret_cast<uint32_t *>(tb + lane * 8 + 4 * hf) = wv[0];
    }
  }
}

// V tile vt under group granularity: the window's single (s, mn) for V, codes of this tile
template <int D, int S, int BITS>
WQ_DEV void quant_v_tile_grp(const uint8_t *vbox, uint8_t *rec, int vt, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr float QMAX = (float)((1 << BITS) - 1);
  constexpr int PPW = 16 / BITS;
  constexpr int CW = D * BITS / 64;
  constexpr int TILE = 2 * D * BITS;
  constexpr int KBYTES = S * D * BITS / 8;
  __half mnh, mxh;
  group_minmax<D, S>(vbox, lane, mnh, mxh);
  const float mn = __half2float(mnh);
  const __half s16 = q17_scale(mn, __half2float(mxh), QMAX);
  const float r = __frcp_rn(__half2float(s16));
  if (vt == 0 && lane == 0)
    *reinterpret_cast<uint32_t *>(rec + 2 * KBYTES + 4) =
        (uint32_t)__half_as_ushort(mnh) | ((uint32_t)__half_as_ushort(s16) << 16);
  const int g = lane >> 2, q = lane & 3;
  uint8_t *tb = rec + KBYTES + vt * TILE;
  constexpr int NG = CW >= 4 ? CW / 4 : 1;
  int qx0[8], qx1[8];
#pragma unroll
  for (int cc = 0; cc < 8; cc++) { qx0[cc] = (cc ^ (2 * q)) << 4; qx1[cc] = 128 + ((cc ^ (2 * q + 1)) << 4); }
  const uint8_t *lb = vbox + (vt * 16 + 2 * q) * 128 + 2 * g;
#pragma unroll
  for (int gi = 0; gi < NG; gi++) {
    uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int e = 0; e < (CW >= 4 ? 4 : CW); e++) {
      const int wl = 4 * gi + e;
      uint32_t acc = PackBias<BITS>::value();
#pragma unroll
      for (int j = 0; j < PPW; j++) {
        const int P = wl * PPW + j, m = P >> 2, rr = P & 3;
        const int cc = (2 * m + (rr & 1)) & 7;
        const uint8_t *rb = lb + (m >> 2) * QG::BOX + 8 * (rr >> 1) * 128;
        const float x0 = __half2float(*reinterpret_cast<const __half *>(rb + qx0[cc]));
        const float x1 = __half2float(*reinterpret_cast<const __half *>(rb + qx1[cc]));
        acc += q17_big(x0, mn, r) * (1u << (BITS * j));
        acc += q17_big(x1, mn, r) * (1u << (16 + BITS * j));
      }
      wv[e] = acc;
    }
    if constexpr (CW >= 4)
      *reinterpret_cast<uint4 *>(tb + gi * 512 + lane * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    else
      *reinterpret_cast<uint2 *>(tb + lane * 8) = make_uint2(wv[0], wv[1]);
  }
}

// FP16 window, task tk: K halves / V tiles copied into fragment order.
template <int D, int S>
WQ_DEV void copy_task_fp16(const uint8_t *kbox, const uint8_t *vbox, uint8_t *rec, int tk, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr int TILE = 2 * D * 16;
  const int g = lane >> 2, q = lane & 3;
  if (tk < 2) {
    // K half tk: groups gi (4 words, m = gi) with 16m in this half, every tile
#pragma unroll 1
    for (int tile = 0; tile < S / 16; tile++) {
      for (int gi = tk * (D / 32); gi < (tk + 1) * (D / 32); gi++) {
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int P = 4 * gi + e, m = P >> 2, r = P & 3;
          const int row = tile * 16 + g + 8 * (r & 1), col = 16 * m + 2 * q + 8 * (r >> 1);
          wv[e] = pair_at(kbox, row, col, QG::BOX);
        }
        *reinterpret_cast<uint4 *>(rec + tile * TILE + gi * 512 + lane * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
  } else {
    const int vt = tk - 2;
    for (int gi = 0; gi < D / 16; gi++) {
      uint32_t wv[4];
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int P = 4 * gi + e, m = P >> 2, r = P & 3;
        const int ch = 16 * m + g + 8 * (r & 1), t = 2 * q + 8 * (r >> 1);
        const uint32_t lo = half_at(vbox, vt * 16 + t, ch, QG::BOX);
        const uint32_t hi = half_at(vbox, vt * 16 + t + 1, ch, QG::BOX);
        wv[e] = lo | (hi << 16);
      }
      *reinterpret_cast<uint4 *>(rec + S * D * 2 + vt * TILE + gi * 512 + lane * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
  }
}

// 4-D tensor-map TMA load of one box into shared memory, completes on mbarrier b
WQ_DEV void tma_load_4d(void *dst, const CUtensorMap *tm, int c0, int c1, int c2, int c3, uint64_t *b,
                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(b)), "l"(policy)
      : "memory");
}

template <int D, int S, bool GRP>
__global__ void __launch_bounds__(QuantGeo<D, S>::TEAMS * 128, 1)
    k_quant(QuantArgs a, const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv) {
  constexpr int GR = GRP ? 1 : 0;
  using QG = QuantGeo<D, S>;
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp >> 2, tw = warp & 3;
  uint8_t *tbase = sm + (size_t)team * QG::PER_TEAM;
  constexpr int NSL = QG::NSL;
  float2 *scr = reinterpret_cast<float2 *>(tbase + NSL * QG::WIN + tw * QG::SCR);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + QG::bar_off) + team * 2 * NSL;   // [NSL] full, [NSL] empty
  uint64_t *empty = full + NSL;
  WinDesc *wdesc = reinterpret_cast<WinDesc *>(sm + QG::desc_off) + team * NSL;
  const int64_t nwin = (int64_t)a.B * a.H * a.perm_stride;
  const int64_t gt = (int64_t)blockIdx.x * QG::TEAMS + team, nt = (int64_t)gridDim.x * QG::TEAMS;
  if (tw == 0 && lane == 0) {
    for (int i = 0; i < NSL; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 4); }
    fence_mbar_init();
  }
  WQ_CHECK((smem_u32(sm) & 1023u) == 0u);        // 128-byte swizzle atoms need 1024-B aligned boxes
  __syncthreads();
  auto locate = [&](int64_t wi, int &b, int &h, int &slot) {
    slot = (int)(wi % a.perm_stride);
    const int64_t bh = wi / a.perm_stride;
    h = (int)(bh % a.H);
    b = (int)(bh / a.H);
  };
  // Window metadata (seg_off, perm, offs) of team window k, loaded by the issuing lane one
  // window AHEAD of its copy: the three loads are independent (issued together, before any
  // branch on their values) and complete while the warp quantizes, so the copy of a window
  // never waits on a global round trip (ncu r01: 75% long_sb on the issue path).
  struct Meta {
    int b, h, slot, w, so[5];
    int64_t base;
    bool valid;
  };
  auto fetch = [&](int64_t k, Meta &m) {
    const int64_t wi = gt + k * nt;
    m.valid = wi < nwin;
    if (!m.valid) return;
    locate(wi, m.b, m.h, m.slot);
    const int32_t *so = a.seg_off + 5 * m.b;
#pragma unroll
    for (int i = 0; i < 5; i++) m.so[i] = __ldg(so + i);
    m.w = __ldg(a.perm + (int64_t)m.b * a.perm_stride + m.slot);
    m.base = __ldg(a.offs + (int64_t)m.b * a.H + m.h);
  };
  // team window k -> slot k % NSL (issued by the team's warp 0, lane 0)
  auto issue = [&](int64_t k, const Meta &m) {
    if (!m.valid) return;
    const int sl = (int)(k % NSL);
    qwait(&empty[sl], (uint32_t)((k / NSL) & 1) ^ 1u);
    const int b = m.b, h = m.h, slot = m.slot;
    if (slot >= m.so[4]) {
      wdesc[sl].bits = 0;
      mbar_arrive(&full[sl]);
      return;
    }
    const int w = m.w;
    WQ_CHECK(w >= 0 && (int64_t)(w + 1) * S <= a.M && slot < a.perm_stride);
    // class of the slot and its record offset (branch-free: no local arrays)
    const int cls = (slot >= m.so[1]) + (slot >= m.so[2]) + (slot >= m.so[3]);
    const int bits = class_bits(cls);
    int64_t roff = m.base;
#pragma unroll
    for (int kk = 0; kk < 3; kk++)
      if (kk < cls) roff += (int64_t)(m.so[kk + 1] - m.so[kk]) * record_bytes(class_bits(kk), D, S, GR);
    const int sbase = cls == 0 ? m.so[0] : cls == 1 ? m.so[1] : cls == 2 ? m.so[2] : m.so[3];
    roff += (int64_t)(slot - sbase) * record_bytes(bits, D, S, GR);
    WQ_CHECK(roff >= a.offs[(int64_t)b * a.H + h] &&
             roff + record_bytes(bits, D, S, GR) <= a.offs[(int64_t)b * a.H + h + 1]);
    wdesc[sl].roff = roff;
    wdesc[sl].bits = bits;
    uint8_t *dst = tbase + (size_t)sl * QG::WIN;
    const uint64_t pol = policy_evict_first();
    mbar_arrive_expect_tx(&full[sl], (uint32_t)QG::WIN);
    const int t0 = a.vis_off + w * S;
    // a window = d/64 boxes of [S tokens][64 channels] per tensor (rows of 128 B)
#pragma unroll
    for (int hb = 0; hb < QG::KH; hb++) {
      tma_load_4d(dst + hb * QG::BOX, &tmk, 64 * hb, t0, h, b, &full[sl], pol);
      tma_load_4d(dst + (QG::KH + hb) * QG::BOX, &tmv, 64 * hb, t0, h, b, &full[sl], pol);
    }
  };
  const bool issuer = tw == 0 && lane == 0;
  Meta nm;                                        // metadata of the next window to issue
  if (issuer) {
    Meta m0;
    for (int i = 0; i < NSL - 1; i++) {
      fetch(i, m0);
      issue(i, m0);
    }
    fetch(NSL - 1, nm);
  }
  for (int64_t k = 0;; k++) {
    const int64_t wi = gt + k * nt;
    if (wi >= nwin) break;
    if (issuer) {                                // the slot released after window k-1
      issue(k + NSL - 1, nm);
      fetch(k + NSL, nm);                          // in flight while this warp quantizes
    }
    const int sl = (int)(k % NSL);
    qwait(&full[sl], (uint32_t)((k / NSL) & 1));
    const int bits = wdesc[sl].bits;
    if (bits) {
      uint8_t *rec = a.packed + wdesc[sl].roff;
      const uint8_t *kbox = tbase + (size_t)sl * QG::WIN, *vbox = kbox + QG::KH * QG::BOX;
      // one task loop per record kind: with the kind tested inside a single loop, ptxas
      // 12.9 mis-allocated k_quant<128, S >= 64, true> (a K task clobbered the thread-index
      // register the next FP16 V task of the same warp reused: odd-token halves of V tiles
      // 2-3 read from wrong rows; tests/test_gpu_group.py caught it)
      if (bits == 16) {
        for (int tk = tw; tk < QG::NT; tk += 4) copy_task_fp16<D, S>(kbox, vbox, rec, tk, lane);
      } else if constexpr (GRP) {
        for (int tk = tw; tk < QG::NT; tk += 4) {
          if (tk < 2) {
            if (bits == 2) quant_k_half_grp<D, S, 2>(kbox, rec, tk, lane);
            else if (bits == 4) quant_k_half_grp<D, S, 4>(kbox, rec, tk, lane);
            else quant_k_half_grp<D, S, 8>(kbox, rec, tk, lane);
          } else {
            if (bits == 2) quant_v_tile_grp<D, S, 2>(vbox, rec, tk - 2, lane);
            else if (bits == 4) quant_v_tile_grp<D, S, 4>(vbox, rec, tk - 2, lane);
            else quant_v_tile_grp<D, S, 8>(vbox, rec, tk - 2, lane);
          }
        }
      } else for (int tk = tw; tk < QG::NT; tk += 4) {
        if (tk < 2) {
          if (bits == 2) quant_k_half<D, S, 2>(kbox, scr, rec, tk, lane);
          else if (bits == 4) quant_k_half<D, S, 4>(kbox, scr, rec, tk, lane);
          else quant_k_half<D, S, 8>(kbox, scr, rec, tk, lane);
        } else {
          if (bits == 2) quant_v_tile<D, S, 2>(vbox, scr, rec, tk - 2, lane);
          else if (bits == 4) quant_v_tile<D, S, 4>(vbox, scr, rec, tk - 2, lane);
          else quant_v_tile<D, S, 8>(vbox, scr, rec, tk - 2, lane);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sl]);       // this warp is done with the slot
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
// [B][H][T][d] fp16 (strides in elements) as a 4-D tensor, boxes of 64 channels x S tokens
// (rows of 128 B), 128-byte swizzle
static bool encode_kv_map(CUtensorMap *tm, const __half *base, int B, int H, int T, int d, int S,
                          int64_t sb, int64_t sh, int64_t st) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t gdim[4] = {(cuuint64_t)d, (cuuint64_t)T, (cuuint64_t)H, (cuuint64_t)B};
  const cuuint64_t gstr[3] = {(cuuint64_t)st * 2, (cuuint64_t)sh * 2, (cuuint64_t)sb * 2};
  const cuuint32_t box[4] = {64, (cuuint32_t)S, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half *>(base), gdim, gstr, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, int S, bool GRP>
static cudaError_t launch_quant_t(const QuantArgs &a, cudaStream_t st) {
  using QG = QuantGeo<D, S>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_quant<D, S, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)QG::total);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t nwin = (int64_t)a.B * a.H * a.perm_stride;
  int64_t grid = device_sm_count();
  const int64_t need = (nwin + QG::TEAMS - 1) / QG::TEAMS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  // tokens read: [vis_off, vis_off + M)
  const int T = a.vis_off + a.M;
  CUtensorMap tmk, tmv;
  if (!encode_kv_map(&tmk, a.k, a.B, a.H, T, D, S, a.sb, a.sh, a.st) ||
      !encode_kv_map(&tmv, a.v, a.B, a.H, T, D, S, a.sb, a.sh, a.st))
    return cudaErrorInvalidValue;
  k_quant<D, S, GRP><<<(unsigned)grid, QG::TEAMS * 128, QG::total, st>>>(a, tmk, tmv);
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
    for (int i = threadIdx.x; i < cnt[k]; i += blockDim.x) {
      WQ_CHECK(start[k] + i < W && lo[k] + i < so[k + 1]);
      perm_r[(int64_t)b * W + start[k] + i] = perm[(int64_t)b * W + lo[k] + i];
    }
  if (threadIdx.x < 5) seg_r[5 * b + threadIdx.x] = start[threadIdx.x];
}


cudaError_t launch_shard_slots(const int32_t *perm, const int32_t *seg, int B, int W, int G, int r,
                               int32_t *perm_r, int32_t *seg_r, cudaStream_t st) {
  k_shard_slots<<<B, 256, 0, st>>>(perm, seg, W, G, r, perm_r, seg_r);
  return cudaGetLastError();
}

cudaError_t launch_layer_layout(const int32_t *seg_off, int B, int H, int d, int S, int gran, int64_t *offs,
                                cudaStream_t st) {
  k_layer_layout<<<1, 256, (size_t)B * sizeof(int64_t), st>>>(seg_off, B, H, d, S, gran, offs);
  return cudaGetLastError();
}

cudaError_t launch_quant(const __half *k, const __half *v, const int64_t strides[3], int vis_off,
                         int B, int H, int d, int S, int M, const int32_t *perm, int perm_stride,
                         const int32_t *seg_off, const int64_t *offs, uint8_t *packed, int gran,
                         cudaStream_t st) {
  QuantArgs a{k, v, strides[0], strides[1], strides[2], vis_off, B, H, d, S, M, perm, perm_stride,
              seg_off, offs, packed};
#define WQ_Q(DD, SS) \
  if (d == DD && S == SS) return gran ? launch_quant_t<DD, SS, true>(a, st) : launch_quant_t<DD, SS, false>(a, st);
  WQ_Q(64, 16) WQ_Q(64, 32) WQ_Q(64, 64) WQ_Q(64, 128)
  WQ_Q(128, 16) WQ_Q(128, 32) WQ_Q(128, 64) WQ_Q(128, 128)
#undef WQ_Q
  return cudaErrorInvalidValue;
}

}  // namespace wq
