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
// k_quant: persistent.  A CTA runs TEAMS teams of 4 warps; a team owns two window
// slots in shared memory (double buffering) and quantizes windows gt, gt + nteams, ...
// of the flattened (request, kv head, slot) space.  A window's K and V rows land by
// two 1-D bulk copies (TMA engine); its work splits into independent warp tasks --
// the two channel halves of K (per-channel parameters) and the 16-token tiles of V
// (per-token parameters) -- so no CTA barrier is ever needed: the slot is released
// through an mbarrier once the team's 4 warps are done with it.  Fragment-order reads
// go through a per-warp work buffer with rows padded by 16 bytes (bank-conflict free).
// ---------------------------------------------------------------------------------
// what a team slot holds, written by the issuing lane with the copy (so the consumer
// warps never wait on the metadata loads): record offset and width, bits = 0 if empty
struct WinDesc {
  int64_t roff;
  int bits, pad;
};

template <int D, int S>
struct QuantGeo {
  static constexpr int WIN = 4 * S * D;                 // K + V rows of a window, as landed
  static constexpr int WRB = 2 * D + 16;                // padded row bytes, work buffer
  static constexpr int WORK = 16 * WRB;                 // one 16-row tile
  static constexpr int SCR = (D > S ? D : S) * 8;       // float2 params scratch per warp
#ifndef WQ_Q_NSL
#define WQ_Q_NSL 0                                      // 0: by window size (below)
#endif
  // window slots per team: double buffering pays while it leaves room for 4 teams; for
  // S >= 64 (32-64 KB windows) one slot per team and more teams per SM win (C4 shape:
  // S = 64 716 -> 583 us, S = 128 992 -> 662 us; S = 32 needs two: 493 vs 641 us)
  static constexpr int NSL = WQ_Q_NSL > 0 ? WQ_Q_NSL : (S >= 64 ? 1 : 2);
  static constexpr int PER_TEAM = NSL * WIN + 4 * (WORK + SCR);
  static constexpr int T0 = (216 * 1024) / PER_TEAM;
  static constexpr int TEAMS = T0 > 4 ? 4 : (T0 < 1 ? 1 : T0);
  static constexpr int NT = S / 16 + 2;                 // tasks per window: 2 K halves + S/16 V tiles
  static constexpr size_t bar_off = (size_t)TEAMS * PER_TEAM;
  static constexpr size_t desc_off = bar_off + TEAMS * 2 * NSL * 8;   // [TEAMS][NSL] WinDesc
  static constexpr size_t total = desc_off + TEAMS * NSL * 16;
};

// K channel half hf (channels [hf*D/2, (hf+1)*D/2)) of a window: per-channel min/max
// over the S rows, parameters, then codes tile by tile (the fragment lane's words whose
// channels fall in this half).
template <int D, int S, int BITS>
WQ_DEV void quant_k_half(const uint8_t *krows, uint8_t *work, float2 *kp, uint8_t *rec, int hf, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr int WRB = QG::WRB;
  constexpr float QMAX = (float)((1 << BITS) - 1);
  constexpr uint32_t MASK = (1u << BITS) - 1u;
  constexpr int PPW = 16 / BITS;
  constexpr int CW = D * BITS / 64;                     // chunk words per lane per tile
  constexpr int TILE = 2 * D * BITS;                    // bytes per 16-token tile
  constexpr int KBYTES = S * D * BITS / 8;
  constexpr int HP = D / 4;                             // channel pairs per half
  // (1) min/max: lane = channel pair (rows read straight from the landed copy)
  if (lane < HP) {
    const int cp = hf * HP + lane;
    __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
#pragma unroll 8
    for (int t = 0; t < S; t++) {
      const __half2 x = *reinterpret_cast<const __half2 *>(krows + t * 2 * D + 4 * cp);
      mn2 = __hmin2(mn2, x);
      mx2 = __hmax2(mx2, x);
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
    *reinterpret_cast<uint2 *>(rec + 2 * KBYTES + (q * (D / 16) + m) * 16 + hh * 8) = pv;
  }
  // (2) codes: words of fragment lane L = lane whose pairs lie in this channel half
  //     (pair P -> m = P/4; m < D/32 is half 0).  WH words per tile per half.
  constexpr int WH = CW / 2 > 0 ? CW / 2 : 1;          // CW >= 2 always (d >= 64, b >= 2)
  const int g = lane >> 2, q = lane & 3;
#pragma unroll 1
  for (int tile = 0; tile < S / 16; tile++) {
    // re-lay the tile's 16 half rows (D bytes each) into padded rows
    __syncwarp();
    {
      constexpr int CPR = D / 16;                       // 16-byte chunks per half row
#pragma unroll
      for (int i = lane; i < 16 * CPR; i += 32) {
        const int t = i / CPR, cc = i - t * CPR;
        *reinterpret_cast<uint4 *>(work + t * WRB + 16 * cc) =
            *reinterpret_cast<const uint4 *>(krows + (tile * 16 + t) * 2 * D + hf * D + 16 * cc);
      }
    }
    __syncwarp();
    uint32_t wv[WH];
#pragma unroll
    for (int e = 0; e < WH; e++) {
      const int wl = hf * WH + e;
      uint32_t acc = PackBias<BITS>::value();
#pragma unroll
      for (int j = 0; j < PPW; j++) {
        const int P = wl * PPW + j, m = P >> 2, r = P & 3;
        const int row = g + 8 * (r & 1), col = 16 * m + 8 * (r >> 1) + 2 * q;     // col in [hf*D/2, ...)
        const float2 x = __half22float2(*reinterpret_cast<const __half2 *>(work + row * WRB + 2 * (col - hf * D / 2)));
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
WQ_DEV void quant_v_tile(const uint8_t *vrows, uint8_t *work, float2 *vp, uint8_t *rec, int vt, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr int WRB = QG::WRB;
  constexpr float QMAX = (float)((1 << BITS) - 1);
  constexpr uint32_t MASK = (1u << BITS) - 1u;
  constexpr int PPW = 16 / BITS;
  constexpr int CW = D * BITS / 64;
  constexpr int TILE = 2 * D * BITS;
  constexpr int KBYTES = S * D * BITS / 8;
  // re-lay the tile's 16 rows into padded rows
  __syncwarp();
  {
    constexpr int CPR = 2 * D / 16;
#pragma unroll
    for (int i = lane; i < 16 * CPR; i += 32) {
      const int t = i / CPR, cc = i - t * CPR;
      *reinterpret_cast<uint4 *>(work + t * WRB + 16 * cc) = *reinterpret_cast<const uint4 *>(vrows + (vt * 16 + t) * 2 * D + 16 * cc);
    }
  }
  __syncwarp();
  // (1) min/max: two lanes per token (each half of the channels), combined by a shuffle
  {
    const int t = lane >> 1, hc = lane & 1;
    __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
#pragma unroll 8
    for (int i = 0; i < D / 4; i++) {
      const __half2 x = *reinterpret_cast<const __half2 *>(work + t * WRB + 2 * D / 2 * hc + 4 * i);
      mn2 = __hmin2(mn2, x);
      mx2 = __hmax2(mx2, x);
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
        const int ch = 16 * m + g + 8 * (r & 1), t = 2 * q + 8 * (r >> 1);
        const float4 pr = *reinterpret_cast<const float4 *>(vp + t);      // {mn, r} of t, t+1
        const float x0 = __half2float(*reinterpret_cast<const __half *>(work + t * WRB + 2 * ch));
        const float x1 = __half2float(*reinterpret_cast<const __half *>(work + (t + 1) * WRB + 2 * ch));
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

// FP16 window, task tk: K halves / V tiles copied into fragment order.
template <int D, int S>
WQ_DEV void copy_task_fp16(const uint8_t *krows, const uint8_t *vrows, uint8_t *work, uint8_t *rec, int tk, int lane) {
  using QG = QuantGeo<D, S>;
  constexpr int WRB = QG::WRB;
  constexpr int TILE = 2 * D * 16;
  const int g = lane >> 2, q = lane & 3;
  if (tk < 2) {
    // K half tk: groups gi (4 words, m = gi) with 16m in this half, every tile
#pragma unroll 1
    for (int tile = 0; tile < S / 16; tile++) {
      __syncwarp();
      for (int i = lane; i < 16 * (2 * D / 16); i += 32) {
        const int t = i / (2 * D / 16), cc = i - t * (2 * D / 16);
        *reinterpret_cast<uint4 *>(work + t * WRB + 16 * cc) = *reinterpret_cast<const uint4 *>(krows + (tile * 16 + t) * 2 * D + 16 * cc);
      }
      __syncwarp();
      for (int gi = tk * (D / 32); gi < (tk + 1) * (D / 32); gi++) {
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int P = 4 * gi + e, m = P >> 2, r = P & 3;
          const int row = g + 8 * (r & 1), col = 16 * m + 2 * q + 8 * (r >> 1);
          wv[e] = *reinterpret_cast<const uint32_t *>(work + row * WRB + 2 * col);
        }
        *reinterpret_cast<uint4 *>(rec + tile * TILE + gi * 512 + lane * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
  } else {
    const int vt = tk - 2;
    __syncwarp();
    for (int i = lane; i < 16 * (2 * D / 16); i += 32) {
      const int t = i / (2 * D / 16), cc = i - t * (2 * D / 16);
      *reinterpret_cast<uint4 *>(work + t * WRB + 16 * cc) = *reinterpret_cast<const uint4 *>(vrows + (vt * 16 + t) * 2 * D + 16 * cc);
    }
    __syncwarp();
    for (int gi = 0; gi < D / 16; gi++) {
      uint32_t wv[4];
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int P = 4 * gi + e, m = P >> 2, r = P & 3;
        const int ch = 16 * m + g + 8 * (r & 1), t = 2 * q + 8 * (r >> 1);
        const uint32_t lo = *reinterpret_cast<const uint16_t *>(work + t * WRB + 2 * ch);
        const uint32_t hi = *reinterpret_cast<const uint16_t *>(work + (t + 1) * WRB + 2 * ch);
        wv[e] = lo | (hi << 16);
      }
      *reinterpret_cast<uint4 *>(rec + S * D * 2 + vt * TILE + gi * 512 + lane * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
  }
}

template <int D, int S>
__global__ void __launch_bounds__(QuantGeo<D, S>::TEAMS * 128, 1) k_quant(QuantArgs a) {
  using QG = QuantGeo<D, S>;
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp >> 2, tw = warp & 3;
  uint8_t *tbase = sm + (size_t)team * QG::PER_TEAM;
  constexpr int NSL = QG::NSL;
  uint8_t *work = tbase + NSL * QG::WIN + tw * (QG::WORK + QG::SCR);
  float2 *scr = reinterpret_cast<float2 *>(work + QG::WORK);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + QG::bar_off) + team * 2 * NSL;   // [NSL] full, [NSL] empty
  uint64_t *empty = full + NSL;
  WinDesc *wdesc = reinterpret_cast<WinDesc *>(sm + QG::desc_off) + team * NSL;
  const int64_t nwin = (int64_t)a.B * a.H * a.perm_stride;
  const int64_t gt = (int64_t)blockIdx.x * QG::TEAMS + team, nt = (int64_t)gridDim.x * QG::TEAMS;
  if (tw == 0 && lane == 0) {
    for (int i = 0; i < NSL; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 4); }
    fence_mbar_init();
  }
  __syncthreads();
  auto locate = [&](int64_t wi, int &b, int &h, int &slot) {
    slot = (int)(wi % a.perm_stride);
    const int64_t bh = wi / a.perm_stride;
    h = (int)(bh % a.H);
    b = (int)(bh / a.H);
  };
  // Window metadata (seg_off, perm, offs) of team window k, loaded by the issuing lane one
  // window AHEAD of its copy: the three loads are independent (issued together, before any
  // branch on their values) and complete while the warp quantizes, so the bulk copy of a
  // window never waits on a global round trip (ncu r01: 75% long_sb on the issue path).
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
      if (kk < cls) roff += (int64_t)(m.so[kk + 1] - m.so[kk]) * record_bytes(class_bits(kk), D, S);
    const int sbase = cls == 0 ? m.so[0] : cls == 1 ? m.so[1] : cls == 2 ? m.so[2] : m.so[3];
    roff += (int64_t)(slot - sbase) * record_bytes(bits, D, S);
    WQ_CHECK(roff >= a.offs[(int64_t)b * a.H + h] && roff + record_bytes(bits, D, S) <= a.offs[(int64_t)b * a.H + h + 1]);
    wdesc[sl].roff = roff;
    wdesc[sl].bits = bits;
    const int64_t ro = b * a.sb + h * a.sh + (int64_t)(a.vis_off + w * S) * a.st;
    uint8_t *dst = tbase + (size_t)sl * QG::WIN;
    const uint64_t pol = policy_evict_first();
    mbar_arrive_expect_tx(&full[sl], (uint32_t)(4 * S * D));
    if (a.st == D) {
      bulk_g2s_evict_first(dst, a.k + ro, S * 2 * D, &full[sl], pol);
      bulk_g2s_evict_first(dst + S * 2 * D, a.v + ro, S * 2 * D, &full[sl], pol);
    } else {
      for (int t = 0; t < S; t++) {
        bulk_g2s_evict_first(dst + t * 2 * D, a.k + ro + t * a.st, 2 * D, &full[sl], pol);
        bulk_g2s_evict_first(dst + S * 2 * D + t * 2 * D, a.v + ro + t * a.st, 2 * D, &full[sl], pol);
      }
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
      const uint8_t *krows = tbase + (size_t)sl * QG::WIN, *vrows = krows + S * 2 * D;
      for (int tk = tw; tk < QG::NT; tk += 4) {
        if (bits == 16) {
          copy_task_fp16<D, S>(krows, vrows, work, rec, tk, lane);
        } else if (tk < 2) {
          if (bits == 2) quant_k_half<D, S, 2>(krows, work, scr, rec, tk, lane);
          else if (bits == 4) quant_k_half<D, S, 4>(krows, work, scr, rec, tk, lane);
          else quant_k_half<D, S, 8>(krows, work, scr, rec, tk, lane);
        } else {
          if (bits == 2) quant_v_tile<D, S, 2>(vrows, work, scr, rec, tk - 2, lane);
          else if (bits == 4) quant_v_tile<D, S, 4>(vrows, work, scr, rec, tk - 2, lane);
          else quant_v_tile<D, S, 8>(vrows, work, scr, rec, tk - 2, lane);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sl]);       // this warp is done with the slot
  }
}

template <int D, int S>
static cudaError_t launch_quant_t(const QuantArgs &a, cudaStream_t st) {
  using QG = QuantGeo<D, S>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_quant<D, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)QG::total);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t nwin = (int64_t)a.B * a.H * a.perm_stride;
  int64_t grid = device_sm_count();
  const int64_t need = (nwin + QG::TEAMS - 1) / QG::TEAMS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  k_quant<D, S><<<(unsigned)grid, QG::TEAMS * 128, QG::total, st>>>(a);
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

cudaError_t launch_layer_layout(const int32_t *seg_off, int B, int H, int d, int S, int64_t *offs,
                                cudaStream_t st) {
  k_layer_layout<<<1, 256, (size_t)B * sizeof(int64_t), st>>>(seg_off, B, H, d, S, offs);
  return cudaGetLastError();
}

cudaError_t launch_quant(const __half *k, const __half *v, const int64_t strides[3], int vis_off,
                         int B, int H, int d, int S, int M, const int32_t *perm, int perm_stride,
                         const int32_t *seg_off, const int64_t *offs, uint8_t *packed,
                         cudaStream_t st) {
  QuantArgs a{k, v, strides[0], strides[1], strides[2], vis_off, B, H, d, S, M, perm, perm_stride,
              seg_off, offs, packed};
#define WQ_Q(DD, SS) \
  if (d == DD && S == SS) return launch_quant_t<DD, SS>(a, st);
  WQ_Q(64, 16) WQ_Q(64, 32) WQ_Q(64, 64) WQ_Q(64, 128)
  WQ_Q(128, 16) WQ_Q(128, 32) WQ_Q(128, 64) WQ_Q(128, 128)
#undef WQ_Q
  return cudaErrorInvalidValue;
}

}  // namespace wq
