// decode.cu -- wq_decode_attention: split-KV flash-decoding over the reordered
// mixed-precision cache (Alg.2 decode branch P:450-458; Eq.2-3 without mask, P:214;
// reorder invariance Eq.12-13; fused dequantization P:510), plus the
// LSE merge of partials (wq_merge_partials, the cross-GPU step of §8(e)).
//
// Design:
//  * Persistent grid, one CTA per SM: 1 producer warp + NCW consumer warps.
//  * Work = the byte stream of all (request, kv-head) "units": each unit's packed
//    image (segments 2|4|8|16 in slot order) followed by its FP16 rest tokens in
//    16-token tiles.  CTA c owns the items whose first byte falls in the c-th
//    equal share of the stream -> byte-balanced split-KV across precisions.
//  * Producer: TMA 1-D bulk copies (cp.async.bulk) of whole items into a 4-stage
//    shared-memory ring (mbarrier full/empty), L2 evict-first.
//  * Consumers: one warp per window.  K side: scores[t][j] = sum_c code[t][c] *
//    q'_j[c] + bias_j with q' = q*s_c folded per window (split hi+lo in fp16 so the
//    product is carried to ~2^-22) and bias_j = sum_c q_j[c]*mn_c, all on
//    mma.sync m16n8k16 (tokens x heads, fp32 accumulate).  Codes are loaded in
//    D-1 fragment order straight into MMA A registers and turned into exact fp16
//    integers with one LOP3 + one HSUB2 per pair (magic-exponent trick).  Online
//    softmax per window in the exp2 domain with a lazy rescale (max may run 2^8
//    ahead).  V side: o[c][j] += sum_t vcode[t][c] * p'_j[t], p' = p*s_t, the
//    per-token zero point contributing sum_t p_t*mn_t to every channel.
//  * Unit epilogue: warps merged in shared memory, the CTA partial (m, l, o) goes
//    to the workspace, and the last CTA of the unit (atomic ticket) merges all
//    partials by log-sum-exp and writes out / partial (Q24).
#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {

constexpr int NCW = 8;                  // consumer warps
constexpr int DT = (NCW + 1) * 32;      // threads per CTA
constexpr int MAXIT = 48;               // items per stage
constexpr int MAX_UNITS = 1024;         // B * H
constexpr int64_t MIN_CTA_BYTES = 49152;
constexpr float LAZY_TH = 8.0f;         // log2 headroom of the lazy softmax rescale
constexpr int KIND_REST = 4;

struct StageDesc {
  int unit, nitems, flags;              // flags: 1 = last stage of unit, 2 = last of CTA
  uint8_t kind[MAXIT];                  // 0..3 = width class, 4 = rest tile
  uint8_t ntok[MAXIT];                  // valid tokens of a rest tile
  uint16_t off[MAXIT];                  // byte offset in the stage
};

struct UnitGeo {
  int b, h, nslots, rl, ntiles;
  int so[5];
  int64_t cs[5];                        // byte start of each class segment; cs[4] = image bytes
};

WQ_DEV void unit_geo(const DecodeArgs &a, int u, UnitGeo &g) {
  g.b = u / a.H;
  g.h = u % a.H;
  const int32_t *so = a.seg_off + 5 * g.b;
  for (int k = 0; k < 5; k++) g.so[k] = so[k];
  g.cs[0] = 0;
  for (int k = 0; k < 4; k++)
    g.cs[k + 1] = g.cs[k] + (int64_t)(g.so[k + 1] - g.so[k]) * record_bytes(class_bits(k), a.d, a.S);
  g.nslots = g.so[4];
  g.rl = a.rest_len ? a.rest_len[g.b] : 0;
  g.ntiles = (g.rl + 15) / 16;
}
WQ_DEV int64_t unit_bytes(const DecodeArgs &a, const UnitGeo &g) { return g.cs[4] + (int64_t)g.rl * 4 * a.d; }

// first item whose start offset (relative to the unit) is >= x
WQ_DEV int first_item(const DecodeArgs &a, const UnitGeo &g, int64_t x) {
  if (x <= 0) return 0;
  for (int k = 0; k < 4; k++) {
    if (x <= g.cs[k]) return g.so[k];
    if (x < g.cs[k + 1]) {
      int64_t rb = record_bytes(class_bits(k), a.d, a.S);
      return g.so[k] + (int)((x - g.cs[k] + rb - 1) / rb);
    }
  }
  if (x <= g.cs[4]) return g.nslots;
  int64_t tb = 64LL * a.d;
  int64_t t = (x - g.cs[4] + tb - 1) / tb;
  return g.nslots + (int)(t < g.ntiles ? t : g.ntiles);
}

WQ_DEV int64_t cta_lo(int c, int G, int64_t T) { return (int64_t)c * T / G; }
WQ_DEV int owner_of(int64_t x, int G, int64_t T) {
  if (T <= 0) return 0;
  int c = (int)((x * G) / T);
  if (c >= G) c = G - 1;
  while (c + 1 < G && cta_lo(c + 1, G, T) <= x) c++;
  while (c > 0 && cta_lo(c, G, T) > x) c--;
  return c;
}

struct WarpState {
  float m[2], l[2], vb[2];
};

// -------------------------------------------------------------------------------------
// consumer: one window (BITS in {2,4,8,16}) or one rest tile
// -------------------------------------------------------------------------------------
// K-side scores for NT token tiles of one quantized / fp16-fragment window.
template <int D, int NT, int BITS>
WQ_DEV void window_scores(const uint8_t *rec, const uint32_t (&qf)[D / 16][2], float (&sc)[NT][4],
                          int lane) {
  constexpr int KT = D / 16;
  constexpr int WPL = D * BITS / 64;          // words per lane per tile
  constexpr int PPW = 16 / BITS;              // pairs per word
  float bias[4] = {0.f, 0.f, 0.f, 0.f};
  uint32_t qh[KT][2], ql[KT][2];
  if constexpr (BITS < 16) {
    const uint8_t *kp = rec + 2 * (NT * 16 * D * BITS / 8);
    const int q = lane & 3;
#pragma unroll
    for (int kt = 0; kt < KT; kt++) {
      uint4 pr = lds128(kp + (q * KT + kt) * 16);   // {s01, s89, mn01, mn89}
      uint32_t am[4] = {pr.z, pr.z, pr.w, pr.w};
      mma16816(bias, am, qf[kt][0], qf[kt][1], bias);
      qh[kt][0] = hmul2u(qf[kt][0], pr.x);
      ql[kt][0] = hfma2u(qf[kt][0], pr.x, hneg2u(qh[kt][0]));
      qh[kt][1] = hmul2u(qf[kt][1], pr.y);
      ql[kt][1] = hfma2u(qf[kt][1], pr.y, hneg2u(qh[kt][1]));
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; nt++) {
    const uint8_t *ch = rec + nt * (2 * D * BITS) + lane * (D * BITS / 16);
    uint32_t wd[WPL];
    if constexpr (WPL >= 4) {
#pragma unroll
      for (int i = 0; i < WPL / 4; i++) {
        uint4 v = lds128(ch + 16 * i);
        wd[4 * i] = v.x; wd[4 * i + 1] = v.y; wd[4 * i + 2] = v.z; wd[4 * i + 3] = v.w;
      }
    } else {
      uint2 v = lds64(ch);
      wd[0] = v.x; wd[1] = v.y;
    }
    float acc[4] = {bias[0], bias[1], bias[2], bias[3]};
#pragma unroll
    for (int kt = 0; kt < KT; kt++) {
      uint32_t a[4];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int P = 4 * kt + r;
        const uint32_t w = wd[P / PPW];
        if constexpr (BITS == 16) a[r] = w;
        else if constexpr (BITS == 2) {
          const uint32_t w8 = w >> 8;
          switch (P % PPW) {
            case 0: a[r] = dq_pair<2, 0>(w, w8); break;
            case 1: a[r] = dq_pair<2, 1>(w, w8); break;
            case 2: a[r] = dq_pair<2, 2>(w, w8); break;
            case 3: a[r] = dq_pair<2, 3>(w, w8); break;
            case 4: a[r] = dq_pair<2, 4>(w, w8); break;
            case 5: a[r] = dq_pair<2, 5>(w, w8); break;
            case 6: a[r] = dq_pair<2, 6>(w, w8); break;
            default: a[r] = dq_pair<2, 7>(w, w8); break;
          }
        } else if constexpr (BITS == 4) {
          const uint32_t w8 = w >> 8;
          switch (P % PPW) {
            case 0: a[r] = dq_pair<4, 0>(w, w8); break;
            case 1: a[r] = dq_pair<4, 1>(w, w8); break;
            case 2: a[r] = dq_pair<4, 2>(w, w8); break;
            default: a[r] = dq_pair<4, 3>(w, w8); break;
          }
        } else {
          a[r] = (P % PPW) == 0 ? dq_pair<8, 0>(w, 0) : dq_pair<8, 1>(w, 0);
        }
      }
      if constexpr (BITS < 16) {
        mma16816(acc, a, qh[kt][0], qh[kt][1], acc);
        mma16816(acc, a, ql[kt][0], ql[kt][1], acc);
      } else {
        mma16816(acc, a, qf[kt][0], qf[kt][1], acc);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) sc[nt][i] = acc[i];
  }
}

// V side for tile nt of a window: o[mt] += Vcode^T(16 ch x 16 tok) * P'(16 tok x 8 heads)
template <int D, int BITS>
WQ_DEV void window_pv(const uint8_t *vtile, uint32_t pb0, uint32_t pb1, float (&o)[D / 16][4],
                      int lane) {
  constexpr int KT = D / 16;
  constexpr int WPL = D * BITS / 64;
  constexpr int PPW = 16 / BITS;
  const uint8_t *ch = vtile + lane * (D * BITS / 16);
  uint32_t wd[WPL];
  if constexpr (WPL >= 4) {
#pragma unroll
    for (int i = 0; i < WPL / 4; i++) {
      uint4 v = lds128(ch + 16 * i);
      wd[4 * i] = v.x; wd[4 * i + 1] = v.y; wd[4 * i + 2] = v.z; wd[4 * i + 3] = v.w;
    }
  } else {
    uint2 v = lds64(ch);
    wd[0] = v.x; wd[1] = v.y;
  }
#pragma unroll
  for (int mt = 0; mt < KT; mt++) {
    uint32_t a[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int P = 4 * mt + r;
      const uint32_t w = wd[P / PPW];
      if constexpr (BITS == 16) a[r] = w;
      else if constexpr (BITS == 2) {
        const uint32_t w8 = w >> 8;
        switch (P % PPW) {
          case 0: a[r] = dq_pair<2, 0>(w, w8); break;
          case 1: a[r] = dq_pair<2, 1>(w, w8); break;
          case 2: a[r] = dq_pair<2, 2>(w, w8); break;
          case 3: a[r] = dq_pair<2, 3>(w, w8); break;
          case 4: a[r] = dq_pair<2, 4>(w, w8); break;
          case 5: a[r] = dq_pair<2, 5>(w, w8); break;
          case 6: a[r] = dq_pair<2, 6>(w, w8); break;
          default: a[r] = dq_pair<2, 7>(w, w8); break;
        }
      } else if constexpr (BITS == 4) {
        const uint32_t w8 = w >> 8;
        switch (P % PPW) {
          case 0: a[r] = dq_pair<4, 0>(w, w8); break;
          case 1: a[r] = dq_pair<4, 1>(w, w8); break;
          case 2: a[r] = dq_pair<4, 2>(w, w8); break;
          default: a[r] = dq_pair<4, 3>(w, w8); break;
        }
      } else {
        a[r] = (P % PPW) == 0 ? dq_pair<8, 0>(w, 0) : dq_pair<8, 1>(w, 0);
      }
    }
    mma16816(o[mt], a, pb0, pb1, o[mt]);
  }
}

// Online softmax over NT tiles of scores (already in the log2 domain), writes P'
// (p * s_t) as fp16 [token][8 heads] rows to the warp scratch.
template <int NT, int KT>
WQ_DEV void softmax_tiles(float (&s)[NT][4], WarpState &st, float (&o)[KT][4],
                          const float (&vs)[NT][2], const float (&vm)[NT][2], bool has_vparams,
                          uint8_t *scratch, int lane) {
  const int g = lane >> 2, q = lane & 3;
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < NT; nt++) {
    mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][2]));
    mx1 = fmaxf(mx1, fmaxf(s[nt][1], s[nt][3]));
  }
#pragma unroll
  for (int off = 4; off <= 16; off <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
  }
  const bool n0 = mx0 > st.m[0] + LAZY_TH || (st.m[0] == -INFINITY && mx0 > -INFINITY);
  const bool n1 = mx1 > st.m[1] + LAZY_TH || (st.m[1] == -INFINITY && mx1 > -INFINITY);
  if (__any_sync(0xffffffffu, n0 || n1)) {
    float a0 = 1.f, a1 = 1.f;
    if (n0) { a0 = exp2f(st.m[0] - mx0); st.m[0] = mx0; }
    if (n1) { a1 = exp2f(st.m[1] - mx1); st.m[1] = mx1; }
    st.l[0] *= a0; st.vb[0] *= a0;
    st.l[1] *= a1; st.vb[1] *= a1;
#pragma unroll
    for (int mt = 0; mt < KT; mt++) {
      o[mt][0] *= a0; o[mt][1] *= a1; o[mt][2] *= a0; o[mt][3] *= a1;
    }
  }
  const float m0 = st.m[0], m1 = st.m[1];
#pragma unroll
  for (int nt = 0; nt < NT; nt++) {
    float p0 = m0 == -INFINITY ? 0.f : exp2f(s[nt][0] - m0);
    float p1 = m1 == -INFINITY ? 0.f : exp2f(s[nt][1] - m1);
    float p2 = m0 == -INFINITY ? 0.f : exp2f(s[nt][2] - m0);
    float p3 = m1 == -INFINITY ? 0.f : exp2f(s[nt][3] - m1);
    st.l[0] += p0 + p2;
    st.l[1] += p1 + p3;
    if (has_vparams) {
      st.vb[0] = fmaf(p0, vm[nt][0], fmaf(p2, vm[nt][1], st.vb[0]));
      st.vb[1] = fmaf(p1, vm[nt][0], fmaf(p3, vm[nt][1], st.vb[1]));
      p0 *= vs[nt][0]; p1 *= vs[nt][0];
      p2 *= vs[nt][1]; p3 *= vs[nt][1];
    }
    sts32(scratch + (16 * nt + g) * 16 + 4 * q, pack_f2h2(p0, p1));
    sts32(scratch + (16 * nt + g + 8) * 16 + 4 * q, pack_f2h2(p2, p3));
  }
  __syncwarp();
}

template <int D, int S, int BITS>
WQ_DEV void do_window(const uint8_t *rec, const uint32_t (&qf)[D / 16][2], float scale2,
                      WarpState &st, float (&o)[D / 16][4], uint8_t *scratch, int lane) {
  constexpr int NT = S / 16;
  constexpr int KT = D / 16;
  float sc[NT][4];
  window_scores<D, NT, BITS>(rec, qf, sc, lane);
#pragma unroll
  for (int nt = 0; nt < NT; nt++)
#pragma unroll
    for (int i = 0; i < 4; i++) sc[nt][i] *= scale2;
  float vs[NT][2], vm[NT][2];
  const int g = lane >> 2;
  if constexpr (BITS < 16) {
    const uint8_t *vp = rec + 2 * (S * D * BITS / 8) + 4 * D;
#pragma unroll
    for (int nt = 0; nt < NT; nt++) {
      uint4 pr = lds128(vp + (4 * nt + (g >> 1)) * 16);
      const __half *hp = reinterpret_cast<const __half *>(&pr);
      const int e = g & 1;
      vs[nt][0] = __half2float(hp[e]);
      vs[nt][1] = __half2float(hp[2 + e]);
      vm[nt][0] = __half2float(hp[4 + e]);
      vm[nt][1] = __half2float(hp[6 + e]);
    }
  }
  softmax_tiles<NT, KT>(sc, st, o, vs, vm, BITS < 16, scratch, lane);
  const uint8_t *vcodes = rec + S * D * BITS / 8;
#pragma unroll
  for (int nt = 0; nt < NT; nt++) {
    uint32_t pb[2];
    // lanes 0-7: tokens 16nt+0..7, lanes 8-15: tokens 16nt+8..15 (rows of 16 B)
    ldsm_x2_t(pb, scratch + (16 * nt + (lane & 15)) * 16);
    window_pv<D, BITS>(vcodes + nt * (2 * D * BITS), pb[0], pb[1], o, lane);
  }
  __syncwarp();
}

// FP16 rest tile: K rows [16][D] at base, V rows [16][D] at base + 32*D (natural layout)
template <int D>
WQ_DEV void do_rest(const uint8_t *base, int ntok, const uint32_t (&qf)[D / 16][2], float scale2,
                    WarpState &st, float (&o)[D / 16][4], uint8_t *scratch, int lane) {
  constexpr int KT = D / 16;
  const __half *Ks = reinterpret_cast<const __half *>(base);
  const __half *Vs = Ks + 16 * D;
  const int g = lane >> 2, q = lane & 3, mi = lane >> 3, rr = lane & 7;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int kt = 0; kt < KT; kt++) {
    uint32_t a[4];
    ldsm_x4(a, Ks + ((mi & 1) * 8 + rr) * D + 16 * kt + (mi >> 1) * 8);
    mma16816(acc, a, qf[kt][0], qf[kt][1], acc);
  }
  float sc[1][4];
  sc[0][0] = g < ntok ? acc[0] * scale2 : -INFINITY;
  sc[0][1] = g < ntok ? acc[1] * scale2 : -INFINITY;
  sc[0][2] = g + 8 < ntok ? acc[2] * scale2 : -INFINITY;
  sc[0][3] = g + 8 < ntok ? acc[3] * scale2 : -INFINITY;
  float vs[1][2], vm[1][2];
  softmax_tiles<1, KT>(sc, st, o, vs, vm, false, scratch, lane);
  uint32_t pb[2];
  ldsm_x2_t(pb, scratch + (lane & 15) * 16);
  // zero masked token columns of V^T (stale shared memory may hold non-finite bits)
  const uint32_t m01 = (2 * q < ntok ? 0xffffu : 0u) | (2 * q + 1 < ntok ? 0xffff0000u : 0u);
  const uint32_t m89 = (2 * q + 8 < ntok ? 0xffffu : 0u) | (2 * q + 9 < ntok ? 0xffff0000u : 0u);
#pragma unroll
  for (int mt = 0; mt < KT; mt++) {
    uint32_t a[4];
    ldsm_x4_t(a, Vs + ((mi >> 1) * 8 + rr) * D + 16 * mt + (mi & 1) * 8);
    a[0] &= m01; a[1] &= m01; a[2] &= m89; a[3] &= m89;
    mma16816(o[mt], a, pb[0], pb[1], o[mt]);
  }
  __syncwarp();
}

// -------------------------------------------------------------------------------------
// the kernel
// -------------------------------------------------------------------------------------
template <int D, int S>
struct DecodeSmem {
  // a stage must hold the largest item (an FP16 window: 4*S*D bytes)
  static constexpr int STAGE = (4 * S * D > 32768) ? 4 * S * D : 32768;
  static constexpr int NST = (STAGE >= 65536) ? 2 : 4;
  static constexpr int KT = D / 16;
  static constexpr int SCRATCH = S * 16;                 // P' rows per warp
  static constexpr int EP_WARP = 8 * D + 24;             // floats per warp in the epilogue
  static constexpr size_t ring = (size_t)NST * STAGE;
  static constexpr size_t scratch_off = ring;
  static constexpr size_t ep_off = scratch_off + (size_t)NCW * SCRATCH;
  static constexpr size_t units_off = ep_off + (size_t)NCW * EP_WARP * 4;
  static constexpr size_t desc_off = units_off + (size_t)(MAX_UNITS + 1) * 8;
  static constexpr size_t bar_off = desc_off + NST * sizeof(StageDesc);
  static constexpr size_t total = bar_off + 2 * NST * 8 + 16;
};

template <int D, int S>
__global__ void __launch_bounds__(DT, 1) k_decode(DecodeArgs a) {
  using SM = DecodeSmem<D, S>;
  constexpr int KT = D / 16;
  constexpr int NST = SM::NST;
  constexpr int STAGE = SM::STAGE;
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t *ring = sm;
  int64_t *ustart = reinterpret_cast<int64_t *>(sm + SM::units_off);
  StageDesc *desc = reinterpret_cast<StageDesc *>(sm + SM::desc_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + SM::bar_off);
  uint64_t *empty = full + NST;
  int *s_flag = reinterpret_cast<int *>(empty + NST);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int U = a.B * a.H;

  // ---- unit byte prefix (warp 0) ----
  if (warp == 0) {
    int64_t carry = 0;
    for (int base = 0; base < U; base += 32) {
      int u = base + lane;
      int64_t v = 0;
      if (u < U) {
        UnitGeo gg;
        unit_geo(a, u, gg);
        v = unit_bytes(a, gg);
      }
      int64_t x = v;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (u < U) ustart[u] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) ustart[U] = carry;
  }
  if (tid == 0) {
    for (int s = 0; s < NST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t T = ustart[U];
  int G = (int)(T / MIN_CTA_BYTES);
  G = G < 1 ? 1 : (G > (int)gridDim.x ? (int)gridDim.x : G);
  const int c = blockIdx.x;
  if (c >= G) return;
  const int64_t lo = cta_lo(c, G, T), hi = cta_lo(c + 1, G, T);

  if (warp == NCW) {
    // =========================== producer ===========================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      int last_u = -1;
      for (int u = 0; u < U; u++) {
        const int64_t us = ustart[u], ue = ustart[u + 1];
        if (ue > us) {
          if (ue <= lo || us >= hi) continue;
        } else if (owner_of(us, G, T) != c) {
          continue;
        }
        last_u = u;
      }
      for (int u = 0; u < U; u++) {
        const int64_t us = ustart[u], ue = ustart[u + 1];
        if (ue > us) {
          if (ue <= lo || us >= hi) continue;
        } else if (owner_of(us, G, T) != c) {
          continue;
        }
        UnitGeo gg;
        unit_geo(a, u, gg);
        const int nitems = gg.nslots + gg.ntiles;
        int i = first_item(a, gg, lo - us);
        const int i1 = hi >= ue ? nitems : first_item(a, gg, hi - us);
        const uint8_t *img = a.packed + a.offs[u];
        const __half *kr = a.k_rest + gg.b * a.rs_b + gg.h * a.rs_h;
        const __half *vr = a.v_rest + gg.b * a.rs_b + gg.h * a.rs_h;
        do {
          mbar_wait(&empty[stage], phase ^ 1);
          StageDesc &dsc = desc[stage];
          uint8_t *dst = ring + (size_t)stage * STAGE;
          int n = 0;
          uint32_t bytes = 0, tx = 0;
          int k = 0;
          while (i < i1 && n < MAXIT) {
            uint32_t sz;
            int kind, ntok = 0;
            if (i < gg.nslots) {
              while (i >= gg.so[k + 1]) k++;
              kind = k;
              sz = (uint32_t)record_bytes(class_bits(k), D, S);
            } else {
              kind = KIND_REST;
              int t0 = 16 * (i - gg.nslots);
              ntok = min(16, gg.rl - t0);
              sz = 64u * D;
            }
            if (bytes + sz > (uint32_t)STAGE) break;
            dsc.kind[n] = (uint8_t)kind;
            dsc.ntok[n] = (uint8_t)ntok;
            dsc.off[n] = (uint16_t)bytes;
            tx += kind == KIND_REST ? (uint32_t)ntok * 4u * D : sz;
            bytes += sz;
            n++;
            i++;
          }
          if (n == 0 && i < i1) __trap();   // an item larger than a stage (never: STAGE >= 4*S*D)
          dsc.unit = u;
          dsc.nitems = n;
          dsc.flags = (i >= i1 ? 1 : 0) | ((i >= i1 && u == last_u) ? 2 : 0);
          mbar_arrive_expect_tx(&full[stage], tx);
          // issue the copies (contiguous runs of packed records merged into one copy)
          int j = 0;
          while (j < n) {
            if (dsc.kind[j] != KIND_REST) {
              int j2 = j + 1;
              while (j2 < n && dsc.kind[j2] != KIND_REST) j2++;
              int first = i - n + j;
              int kk = 0;
              while (first >= gg.so[kk + 1]) kk++;
              int64_t src = gg.cs[kk] + (int64_t)(first - gg.so[kk]) * record_bytes(class_bits(kk), D, S);
              uint32_t nb = (j2 < n ? dsc.off[j2] : bytes) - dsc.off[j];
              bulk_g2s_evict_first(dst + dsc.off[j], img + src, nb, &full[stage], pol);
              j = j2;
            } else {
              int t0 = 16 * (i - n + j - gg.nslots);
              int nt = dsc.ntok[j];
              bulk_g2s_evict_first(dst + dsc.off[j], kr + (int64_t)t0 * D, (uint32_t)nt * 2 * D,
                                   &full[stage], pol);
              bulk_g2s_evict_first(dst + dsc.off[j] + 32 * D, vr + (int64_t)t0 * D,
                                   (uint32_t)nt * 2 * D, &full[stage], pol);
              j++;
            }
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        } while (i < i1);
      }
    }
    return;
  }

  // =========================== consumers ===========================
  uint8_t *scratch = sm + SM::scratch_off + warp * SM::SCRATCH;
  float *ep = reinterpret_cast<float *>(sm + SM::ep_off);
  const int g = lane >> 2, q = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  int cur_u = -1;
  uint32_t qf[KT][2];
  float o[KT][4];
  WarpState st;
  for (int mt = 0; mt < KT; mt++) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = st.vb[0] = st.vb[1] = 0.f;

  for (;;) {
    mbar_wait(&full[stage], phase);
    const StageDesc &dsc = desc[stage];
    const int u = dsc.unit, n = dsc.nitems, flags = dsc.flags;
    if (u != cur_u) {
      cur_u = u;
      const int b = u / a.H, h = u % a.H;
      const __half *qrow = a.q + ((int64_t)b * a.Hq + h * a.grp + g) * D;
#pragma unroll
      for (int kt = 0; kt < KT; kt++) {
        qf[kt][0] = g < a.grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q) : 0u;
        qf[kt][1] = g < a.grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q + 8) : 0u;
      }
    }
    const uint8_t *sbase = ring + (size_t)stage * STAGE;
    for (int it = warp; it < n; it += NCW) {
      const uint8_t *rec = sbase + dsc.off[it];
      switch (dsc.kind[it]) {
        case 0: do_window<D, S, 2>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        case 1: do_window<D, S, 4>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        case 2: do_window<D, S, 8>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        case 3: do_window<D, S, 16>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        default: do_rest<D>(rec, dsc.ntok[it], qf, a.scale_log2, st, o, scratch, lane); break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == NST) { stage = 0; phase ^= 1; }
    if (!(flags & 1)) continue;

    // ---------------- unit epilogue ----------------
    {
      // reduce lane partials over the 8 lanes sharing a head pair (xor 4, 8, 16)
      for (int off = 4; off <= 16; off <<= 1) {
        st.l[0] += __shfl_xor_sync(0xffffffffu, st.l[0], off);
        st.l[1] += __shfl_xor_sync(0xffffffffu, st.l[1], off);
        st.vb[0] += __shfl_xor_sync(0xffffffffu, st.vb[0], off);
        st.vb[1] += __shfl_xor_sync(0xffffffffu, st.vb[1], off);
      }
      float *mine = ep + warp * SM::EP_WARP;     // [m 8][l 8][vb 8][o D x 8]
      if (g == 0) {
        mine[2 * q] = st.m[0]; mine[2 * q + 1] = st.m[1];
        mine[8 + 2 * q] = st.l[0]; mine[8 + 2 * q + 1] = st.l[1];
        mine[16 + 2 * q] = st.vb[0]; mine[16 + 2 * q + 1] = st.vb[1];
      }
#pragma unroll
      for (int mt = 0; mt < KT; mt++) {
        float *oc = mine + 24 + (16 * mt + g) * 8 + 2 * q;
        oc[0] = o[mt][0]; oc[1] = o[mt][1];
        oc[64] = o[mt][2]; oc[65] = o[mt][3];     // channel + 8
      }
      named_bar_sync(1, NCW * 32);
      const int b = u / a.H, h = u % a.H;
      const int64_t us = ustart[u], ue = ustart[u + 1];
      const int cf = owner_of(us, G, T);
      const int cl = ue > us ? owner_of(ue - 1, G, T) : cf;
      float *slot = a.ws_part + (int64_t)(c + u) * a.grp * (D + 2);
      for (int idx = tid; idx < a.grp * (D + 2); idx += NCW * 32) {
        const int j = idx / (D + 2), e = idx % (D + 2);
        float M = -INFINITY;
        for (int w = 0; w < NCW; w++) M = fmaxf(M, ep[w * SM::EP_WARP + j]);
        float acc = 0.f;
        for (int w = 0; w < NCW; w++) {
          const float *pw = ep + w * SM::EP_WARP;
          const float f = (M == -INFINITY) ? 0.f : exp2f(pw[j] - M);
          if (e == 1) acc += f * pw[8 + j];
          else if (e >= 2) acc += f * (pw[24 + (e - 2) * 8 + j] + pw[16 + j]);
        }
        slot[idx] = e == 0 ? M : acc;
      }
      __threadfence();
      named_bar_sync(1, NCW * 32);
      if (tid == 0) {
        const int old = atomicAdd(a.ws_cnt + u, 1);
        *s_flag = (old == cl - cf);
      }
      named_bar_sync(1, NCW * 32);
      if (*s_flag) {
        __threadfence();
        for (int idx = tid; idx < a.grp * D; idx += NCW * 32) {
          const int j = idx / D, cc = idx % D;
          float M = -INFINITY;
          for (int c2 = cf; c2 <= cl; c2++) {
            const float *sp = a.ws_part + (int64_t)(c2 + u) * a.grp * (D + 2) + j * (D + 2);
            M = fmaxf(M, __ldcg(sp));
          }
          float L = 0.f, O = 0.f;
          for (int c2 = cf; c2 <= cl; c2++) {
            const float *sp = a.ws_part + (int64_t)(c2 + u) * a.grp * (D + 2) + j * (D + 2);
            const float f = (M == -INFINITY) ? 0.f : exp2f(__ldcg(sp) - M);
            L += f * __ldcg(sp + 1);
            O += f * __ldcg(sp + 2 + cc);
          }
          const int64_t row = (int64_t)b * a.Hq + h * a.grp + j;
          if (a.out) a.out[row * D + cc] = __float2half_rn(L > 0.f ? O / L : 0.f);
          if (a.partial) {
            float *pp = a.partial + row * (D + 2);
            if (cc == 0) {
              pp[0] = M * 0.69314718055994530942f;   // log2 domain -> natural
              pp[1] = L;
            }
            pp[2 + cc] = O;
          }
        }
        if (tid == 0) a.ws_cnt[u] = 0;
      }
      named_bar_sync(1, NCW * 32);
      // reset warp state for the next unit
      for (int mt = 0; mt < KT; mt++) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
      st.m[0] = st.m[1] = -INFINITY;
      st.l[0] = st.l[1] = st.vb[0] = st.vb[1] = 0.f;
    }
    if (flags & 2) break;
  }
}

__global__ void k_merge(const float *__restrict__ parts, int G, int BHq, int d, __half *__restrict__ out) {
  const int row = blockIdx.x;
  for (int cc = threadIdx.x; cc < d; cc += blockDim.x) {
    float M = -INFINITY;
    for (int g = 0; g < G; g++) {
      const float *p = parts + ((int64_t)g * BHq + row) * (d + 2);
      if (p[1] > 0.f) M = fmaxf(M, p[0]);
    }
    float L = 0.f, O = 0.f;
    for (int g = 0; g < G; g++) {
      const float *p = parts + ((int64_t)g * BHq + row) * (d + 2);
      if (!(p[1] > 0.f)) continue;
      const float f = expf(p[0] - M);
      L += f * p[1];
      O += f * p[2 + cc];
    }
    out[(int64_t)row * d + cc] = __float2half_rn(L > 0.f ? O / L : 0.f);
  }
}

size_t decode_workspace_bytes(int B, int H, int Hq, int d, int num_sms) {
  const int grp = Hq / H;
  size_t part = (size_t)(num_sms + B * H) * grp * (d + 2) * sizeof(float);
  part = (part + 255) / 256 * 256;
  return part + (size_t)B * H * sizeof(int32_t);
}

template <int D, int S>
static cudaError_t launch_decode_t(const DecodeArgs &a, int num_sms, cudaStream_t st) {
  using SM = DecodeSmem<D, S>;
  cudaError_t e = cudaFuncSetAttribute(k_decode<D, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SM::total);
  if (e != cudaSuccess) return e;
  k_decode<D, S><<<num_sms, DT, SM::total, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_decode(const DecodeArgs &a, int num_sms, cudaStream_t st) {
#define WQ_D(DD, SS) \
  if (a.d == DD && a.S == SS) return launch_decode_t<DD, SS>(a, num_sms, st);
  WQ_D(64, 16) WQ_D(64, 32) WQ_D(64, 64) WQ_D(64, 128)
  WQ_D(128, 16) WQ_D(128, 32) WQ_D(128, 64) WQ_D(128, 128)
#undef WQ_D
  return cudaErrorInvalidValue;
}

cudaError_t launch_merge(const float *parts, int G, int BHq, int d, __half *out, cudaStream_t st) {
  k_merge<<<BHq, 128, 0, st>>>(parts, G, BHq, d, out);
  return cudaGetLastError();
}

}  // namespace wq
