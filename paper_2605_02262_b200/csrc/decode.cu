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

#ifndef WQ_DEC_NCW
#define WQ_DEC_NCW 11
#endif
#ifndef WQ_DEC_RING
#define WQ_DEC_RING 163840
#endif
constexpr int NCW = WQ_DEC_NCW;                 // consumer warps
constexpr int DT = (NCW + 1) * 32;      // threads per CTA
constexpr int MAX_UNITS = 1024;         // B * H
constexpr int64_t MIN_CTA_BYTES = 49152;
#ifndef WQ_DEC_STAGE
#define WQ_DEC_STAGE 32768
#endif
constexpr float LAZY_TH = 8.0f;         // log2 headroom of the lazy softmax rescale
constexpr int KIND_REST = 4;

// Geometry of one unit (request b, kv head h).  Work is partitioned across CTAs in
// COST space, not bytes: every item costs its bytes plus a per-item compute term
// (a window's dequant + MMA work is nearly independent of its width), so CTAs that
// get many narrow windows get fewer of them.  kappa ~ bytes the HBM delivers to
// one SM while it computes one window (0.75 B per element of a quantized window).
struct UnitGeo {
  int b, h, nslots, rl, ntiles;
  int so[5];
  int64_t cs[5];                        // byte start of each class segment; cs[4] = image bytes
  int64_t cc[5];                        // cost start of each class segment; cc[4] = windows' cost
};

WQ_DEV int64_t item_cost(int k, int d, int S) {   // k = 0..3 class, 4 = rest tile
  if (k == 4) return 64LL * d + 176LL * d;
  return record_bytes(class_bits(k), d, S) + (k == 3 ? 6LL * S * d : 12LL * S * d);
}

WQ_DEV void unit_geo(const DecodeArgs &a, int u, UnitGeo &g) {
  g.b = u / a.H;
  g.h = u % a.H;
  const int32_t *so = a.seg_off + 5 * g.b;
  for (int k = 0; k < 5; k++) g.so[k] = so[k];
  g.cs[0] = 0;
  g.cc[0] = 0;
  for (int k = 0; k < 4; k++) {
    const int64_t n = g.so[k + 1] - g.so[k];
    g.cs[k + 1] = g.cs[k] + n * record_bytes(class_bits(k), a.d, a.S);
    g.cc[k + 1] = g.cc[k] + n * item_cost(k, a.d, a.S);
  }
  g.nslots = g.so[4];
  g.rl = a.rest_len ? a.rest_len[g.b] : 0;
  g.rl = g.rl < 0 ? 0 : (g.rl > a.R_max ? a.R_max : g.rl);     // defensive: rest_len <= R_max
  g.ntiles = (g.rl + 15) / 16;
}
// Fixed per-unit costs: the unit epilogue (warp merge tree + CTA partial + ticket)
// is charged at the unit's start and the cross-CTA log-sum-exp merge at its end,
// so a CTA that crosses a unit boundary or finishes a unit gets fewer windows.
constexpr int64_t COST_UNIT_HEAD = 0;
constexpr int64_t COST_UNIT_TAIL = 0;
WQ_DEV int64_t unit_cost(const DecodeArgs &a, const UnitGeo &g) {
  return COST_UNIT_HEAD + g.cc[4] + (int64_t)g.ntiles * item_cost(4, a.d, a.S) + COST_UNIT_TAIL;
}

// first item whose start (in cost units, relative to the unit) is >= x
WQ_DEV int first_item(const DecodeArgs &a, const UnitGeo &g, int64_t x) {
  x -= COST_UNIT_HEAD;
  if (x <= 0) return 0;
  for (int k = 0; k < 4; k++) {
    if (x <= g.cc[k]) return g.so[k];
    if (x < g.cc[k + 1]) {
      const int64_t c = item_cost(k, a.d, a.S);
      return g.so[k] + (int)((x - g.cc[k] + c - 1) / c);
    }
  }
  if (x <= g.cc[4]) return g.nslots;
  const int64_t tc = item_cost(4, a.d, a.S);
  const int64_t t = (x - g.cc[4] + tc - 1) / tc;
  return g.nslots + (int)(t < g.ntiles ? t : g.ntiles);
}

// Stage plan of one unit's item range [i0, i1): five "pieces" (the width-class
// segments 2|4|8|16 and the FP16 rest tiles), each cut into stages of cap
// equal-size items.  Producer and consumers evaluate the same arithmetic, so no
// per-item descriptors are exchanged.
struct UnitPlan {
  int lo[5], hi[5], cap[5], nst[5];
  int sz[5];
};
// The unit the consumers work on, published in shared memory by warp 0 (keeps
// the plan out of the per-thread registers of the window loop).
struct UnitSm {
  int u, n_u, sg_base, rl, nslots, tag;
  int len[5], nst[5], cap[5], lo[5], sz[5];
  float rcap[5];                        // 1 / cap (exact integer division for idx < 2^20)
  int c0, c1;                           // CTAs sharing this unit
};

template <int STAGE>
WQ_DEV void plan_unit(const DecodeArgs &a, const UnitGeo &g, int i0, int i1, UnitPlan &pl) {
  for (int p = 0; p < 5; p++) {
    const int a0 = p < 4 ? g.so[p] : g.nslots;
    const int a1 = p < 4 ? g.so[p + 1] : g.nslots + g.ntiles;
    const int lo = i0 > a0 ? i0 : a0;
    const int hi = i1 < a1 ? i1 : a1;
    const int sz = p < 4 ? (int)record_bytes(class_bits(p), a.d, a.S) : 32 * (2 * a.d + 16);
    pl.lo[p] = lo;
    pl.hi[p] = hi > lo ? hi : lo;
    pl.sz[p] = sz;
    pl.cap[p] = STAGE / sz;
    pl.nst[p] = (pl.hi[p] - pl.lo[p] + pl.cap[p] - 1) / pl.cap[p];
  }
}

WQ_DEV int64_t cta_lo(int c, int G, int64_t T) { return (int64_t)c * T / G; }

// CTAs [c0, c1) that share unit u.  With at least as many units as CTAs, whole
// units go to the CTA owning their cost midpoint (no cross-CTA merge); with fewer
// units, every unit gets 1 + its cost share of the remaining CTAs, so no CTA
// ever spans two split units (one epilogue per CTA).
WQ_DEV void unit_ctas(int u, int U, int G, int64_t T, const int64_t *ustart, int &c0, int &c1) {
  if (T <= 0) { c0 = 0; c1 = 1; return; }
  if (U >= G) {
    const int64_t mid = ustart[u] + (ustart[u + 1] - ustart[u]) / 2;
    c0 = (int)((mid * G) / T);
    if (c0 >= G) c0 = G - 1;
    c1 = c0 + 1;
  } else {
    const int64_t extra = G - U;
    c0 = u + (int)((ustart[u] * extra + T / 2) / T);
    c1 = (u + 1 < U) ? (u + 1) + (int)((ustart[u + 1] * extra + T / 2) / T) : G;
  }
}
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
// Exact fp16 value pair of pair-slot P (compile-time after unrolling) of a lane chunk.
template <int BITS>
WQ_DEV uint32_t deq_pair(const uint32_t *wd, int P) {
  constexpr int PPW = 16 / BITS;
  const uint32_t w = wd[P / PPW];
  if constexpr (BITS == 16) {
    return w;
  } else if constexpr (BITS == 8) {
    return (P % 2) == 0 ? dq_pair<8, 0>(w, 0) : dq_pair<8, 1>(w, 0);
  } else if constexpr (BITS == 4) {
    const uint32_t w8 = w >> 8;
    switch (P % 4) {
      case 0: return dq_pair<4, 0>(w, w8);
      case 1: return dq_pair<4, 1>(w, w8);
      case 2: return dq_pair<4, 2>(w, w8);
      default: return dq_pair<4, 3>(w, w8);
    }
  } else {
    const uint32_t w8 = w >> 8;
    switch (P % 8) {
      case 0: return dq_pair<2, 0>(w, w8);
      case 1: return dq_pair<2, 1>(w, w8);
      case 2: return dq_pair<2, 2>(w, w8);
      case 3: return dq_pair<2, 3>(w, w8);
      case 4: return dq_pair<2, 4>(w, w8);
      case 5: return dq_pair<2, 5>(w, w8);
      case 6: return dq_pair<2, 6>(w, w8);
      default: return dq_pair<2, 7>(w, w8);
    }
  }
}

// Load a lane's chunk of one code tile (D*BITS/16 bytes) into words.
template <int D, int BITS>
WQ_DEV void load_chunk(uint32_t (&wd)[D * BITS / 64], const uint8_t *tile, int lane) {
  constexpr int WPL = D * BITS / 64;
  if constexpr (WPL >= 4) {
    // D-1: 16-byte groups interleaved across lanes (conflict-free LDS.128)
    const uint8_t *ch = tile + lane * 16;
#pragma unroll
    for (int i = 0; i < WPL / 4; i++) {
      uint4 v = lds128(ch + 512 * i);
      wd[4 * i] = v.x; wd[4 * i + 1] = v.y; wd[4 * i + 2] = v.z; wd[4 * i + 3] = v.w;
    }
  } else {
    uint2 v = lds64(tile + lane * (D * BITS / 16));
    wd[0] = v.x; wd[1] = v.y;
  }
}

// V side of one tile: o[mt] += Vcode^T(16 ch x 16 tok) * P'(16 tok x 8 heads)
template <int D, int BITS>
WQ_DEV void tile_pv(const uint32_t (&wd)[D * BITS / 64], uint32_t pb0, uint32_t pb1, float (&o)[D / 16][4]) {
  constexpr int KT = D / 16;
#pragma unroll
  for (int mt = 0; mt < KT; mt++) {
    uint32_t a[4];
#pragma unroll
    for (int r = 0; r < 4; r++) a[r] = deq_pair<BITS>(wd, 4 * mt + r);
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
  const float m0 = st.m[0] == -INFINITY ? 0.f : st.m[0];
  const float m1 = st.m[1] == -INFINITY ? 0.f : st.m[1];
#pragma unroll
  for (int nt = 0; nt < NT; nt++) {
    float p0 = exp2f(s[nt][0] - m0);
    float p1 = exp2f(s[nt][1] - m1);
    float p2 = exp2f(s[nt][2] - m0);
    float p3 = exp2f(s[nt][3] - m1);
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

// One window, processed in chunks of CH 16-token tiles.  Per k-tile the channel
// scales/zero points are read once, q' = q*s is formed as an fp16 hi+lo pair
// (HMUL2 + exact-residual HFMA2) and the bias q.mn accumulates on the tensor core;
// each tile keeps independent hi/lo accumulators (short dependency chains).
template <int D, int S, int BITS>
WQ_DEV void do_window(const uint8_t *rec, const uint32_t (&qf)[D / 16][2], float scale2,
                      WarpState &st, float (&o)[D / 16][4], uint8_t *scratch, int lane) {
  constexpr int NTT = S / 16;
  constexpr int CH = (BITS == 16 || NTT < 2) ? 1 : 2;
  constexpr int KT = D / 16;
  constexpr int WPL = D * BITS / 64;
  constexpr int TILE = 2 * D * BITS;          // bytes of one 16-token code tile
  const uint8_t *kcodes = rec;
  const uint8_t *vcodes = rec + S * D * BITS / 8;
  const uint8_t *kp = rec + 2 * (S * D * BITS / 8);
  const int g = lane >> 2, q = lane & 3;
  float b0[4] = {0.f, 0.f, 0.f, 0.f}, b1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c0 = 0; c0 < NTT; c0 += CH) {
    uint32_t wk[CH][WPL];
#pragma unroll
    for (int t = 0; t < CH; t++) load_chunk<D, BITS>(wk[t], kcodes + (c0 + t) * TILE, lane);
    float ah[CH][4], al[CH][4];
#pragma unroll
    for (int t = 0; t < CH; t++)
#pragma unroll
      for (int i = 0; i < 4; i++) { ah[t][i] = 0.f; al[t][i] = 0.f; }
#pragma unroll
    for (int kt = 0; kt < KT; kt++) {
      uint32_t h0, h1, l0, l1;
      if constexpr (BITS < 16) {
        const uint4 pr = lds128(kp + (q * KT + kt) * 16);   // {s01, s89, mn01, mn89}
        if (c0 == 0) {
          const uint32_t am[4] = {pr.z, pr.z, pr.w, pr.w};
          if (kt & 1) mma16816(b1, am, qf[kt][0], qf[kt][1], b1);
          else mma16816(b0, am, qf[kt][0], qf[kt][1], b0);
        }
        h0 = hmul2u(qf[kt][0], pr.x);
        l0 = h2u(__hfma2(u2h(qf[kt][0]), u2h(pr.x), __hneg2(u2h(h0))));
        h1 = hmul2u(qf[kt][1], pr.y);
        l1 = h2u(__hfma2(u2h(qf[kt][1]), u2h(pr.y), __hneg2(u2h(h1))));
      }
#pragma unroll
      for (int t = 0; t < CH; t++) {
        uint32_t a[4];
#pragma unroll
        for (int r = 0; r < 4; r++) a[r] = deq_pair<BITS>(wk[t], 4 * kt + r);
        if constexpr (BITS < 16) {
          mma16816(ah[t], a, h0, h1, ah[t]);
          mma16816(al[t], a, l0, l1, al[t]);
        } else {
          if (kt & 1) mma16816(al[t], a, qf[kt][0], qf[kt][1], al[t]);
          else mma16816(ah[t], a, qf[kt][0], qf[kt][1], ah[t]);
        }
      }
    }
    float sc[CH][4];
#pragma unroll
    for (int t = 0; t < CH; t++)
#pragma unroll
      for (int i = 0; i < 4; i++) sc[t][i] = ((ah[t][i] + al[t][i]) + (b0[i] + b1[i])) * scale2;
    float vs[CH][2], vm[CH][2];
    if constexpr (BITS < 16) {
      const uint8_t *vp = kp + 4 * D;
#pragma unroll
      for (int t = 0; t < CH; t++) {
        // group (tile, g/2): {s(t0),s(t0+1)}, {s(t0+8),s(t0+9)}, {mn..}, {mn..}; token g = t0 + (g&1)
        const uint4 pr = lds128(vp + (4 * (c0 + t) + (g >> 1)) * 16);
        const uint32_t sh = (g & 1) * 16;
        vs[t][0] = __half2float(__ushort_as_half((unsigned short)(pr.x >> sh)));
        vs[t][1] = __half2float(__ushort_as_half((unsigned short)(pr.y >> sh)));
        vm[t][0] = __half2float(__ushort_as_half((unsigned short)(pr.z >> sh)));
        vm[t][1] = __half2float(__ushort_as_half((unsigned short)(pr.w >> sh)));
      }
    }
    softmax_tiles<CH, KT>(sc, st, o, vs, vm, BITS < 16, scratch, lane);
#pragma unroll
    for (int t = 0; t < CH; t++) {
      uint32_t pb[2];
      // lanes 0-7: tokens 16t+0..7, lanes 8-15: tokens 16t+8..15 (rows of 16 B)
      ldsm_x2_t(pb, scratch + (16 * t + (lane & 15)) * 16);
      uint32_t wv[WPL];
      load_chunk<D, BITS>(wv, vcodes + (c0 + t) * TILE, lane);
      tile_pv<D, BITS>(wv, pb[0], pb[1], o);
    }
    __syncwarp();
  }
}

// FP16 rest tile: K rows [16][D] at base, V rows [16][D] after them, rows padded to 2D+16 bytes
template <int D>
WQ_DEV void do_rest(const uint8_t *base, int ntok, const uint32_t (&qf)[D / 16][2], float scale2,
                    WarpState &st, float (&o)[D / 16][4], uint8_t *scratch, int lane) {
  constexpr int KT = D / 16;
  constexpr int RPH = D + 8;                       // padded row stride (halves)
  const __half *Ks = reinterpret_cast<const __half *>(base);
  const __half *Vs = Ks + 16 * RPH;
  const int g = lane >> 2, q = lane & 3, mi = lane >> 3, rr = lane & 7;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int kt = 0; kt < KT; kt++) {
    uint32_t a[4];
    ldsm_x4(a, Ks + ((mi & 1) * 8 + rr) * RPH + 16 * kt + (mi >> 1) * 8);
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
    ldsm_x4_t(a, Vs + ((mi >> 1) * 8 + rr) * RPH + 16 * mt + (mi & 1) * 8);
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
  // a stage must hold the largest item (an FP16 window: 4*S*D bytes); small stages
  // release shared memory item-group by item-group, a deep ring gives lookahead.
  static constexpr int STAGE = (4 * S * D > WQ_DEC_STAGE) ? 4 * S * D : WQ_DEC_STAGE;
  static constexpr int RING = WQ_DEC_RING;
  static constexpr int NST = (RING / STAGE) < 2 ? 2 : RING / STAGE;
  static constexpr int KT = D / 16;
  static constexpr int SCRATCH = 2 * 16 * 16;            // P' rows of one 2-tile chunk per warp
  // epilogue: every warp's o as [8 heads][D] + (m, l, vb)[8]; 1200+ floats reused by
  // the cross-CTA merge of the last CTA
  static constexpr int EPW = 8 * D + 24;
  static constexpr int EP_SLOTS = NCW;
  static constexpr size_t ring = (size_t)NST * STAGE;
  static constexpr size_t scratch_off = ring;
  static constexpr size_t ep_off = scratch_off + (size_t)NCW * SCRATCH;
  static constexpr size_t units_off = ep_off + (size_t)EP_SLOTS * EPW * 4;
  static constexpr size_t cnt_off = units_off + (size_t)(MAX_UNITS + 1) * 8;
  static constexpr size_t usm_off = (cnt_off + (size_t)(3 * NST + 4) * 4 + 15) / 16 * 16;
  static constexpr int NUS = 4;                          // unit-plan ring published by the producer
  static constexpr size_t bar_off = usm_off + NUS * sizeof(UnitSm);
  static constexpr size_t total = bar_off + 2 * NST * 8 + 16;
};

WQ_DEV uint64_t gtime() {      // profiling clock: SM cycles scaled to ~ns at 1.965 GHz
  return (uint64_t)((double)clock64() * (1.0 / 1.965));
}

WQ_DEV void mbar_wait_sleep(uint64_t *b, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}

template <int D, int S>
__global__ void __launch_bounds__(DT, 1) k_decode(DecodeArgs a) {
  using SM = DecodeSmem<D, S>;
  constexpr int KT = D / 16;
  constexpr int NST = SM::NST;
  constexpr int STAGE = SM::STAGE;
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t *ring = sm;
  int64_t *ustart = reinterpret_cast<int64_t *>(sm + SM::units_off);
  int *stage_n = reinterpret_cast<int *>(sm + SM::cnt_off);      // items per stage fill
  int *stage_done = stage_n + NST;                                // completed items per stage
  int *stage_fill = stage_done + NST;                             // fill number a slot holds
  int *claim = stage_fill + NST;                                  // [2] per-unit claim counters
  int *s_flag = claim + 2;
  int *units_done = s_flag + 1;
  UnitSm *usm = reinterpret_cast<UnitSm *>(sm + SM::usm_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + SM::bar_off);
  uint64_t *empty = full + NST;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int U = a.B * a.H;
  uint64_t *ts = a.ws_ts ? a.ws_ts + (size_t)blockIdx.x * 72 : nullptr;
  if (ts && tid == 0) ts[0] = gtime();

  // ---- unit byte prefix (warp 0) ----
  if (warp == 0) {
    int64_t carry = 0;
    for (int base = 0; base < U; base += 32) {
      int u = base + lane;
      int64_t v = 0;
      if (u < U) {
        UnitGeo gg;
        unit_geo(a, u, gg);
        v = unit_cost(a, gg);
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
      mbar_init(&empty[s], 1);
      stage_n[s] = 0;
      stage_done[s] = 0;
      stage_fill[s] = -1;
    }
    claim[0] = claim[1] = 0;
    *units_done = 0;
    for (int i = 0; i < SM::NUS; i++) usm[i].tag = -1;
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t T = ustart[U];
  int G = (int)(T / MIN_CTA_BYTES);
  G = G < 1 ? 1 : (G > (int)gridDim.x ? (int)gridDim.x : G);
  const int c = blockIdx.x;
  if (c >= G) return;
  if (ts && tid == 0) ts[1] = gtime();

  if (warp == NCW) {
    // =========================== producer ===========================
    // One elected lane walks the stage plan: per stage, wait until the ring slot
    // is free, arm the tx bytes and issue one bulk copy (a run of equal-size
    // records) or two per FP16 rest tile.
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const bool nocopy = (a.debug & 2) != 0;
      int sg = 0;                                  // global stage number of this CTA
      int uix = 0;                                 // index of the unit among this CTA's units
      // publish a unit plan for the consumers (ring of NUS slots, tag written last)
      auto publish = [&](int u, int n_u, const UnitGeo *gg, const UnitPlan *pl, int c0, int c1) {
        while (*reinterpret_cast<volatile int *>(units_done) < uix - (SM::NUS - 1)) {
        }
        UnitSm &d = usm[uix % SM::NUS];
        d.u = u;
        d.n_u = n_u;
        d.sg_base = sg;
        d.c0 = c0;
        d.c1 = c1;
        d.rl = gg ? gg->rl : 0;
        d.nslots = gg ? gg->nslots : 0;
        for (int pp = 0; pp < 5; pp++) {
          d.len[pp] = pl ? pl->hi[pp] - pl->lo[pp] : 0;
          d.nst[pp] = pl ? pl->nst[pp] : 0;
          d.cap[pp] = pl ? pl->cap[pp] : 1;
          d.rcap[pp] = 1.0f / (float)d.cap[pp];
          d.lo[pp] = pl ? pl->lo[pp] : 0;
          d.sz[pp] = pl ? pl->sz[pp] : 0;
        }
        __threadfence_block();
        *reinterpret_cast<volatile int *>(&d.tag) = uix;
        uix++;
      };
      for (int u = 0; u < U; u++) {
        int c0, c1;
        unit_ctas(u, U, G, T, ustart, c0, c1);
        if (c < c0 || c >= c1) continue;
        const int64_t us = ustart[u], ue = ustart[u + 1];
        if (ue <= us) {
          publish(u, 0, nullptr, nullptr, c0, c1);
          continue;
        }
        UnitGeo gg;
        unit_geo(a, u, gg);
        const int nitems = gg.nslots + gg.ntiles;
        const int64_t ucost = ue - us, k = c - c0, n = c1 - c0;
        const int i0 = first_item(a, gg, k * ucost / n);
        const int i1 = (k == n - 1) ? nitems : first_item(a, gg, (k + 1) * ucost / n);
        UnitPlan pl;
        plan_unit<STAGE>(a, gg, i0, i1, pl);
        publish(u, i1 - i0, &gg, &pl, c0, c1);
        const uint8_t *img = a.packed + a.offs[u];
        const __half *kr = a.k_rest + gg.b * a.rs_b + gg.h * a.rs_h;
        const __half *vr = a.v_rest + gg.b * a.rs_b + gg.h * a.rs_h;
        for (int p = 0; p < 5; p++) {
          for (int t = 0; t < pl.nst[p]; t++, sg++) {
            const int slot = sg % NST;
            const uint32_t fill = (uint32_t)(sg / NST);
            const int f0 = pl.lo[p] + t * pl.cap[p];
            const int f1 = min(pl.hi[p], f0 + pl.cap[p]);
            mbar_wait(&empty[slot], (fill & 1) ^ 1);
            stage_n[slot] = f1 - f0;
            *reinterpret_cast<volatile int *>(stage_fill + slot) = (int)fill;
            uint8_t *dst = ring + (size_t)slot * STAGE;
            if (nocopy) {
              mbar_arrive(&full[slot]);
            } else if (p < 4) {
              const uint32_t nb = (uint32_t)(f1 - f0) * pl.sz[p];
              mbar_arrive_expect_tx(&full[slot], nb);
              bulk_g2s_evict_first(dst, img + gg.cs[p] + (int64_t)(f0 - gg.so[p]) * pl.sz[p], nb, &full[slot], pol);
            } else {
              uint32_t tx = 0;
              for (int i = f0; i < f1; i++) tx += (uint32_t)min(16, gg.rl - 16 * (i - gg.nslots)) * 4u * D;
              mbar_arrive_expect_tx(&full[slot], tx);
              // FP16 rest rows land in padded rows (stride 2D+16 B) so the ldmatrix
              // reads of do_rest are bank-conflict free
              constexpr int RP = 2 * D + 16;
              for (int i = f0; i < f1; i++) {
                const int t0 = 16 * (i - gg.nslots);
                const int nt = min(16, gg.rl - t0);
                uint8_t *d2 = dst + (size_t)(i - f0) * pl.sz[4];
                for (int r = 0; r < nt; r++) {
                  bulk_g2s_evict_first(d2 + r * RP, kr + (int64_t)(t0 + r) * D, 2 * D, &full[slot], pol);
                  bulk_g2s_evict_first(d2 + (16 + r) * RP, vr + (int64_t)(t0 + r) * D, 2 * D, &full[slot], pol);
                }
              }
            }
          }
        }
      }
      publish(-1, 0, nullptr, nullptr, 0, 1);     // terminator
      if (ts) ts[2] = gtime();
    }
    return;
  }

  // =========================== consumers ===========================
  // Units in the same order as the producer; items of a unit are claimed
  // dynamically (shared-memory ticket), so faster warps take more windows.
  uint8_t *scratch = sm + SM::scratch_off + warp * SM::SCRATCH;
  float *ep = reinterpret_cast<float *>(sm + SM::ep_off);
  const int g = lane >> 2, q = lane & 3;
  uint32_t qf[KT][2];
  float o[KT][4];
  WarpState st;
  int uidx = 0;
  uint64_t acc_tag = 0, acc_full = 0, acc_comp = 0, t_ep = 0;
  for (;;) {
    const UnitSm &U_ = usm[uidx % SM::NUS];
    while (*reinterpret_cast<const volatile int *>(&U_.tag) != uidx) {
    }
    __threadfence_block();
    const int u = *reinterpret_cast<const volatile int *>(&U_.u);
    if (u < 0) break;
    const int n_u = U_.n_u;
    const int sg_base = U_.sg_base;
    const int cf = U_.c0, cl = U_.c1 - 1;
    const int b = u / a.H, h = u % a.H;
    {
      const __half *qrow = a.q + ((int64_t)b * a.Hq + h * a.grp + g) * D;
#pragma unroll
      for (int kt = 0; kt < KT; kt++) {
        qf[kt][0] = g < a.grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q) : 0u;
        qf[kt][1] = g < a.grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q + 8) : 0u;
      }
    }
#pragma unroll
    for (int mt = 0; mt < KT; mt++) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    st.m[0] = st.m[1] = -INFINITY;
    st.l[0] = st.l[1] = st.vb[0] = st.vb[1] = 0.f;
    int *cl_ctr = claim + (uidx & 1);
    int j = 0;
    if (lane == 0) j = atomicAdd(cl_ctr, 1);
    j = __shfl_sync(0xffffffffu, j, 0);
    for (;;) {
      uint64_t t_a = ts ? gtime() : 0;
      if (j >= n_u) break;
      // claim the next item now; its ticket is only needed after this window
      int jn = 0;
      if (lane == 0) jn = atomicAdd(cl_ctr, 1);
      // locate item j of the unit in the stage plan (shared-memory plan)
      int p = 0, sbase = sg_base, idx = j;
      while (idx >= U_.len[p]) { idx -= U_.len[p]; sbase += U_.nst[p]; p++; }
      const int cap = U_.cap[p];
      const int qs = (int)(((float)idx + 0.5f) * U_.rcap[p]);   // idx / cap
      const int sgi = sbase + qs;
      const int es = sgi % NST;
      const int fill = sgi / NST;
      const uint32_t par = (uint32_t)fill & 1u;
      const int kind = p;
      const int ii = U_.lo[p] + idx;
      const int ntok = p == 4 ? min(16, U_.rl - 16 * (ii - U_.nslots)) : 0;
      const uint8_t *rec = ring + (size_t)es * STAGE + (size_t)(idx - qs * cap) * U_.sz[p];
      uint64_t t_b = ts ? gtime() : 0;
      // the slot must be on this fill before its parity is meaningful (a claim can
      // run more than one ring lap ahead of a slot that is still loading)
      while (*reinterpret_cast<volatile int *>(stage_fill + es) < fill) {
      }
      mbar_wait(&full[es], par);
      uint64_t t_c = ts ? gtime() : 0;
      if (ts) { acc_tag += t_b - t_a; acc_full += t_c - t_b; }
      if (a.debug & 1) {
        st.l[0] += (float)lds32(rec + 16 * lane);
      } else switch (kind) {
        case 0: do_window<D, S, 2>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        case 1: do_window<D, S, 4>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        case 2: do_window<D, S, 8>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        case 3: do_window<D, S, 16>(rec, qf, a.scale_log2, st, o, scratch, lane); break;
        default: do_rest<D>(rec, ntok, qf, a.scale_log2, st, o, scratch, lane); break;
      }
      __syncwarp();
      jn = __shfl_sync(0xffffffffu, jn, 0);
      if (ts) {
        const uint64_t dt = gtime() - t_c;
        acc_comp += dt;
        if (lane == 0) {
          atomicAdd(reinterpret_cast<unsigned long long *>(ts + 56 + kind), (unsigned long long)dt);
          atomicAdd(reinterpret_cast<unsigned long long *>(ts + 61 + kind), 1ull);
        }
      }
      if (lane == 0) {
        const int nd = atomicAdd(stage_done + es, 1) + 1;
        if (nd == *reinterpret_cast<volatile int *>(stage_n + es)) {
          stage_done[es] = 0;
          mbar_arrive(&empty[es]);
        }
      }
      j = jn;
    }
    if (ts && tid == 0) ts[3] = gtime();
    const uint64_t t_e0 = ts ? gtime() : 0;

    // ---------------- unit epilogue: merge tree over the warps ----------------
    named_bar_sync(1, NCW * 32);
    const uint64_t t_e1 = ts ? gtime() : 0;
    uint64_t t_e2 = 0, t_e3 = 0;
    if (tid == 0) claim[uidx & 1] = 0;            // reused by the unit after next
    uidx++;
    {
      // every warp parks its state (l, vb reduced over the 8 lanes of a head pair)
      for (int off = 4; off <= 16; off <<= 1) {
        st.l[0] += __shfl_xor_sync(0xffffffffu, st.l[0], off);
        st.l[1] += __shfl_xor_sync(0xffffffffu, st.l[1], off);
        st.vb[0] += __shfl_xor_sync(0xffffffffu, st.vb[0], off);
        st.vb[1] += __shfl_xor_sync(0xffffffffu, st.vb[1], off);
      }
      float *mine = ep + warp * SM::EPW;           // [8][D] o, then m[8], l[8], vb[8]
#pragma unroll
      for (int mt = 0; mt < KT; mt++) {
        mine[(2 * q) * D + 16 * mt + g] = o[mt][0];
        mine[(2 * q + 1) * D + 16 * mt + g] = o[mt][1];
        mine[(2 * q) * D + 16 * mt + g + 8] = o[mt][2];
        mine[(2 * q + 1) * D + 16 * mt + g + 8] = o[mt][3];
      }
      if (g == 0) {
        mine[8 * D + 2 * q] = st.m[0]; mine[8 * D + 2 * q + 1] = st.m[1];
        mine[8 * D + 8 + 2 * q] = st.l[0]; mine[8 * D + 8 + 2 * q + 1] = st.l[1];
        mine[8 * D + 16 + 2 * q] = st.vb[0]; mine[8 * D + 16 + 2 * q + 1] = st.vb[1];
      }
      named_bar_sync(1, NCW * 32);
      // per head: M, L and the warp weights f[w] (thread j < grp); weights overwrite m
      float *Mh = reinterpret_cast<float *>(sm + SM::scratch_off);   // [8] M, [8] L (scratch is free now)
      if (tid < a.grp) {
        const int j = tid;
        float M = -INFINITY;
        for (int w = 0; w < NCW; w++) M = fmaxf(M, ep[w * SM::EPW + 8 * D + j]);
        float L = 0.f;
        for (int w = 0; w < NCW; w++) {
          float *pw = ep + w * SM::EPW + 8 * D;
          const float f = (M == -INFINITY) ? 0.f : exp2f(pw[j] - M);
          L += f * pw[8 + j];
          pw[j] = f;
        }
        Mh[j] = M;
        Mh[8 + j] = L;
      }
      named_bar_sync(1, NCW * 32);
      t_e2 = ts ? gtime() : 0;
      float *slot = a.ws_part + (int64_t)(c + u) * a.grp * (D + 2);
      // CTA partial (m, l, o + vb) [grp][D + 2], coalesced over channels
      for (int idx = tid; idx < a.grp * D; idx += NCW * 32) {
        const int j = idx / D, cc = idx % D;
        float O = 0.f;
#pragma unroll 5
        for (int w = 0; w < NCW; w++) {
          const float *pw = ep + w * SM::EPW;
          O += pw[8 * D + j] * (pw[j * D + cc] + pw[8 * D + 16 + j]);
        }
        slot[j * (D + 2) + 2 + cc] = O;
        if (cc == 0) { slot[j * (D + 2)] = Mh[j]; slot[j * (D + 2) + 1] = Mh[8 + j]; }
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      named_bar_sync(1, NCW * 32);
      if (tid == 0) {
        const int old = atomicAdd(a.ws_cnt + u, 1);
        *s_flag = (old == cl - cf);
      }
      named_bar_sync(1, NCW * 32);
      t_e3 = ts ? gtime() : 0;
      if (*s_flag) {
        // last CTA of the unit: log-sum-exp merge of the unit's CTA partials.
        // (m, l) of every partial -> per-partial weights in shared memory (reusing
        // the merge-tree buffer), then each thread sums its output columns.
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const int np = cl - cf + 1;
        float *wgt = ep;                              // [np][8] weights, then [8] M, [8] L
        float *Ms = ep + (size_t)np * 8, *Ls = Ms + 8;
        // (m, l) of all partials in one parallel round trip
        for (int t = tid; t < np * 8; t += NCW * 32) {
          const int c2 = t >> 3, j = t & 7;
          float mv = -INFINITY, lv = 0.f;
          if (j < a.grp) {
            const float *sp = a.ws_part + (int64_t)(cf + c2 + u) * a.grp * (D + 2) + j * (D + 2);
            mv = __ldcg(sp);
            lv = __ldcg(sp + 1);
          }
          wgt[t] = mv;
          Ls[8 + t] = lv;                               // scratch: l of partial c2, head j
        }
        named_bar_sync(1, NCW * 32);
        if (tid < a.grp) {
          const int j = tid;
          float M = -INFINITY;
          for (int c2 = 0; c2 < np; c2++) M = fmaxf(M, wgt[c2 * 8 + j]);
          float L = 0.f;
          for (int c2 = 0; c2 < np; c2++) {
            const float f = (M == -INFINITY) ? 0.f : exp2f(wgt[c2 * 8 + j] - M);
            wgt[c2 * 8 + j] = f;
            L += f * Ls[8 + c2 * 8 + j];
          }
          Ms[j] = M;
          Ls[j] = L;
        }
        named_bar_sync(1, NCW * 32);
        for (int idx = tid; idx < a.grp * D; idx += NCW * 32) {
          const int j = idx / D, cc = idx % D;
          float O = 0.f;
          const float *base = a.ws_part + (int64_t)(cf + u) * a.grp * (D + 2) + j * (D + 2) + 2 + cc;
          const int64_t stride = (int64_t)a.grp * (D + 2);
          int c2 = 0;
          for (; c2 + 4 <= np; c2 += 4) {
            const float o0 = __ldcg(base + (c2 + 0) * stride), o1 = __ldcg(base + (c2 + 1) * stride);
            const float o2 = __ldcg(base + (c2 + 2) * stride), o3 = __ldcg(base + (c2 + 3) * stride);
            O += wgt[(c2 + 0) * 8 + j] * o0 + wgt[(c2 + 1) * 8 + j] * o1 + wgt[(c2 + 2) * 8 + j] * o2 +
                 wgt[(c2 + 3) * 8 + j] * o3;
          }
          for (; c2 < np; c2++) O += wgt[c2 * 8 + j] * __ldcg(base + c2 * stride);
          const float L = Ls[j];
          const int64_t row = (int64_t)b * a.Hq + h * a.grp + j;
          if (a.out) a.out[row * D + cc] = __float2half_rn(L > 0.f ? O / L : 0.f);
          if (a.partial) {
            float *pp = a.partial + row * (D + 2);
            if (cc == 0) {
              pp[0] = Ms[j] * 0.69314718055994530942f;   // log2 domain -> natural
              pp[1] = L;
            }
            pp[2 + cc] = O;
          }
        }
        if (tid == 0) a.ws_cnt[u] = 0;
      }
      named_bar_sync(1, NCW * 32);
    }
    if (tid == 0) atomicAdd(units_done, 1);
    if (ts && tid == 0) {
      const uint64_t t_e4 = gtime();
      ts[68] += t_e1 - t_e0; ts[69] += t_e2 - t_e1; ts[70] += t_e3 - t_e2; ts[71] += t_e4 - t_e3;
    }
    if (ts && tid == 0) { ts[4] = gtime(); ts[5] += (uint64_t)n_u; }
    if (ts) t_ep += gtime() - t_e0;
  }
  if (ts && lane == 0) {
    uint64_t *wt = ts + 8 + warp * 4;
    wt[0] = acc_tag; wt[1] = acc_full; wt[2] = acc_comp; wt[3] = t_ep;
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
  size_t cnt = ((size_t)B * H * sizeof(int32_t) + 255) / 256 * 256;
  return part + cnt + (size_t)num_sms * 72 * sizeof(uint64_t);
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
