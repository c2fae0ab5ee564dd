#include <cstdlib>
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
//    mma.sync m16n8k16 (tokens x heads, fp32 accumulate).  2-bit windows instead put
//    the scale on the A side: (code - 2) * s_c in {-2s, -s, 0, s} is exact in fp16, so
//    one MMA against the raw q has exact products (WQ_DEC_K2S).  Codes are loaded in
//    D-1 fragment order straight into MMA A registers and turned into exact fp16
//    integers with one LOP3 + one HSUB2 per pair (magic-exponent trick).  Online
//    softmax per window in the exp2 domain with a lazy rescale (max may run 2^8
//    ahead).  V side: o[c][j] += sum_t (vcode[t][c] - 2^(b-1)) * p'_j[t], p' = p*s_t
//    (centered codes halve the fp16 rounding of p' in the result), the per-token
//    zero point mn_t + s_t*2^(b-1) contributing sum_t p_t*(mn_t + s_t 2^(b-1)) in fp32.
//  * Unit epilogue: warps merged in shared memory, the CTA partial (m, l, o) goes
//    to the workspace, and the last CTA of the unit (atomic ticket) merges all
//    partials by log-sum-exp and writes out / partial (Q24).
#include "decode_common.cuh"

namespace wq {

#ifndef WQ_DEC_NCW
#define WQ_DEC_NCW 11
#endif
#ifndef WQ_DEC_RING
#define WQ_DEC_RING 163840
#endif
constexpr int NCW = WQ_DEC_NCW;                 // consumer warps
constexpr int DT = (NCW + 1) * 32;      // threads per CTA: consumers + the producer warp
#ifndef WQ_DEC_QLO
#define WQ_DEC_QLO 1                     // carry q*s as fp16 hi + lo (0: hi only, experiment)
#endif
#ifndef WQ_DEC_KCENTER
#define WQ_DEC_KCENTER 0                 // 1: centered K codes, q' = q*s in fp16 hi only (no lo MMA); 0: hi + lo
#endif
#ifndef WQ_DEC_K2S
#define WQ_DEC_K2S 1                     // 2-bit K side: A = (code - 2) * s_c (exact in fp16), B = q, one MMA
#endif
#ifndef WQ_DEC_PAIR
#define WQ_DEC_PAIR 0                    // 1: 2-bit windows in pairs (do_window2), S <= 32 (A/B: slower)
#endif
#ifndef WQ_EXP_NOZP
#define WQ_EXP_NOZP 0                    // timing experiments only: skip the zero-point MMA (wrong values)
#endif
#ifndef WQ_DEC_PROFILE
#define WQ_DEC_PROFILE 0                 // per-CTA timestamps into the workspace (debug & 8)
#endif
#ifndef WQ_DEC_STAGE
#define WQ_DEC_STAGE 40960               // stage bytes for S <= 64 (4 stages; 32 KB x 5: C5 32.85 -> 32.64 us,
                                         // C4 106.9 -> 106.5; S = 128 keeps 32 KB: its FP16 records split)
#endif
constexpr float LAZY_TH = 8.0f;         // log2 headroom of the lazy softmax rescale
constexpr int KIND_REST = 4;

struct WarpState {
  float m[2], l[2], vb[2];
};

// -------------------------------------------------------------------------------------
// consumer: one window (BITS in {2,4,8,16}) or one rest tile
// -------------------------------------------------------------------------------------
// V side of one tile: o[mt] += Vcode^T(16 ch x 16 tok) * P'(16 tok x 8 heads)
template <int D, int BITS>
WQ_DEV void tile_pv(const uint32_t (&wd)[D * BITS / 64], uint32_t pb0, uint32_t pb1, float (&o)[D / 16][4]) {
  constexpr int KT = D / 16;
#pragma unroll
  for (int mt = 0; mt < KT; mt++) {
    uint32_t a[4];
#pragma unroll
    for (int r = 0; r < 4; r++) a[r] = deq_pair<BITS, true>(wd, 4 * mt + r);
    mma16816(o[mt], a, pb0, pb1, o[mt]);
  }
}


// Online softmax over NT tiles of raw scores t (logit = t * scale2 in the log2
// domain), writes P' (p * s_t) as fp16 [token][8 heads] rows to the warp scratch.
// The running max is lazy: a tile only triggers the cross-lane max reduction (and a
// rescale) when one of its logits exceeds the current max by LAZY_TH, so most
// windows skip the shuffles (p <= 2^LAZY_TH keeps fp32 sums and fp16 P' in range).
template <int NT, int KT>
WQ_DEV void softmax_tiles(const float (&s)[NT][4], float scale2, WarpState &st, float (&o)[KT][4],
                          const float (&vs)[NT][2], const float (&vm)[NT][2], bool has_vparams,
                          uint8_t *scratch, int lane) {
  const int g = lane >> 2, q = lane & 3;
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < NT; nt++) {
    mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][2]));
    mx1 = fmaxf(mx1, fmaxf(s[nt][1], s[nt][3]));
  }
  mx0 *= scale2;
  mx1 *= scale2;
  const bool up0 = mx0 > st.m[0] + LAZY_TH || (st.m[0] == -INFINITY && mx0 > -INFINITY);
  const bool up1 = mx1 > st.m[1] + LAZY_TH || (st.m[1] == -INFINITY && mx1 > -INFINITY);
  if (__any_sync(0xffffffffu, up0 || up1)) {
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    // uniform over the 8 lanes of a head after the reduction
    const bool n0 = mx0 > st.m[0] + LAZY_TH || (st.m[0] == -INFINITY && mx0 > -INFINITY);
    const bool n1 = mx1 > st.m[1] + LAZY_TH || (st.m[1] == -INFINITY && mx1 > -INFINITY);
    float a0 = 1.f, a1 = 1.f;
    if (n0) { a0 = ex2f(st.m[0] - mx0); st.m[0] = mx0; }
    if (n1) { a1 = ex2f(st.m[1] - mx1); st.m[1] = mx1; }
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
    float p0 = ex2f(fmaf(s[nt][0], scale2, -m0));
    float p1 = ex2f(fmaf(s[nt][1], scale2, -m1));
    float p2 = ex2f(fmaf(s[nt][2], scale2, -m0));
    float p3 = ex2f(fmaf(s[nt][3], scale2, -m1));
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
// GRP (reading Q37, the paper-literal groups of P:508): one (s, mn) per window and tensor, so
// logit = s_K * sum_c code*q_c + mn_K * sum_c q_c: the K side runs on the raw q (no hi/lo
// split, no zero-point MMA; qsum = the lane's heads' sum_c q_c, per unit), and the V side
// takes P' = p * s_V.
// S tokens of a record of SR tokens (SR = S: the whole record): part `part` = tokens
// [part*S, part*S + S) read in place -- its K and V code tiles, the record's K parameters,
// the part's V parameters (large windows are consumed as 32-token parts by several warps).
template <int D, int S, int BITS, bool GRP = false, int SR = S>
WQ_DEV void do_window(const uint8_t *rec, const uint8_t *qs, float scale2,
                      WarpState &st, float (&o)[D / 16][4], uint8_t *scratch, int lane,
                      float2 qsum = make_float2(0.f, 0.f), int part = 0) {
  constexpr int KBR = SR * D * BITS / 8;                 // K code bytes of the record
  if constexpr (GRP && BITS < 16) {
    constexpr int NTT = S / 16;
    constexpr int CH = NTT < 2 ? 1 : 2;
    constexpr int KT = D / 16;
    constexpr int WPL = D * BITS / 64;
    constexpr int TILE = 2 * D * BITS;
    constexpr int KB = S * D * BITS / 8;
    const uint8_t *kc = rec + part * KB, *vc = rec + KBR + part * KB;
    const uint2 pg = lds64(rec + 2 * KBR);               // {mn_K, s_K, mn_V, s_V}
    const float mnK = __half2float(__ushort_as_half((unsigned short)pg.x));
    const float sK = __half2float(__ushort_as_half((unsigned short)(pg.x >> 16)));
    const float mnV = __half2float(__ushort_as_half((unsigned short)pg.y));
    const float sV = __half2float(__ushort_as_half((unsigned short)(pg.y >> 16)));
    constexpr float HALF = (float)(1 << (BITS - 1));
    const float bias0 = mnK * qsum.x, bias1 = mnK * qsum.y;
#pragma unroll
    for (int c0 = 0; c0 < NTT; c0 += CH) {
      uint32_t wk[CH][WPL];
#pragma unroll
      for (int t = 0; t < CH; t++) load_chunk<D, BITS>(wk[t], kc + (c0 + t) * TILE, lane);
      float ah[CH][4], al[CH][4];
#pragma unroll
      for (int t = 0; t < CH; t++)
#pragma unroll
        for (int i = 0; i < 4; i++) { ah[t][i] = 0.f; al[t][i] = 0.f; }
#pragma unroll
      for (int kt = 0; kt < KT; kt++) {
        const uint2 qk = lds64(qs + (kt * 32 + lane) * 8);
#pragma unroll
        for (int t = 0; t < CH; t++) {
          uint32_t a[4];
#pragma unroll
          for (int r = 0; r < 4; r++) a[r] = deq_pair<BITS>(wk[t], 4 * kt + r);
          if (kt & 1) mma16816(al[t], a, qk.x, qk.y, al[t]);
          else mma16816(ah[t], a, qk.x, qk.y, ah[t]);
        }
      }
      float sc[CH][4], vs[CH][2], vm[CH][2];
#pragma unroll
      for (int t = 0; t < CH; t++) {
#pragma unroll
        for (int i = 0; i < 4; i++) sc[t][i] = fmaf(sK, ah[t][i] + al[t][i], (i & 1) ? bias1 : bias0);
        vs[t][0] = vs[t][1] = sV;
        vm[t][0] = vm[t][1] = fmaf(sV, HALF, mnV);
      }
      softmax_tiles<CH, KT>(sc, scale2, st, o, vs, vm, true, scratch, lane);
#pragma unroll
      for (int t = 0; t < CH; t++) {
        uint32_t pb[2];
        ldsm_x2_t(pb, scratch + (16 * t + (lane & 15)) * 16);
        uint32_t wv[WPL];
        load_chunk<D, BITS>(wv, vc + (c0 + t) * TILE, lane);
        tile_pv<D, BITS>(wv, pb[0], pb[1], o);
      }
      __syncwarp();
    }
    return;
  }
  constexpr int NTT = S / 16;
  constexpr int CH = (BITS == 16 || NTT < 2) ? 1 : 2;
  constexpr int KT = D / 16;
  constexpr int WPL = D * BITS / 64;
  constexpr int TILE = 2 * D * BITS;          // bytes of one 16-token code tile
  const uint8_t *kcodes = rec + part * (S * D * BITS / 8);
  const uint8_t *vcodes = rec + KBR + part * (S * D * BITS / 8);
  const uint8_t *kp = rec + 2 * KBR;
  const int g = lane >> 2, q = lane & 3;
  // K2: 2-bit windows carry the channel scale on the A side: (code - 2) * s_c is one of
  // {-2s, -s, 0, s}, exact in fp16, so one MMA against the raw q gives exact products
  // (no hi/lo split of q * s_c); the centering adds 2 * sum_c q_c s_c (zero-point rows g + 8).
  constexpr bool K2 = (BITS == 2) && (WQ_DEC_K2S != 0);
  constexpr bool KC = K2 || (WQ_DEC_KCENTER != 0 && BITS < 16);
  constexpr bool LO = (BITS < 16) && !KC && (WQ_DEC_QLO != 0);
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
      const uint2 qk = lds64(qs + (kt * 32 + lane) * 8);   // q fragment (B operand) of k-tile kt
      uint32_t h0 = 0, h1 = 0, l0 = 0, l1 = 0;
      if constexpr (BITS < 16) {
        // {mn01, s01, mn89, s89}: the quad is the zero-point term's A fragment as
        // loaded (rows g: mn, rows g+8: don't-care -- only d0/d1 of b0/b1 are used)
        // group (q, kt) at (4 kt + q) * 16: the quads' 4 groups are adjacent 16-byte chunks
        // (conflict-free; the former q-major order was a 4-way conflict, 2 % of a C5 launch)
        const uint4 pr = lds128(kp + (4 * kt + q) * 16);
        if (c0 == 0 && !WQ_EXP_NOZP) {
          const uint32_t am[4] = {pr.x, pr.y, pr.z, pr.w};
          if (kt & 1) mma16816(b1, am, qk.x, qk.y, b1);
          else mma16816(b0, am, qk.x, qk.y, b0);
        }
        if constexpr (K2) {
          h0 = pr.y;                                       // s01, s89: A-side scales
          h1 = pr.w;
        } else {
          h0 = hmul2u(qk.x, pr.y);
          h1 = hmul2u(qk.y, pr.w);
        }
        if constexpr (LO) {
          l0 = h2u(__hfma2(u2h(qk.x), u2h(pr.y), __hneg2(u2h(h0))));
          l1 = h2u(__hfma2(u2h(qk.y), u2h(pr.w), __hneg2(u2h(h1))));
        }
      }
#pragma unroll
      for (int t = 0; t < CH; t++) {
        uint32_t a[4];
#pragma unroll
        for (int r = 0; r < 4; r++) a[r] = deq_pair<BITS, KC>(wk[t], 4 * kt + r);
        if constexpr (K2) {
          // a[0], a[1]: channels 16 kt + 2q, +1 (rows g, g + 8); a[2], a[3]: + 8
          a[0] = hmul2u(a[0], h0); a[1] = hmul2u(a[1], h0);
          a[2] = hmul2u(a[2], h1); a[3] = hmul2u(a[3], h1);
          if (kt & 1) mma16816(al[t], a, qk.x, qk.y, al[t]);
          else mma16816(ah[t], a, qk.x, qk.y, ah[t]);
        } else if constexpr (BITS < 16) {
          if constexpr (LO) {
            mma16816(ah[t], a, h0, h1, ah[t]);
            mma16816(al[t], a, l0, l1, al[t]);
          } else {
            if (kt & 1) mma16816(al[t], a, h0, h1, al[t]);
            else mma16816(ah[t], a, h0, h1, ah[t]);
          }
        } else {
          if (kt & 1) mma16816(al[t], a, qk.x, qk.y, al[t]);
          else mma16816(ah[t], a, qk.x, qk.y, ah[t]);
        }
      }
    }
    float sc[CH][4];
#pragma unroll
    for (int t = 0; t < CH; t++)
#pragma unroll
      for (int i = 0; i < 4; i++) {
        sc[t][i] = (ah[t][i] + al[t][i]) + (b0[i & 1] + b1[i & 1]);
        // centered K codes: + 2^(BITS-1) * sum_c q_c s_c (rows g + 8 of the zero-point MMA)
        if constexpr (KC)
          sc[t][i] += (float)(1 << (BITS - 1)) * (b0[2 + (i & 1)] + b1[2 + (i & 1)]);
      }
    float vs[CH][2], vm[CH][2];
    if constexpr (BITS < 16) {
      const uint8_t *vp = kp + 4 * D + part * 4 * S;
#pragma unroll
      for (int t = 0; t < CH; t++) {
        // group (tile, g/2): {s(t0),s(t0+1)}, {s(t0+8),s(t0+9)}, {mn..}, {mn..}; token g = t0 + (g&1)
        const uint4 pr = lds128(vp + (4 * (c0 + t) + (g >> 1)) * 16);
        const uint32_t sh = (g & 1) * 16;
        vs[t][0] = __half2float(__ushort_as_half((unsigned short)(pr.x >> sh)));
        vs[t][1] = __half2float(__ushort_as_half((unsigned short)(pr.y >> sh)));
        // centered V codes (code - 2^(BITS-1)) move s * 2^(BITS-1) into the fp32 zero-point term
        constexpr float HALF = (float)(1 << (BITS - 1));
        vm[t][0] = fmaf(vs[t][0], HALF, __half2float(__ushort_as_half((unsigned short)(pr.z >> sh))));
        vm[t][1] = fmaf(vs[t][1], HALF, __half2float(__ushort_as_half((unsigned short)(pr.w >> sh))));
      }
    }
    softmax_tiles<CH, KT>(sc, scale2, st, o, vs, vm, BITS < 16, scratch, lane);
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

// Two windows A and B of the same b-bit class (S <= 32) in one pass: their 2*S/16 tiles
// share the k-tile loop (one q fragment load per k-tile, four independent K-side MMA
// chains for S = 32), ONE zero-point MMA per k-tile serves both (A rows g = window A's
// minima, rows g + 8 = window B's: the rows the single-window path leaves unused), and one
// softmax pass covers the pair.  Same products and accumulations per window as do_window.
template <int D, int S, int BITS>
WQ_DEV void do_window2(const uint8_t *recA, const uint8_t *recB, const uint8_t *qs, float scale2,
                       WarpState &st, float (&o)[D / 16][4], uint8_t *scratch, int lane) {
  constexpr int NTT = S / 16;                 // tiles per window (1 or 2)
  constexpr int T = 2 * NTT;                  // tiles of the pair: A's, then B's
  constexpr int KT = D / 16;
  constexpr int WPL = D * BITS / 64;
  constexpr int TILE = 2 * D * BITS;
  constexpr int KB = S * D * BITS / 8;        // K (or V) code bytes of a window
  static_assert(BITS < 16 && NTT >= 1 && NTT <= 2, "pairs of b-bit windows with S <= 32");
  const uint8_t *kpA = recA + 2 * KB, *kpB = recB + 2 * KB;
  const int g = lane >> 2, q = lane & 3;
  uint32_t wk[T][WPL];
#pragma unroll
  for (int t = 0; t < NTT; t++) {
    load_chunk<D, BITS>(wk[t], recA + t * TILE, lane);
    load_chunk<D, BITS>(wk[NTT + t], recB + t * TILE, lane);
  }
  float ah[T][4], al[T][4];
  float b0[4] = {0.f, 0.f, 0.f, 0.f}, b1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int t = 0; t < T; t++)
#pragma unroll
    for (int i = 0; i < 4; i++) { ah[t][i] = 0.f; al[t][i] = 0.f; }
#pragma unroll
  for (int kt = 0; kt < KT; kt++) {
    const uint2 qk = lds64(qs + (kt * 32 + lane) * 8);
    const uint4 pa = lds128(kpA + (4 * kt + q) * 16);     // {mn01, s01, mn89, s89} of A
    const uint4 pb = lds128(kpB + (4 * kt + q) * 16);     // ... of B
    {
      const uint32_t am[4] = {pa.x, pb.x, pa.z, pb.z};     // rows g: A's minima, rows g + 8: B's
      if (kt & 1) mma16816(b1, am, qk.x, qk.y, b1);
      else mma16816(b0, am, qk.x, qk.y, b0);
    }
    const uint32_t hA0 = hmul2u(qk.x, pa.y), hA1 = hmul2u(qk.y, pa.w);
    const uint32_t lA0 = h2u(__hfma2(u2h(qk.x), u2h(pa.y), __hneg2(u2h(hA0))));
    const uint32_t lA1 = h2u(__hfma2(u2h(qk.y), u2h(pa.w), __hneg2(u2h(hA1))));
    const uint32_t hB0 = hmul2u(qk.x, pb.y), hB1 = hmul2u(qk.y, pb.w);
    const uint32_t lB0 = h2u(__hfma2(u2h(qk.x), u2h(pb.y), __hneg2(u2h(hB0))));
    const uint32_t lB1 = h2u(__hfma2(u2h(qk.y), u2h(pb.w), __hneg2(u2h(hB1))));
#pragma unroll
    for (int t = 0; t < T; t++) {
      uint32_t a[4];
#pragma unroll
      for (int r = 0; r < 4; r++) a[r] = deq_pair<BITS>(wk[t], 4 * kt + r);
      if (t < NTT) {
        mma16816(ah[t], a, hA0, hA1, ah[t]);
        mma16816(al[t], a, lA0, lA1, al[t]);
      } else {
        mma16816(ah[t], a, hB0, hB1, ah[t]);
        mma16816(al[t], a, lB0, lB1, al[t]);
      }
    }
  }
  float sc[T][4];
#pragma unroll
  for (int t = 0; t < T; t++)
#pragma unroll
    for (int i = 0; i < 4; i++)
      sc[t][i] = (ah[t][i] + al[t][i]) + (b0[(t < NTT ? 0 : 2) + (i & 1)] + b1[(t < NTT ? 0 : 2) + (i & 1)]);
  float vs[T][2], vm[T][2];
#pragma unroll
  for (int t = 0; t < T; t++) {
    const uint8_t *vp = (t < NTT ? kpA : kpB) + 4 * D;
    const uint4 pr = lds128(vp + (4 * (t % NTT) + (g >> 1)) * 16);
    const uint32_t sh = (g & 1) * 16;
    vs[t][0] = __half2float(__ushort_as_half((unsigned short)(pr.x >> sh)));
    vs[t][1] = __half2float(__ushort_as_half((unsigned short)(pr.y >> sh)));
    constexpr float HALF = (float)(1 << (BITS - 1));
    vm[t][0] = fmaf(vs[t][0], HALF, __half2float(__ushort_as_half((unsigned short)(pr.z >> sh))));
    vm[t][1] = fmaf(vs[t][1], HALF, __half2float(__ushort_as_half((unsigned short)(pr.w >> sh))));
  }
  softmax_tiles<T, KT>(sc, scale2, st, o, vs, vm, true, scratch, lane);
#pragma unroll
  for (int t = 0; t < T; t++) {
    uint32_t pbv[2];
    ldsm_x2_t(pbv, scratch + (16 * t + (lane & 15)) * 16);
    uint32_t wv[WPL];
    load_chunk<D, BITS>(wv, (t < NTT ? recA : recB) + KB + (t % NTT) * TILE, lane);
    tile_pv<D, BITS>(wv, pbv[0], pbv[1], o);
  }
  __syncwarp();
}

// FP16 rest tile: K rows [16][D] at Kb, V rows [16][D] at Vb (unpadded rows as the
// bulk copies land them; rows past ntok hold stale bytes and are masked)
template <int D>
WQ_DEV void do_rest(const uint8_t *Kb, const uint8_t *Vb, int ntok, const uint8_t *qs, float scale2,
                    WarpState &st, float (&o)[D / 16][4], uint8_t *scratch, int lane) {
  constexpr int KT = D / 16;
  constexpr int RPH = D;                           // row stride (halves)
  const __half *Ks = reinterpret_cast<const __half *>(Kb);
  const __half *Vs = reinterpret_cast<const __half *>(Vb);
  const int g = lane >> 2, q = lane & 3, mi = lane >> 3, rr = lane & 7;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int kt = 0; kt < KT; kt++) {
    const uint2 qk = lds64(qs + (kt * 32 + lane) * 8);
    uint32_t a[4];
    ldsm_x4(a, Ks + ((mi & 1) * 8 + rr) * RPH + 16 * kt + (mi >> 1) * 8);
    mma16816(acc, a, qk.x, qk.y, acc);
  }
  float sc[1][4];
  sc[0][0] = g < ntok ? acc[0] : -INFINITY;
  sc[0][1] = g < ntok ? acc[1] : -INFINITY;
  sc[0][2] = g + 8 < ntok ? acc[2] : -INFINITY;
  sc[0][3] = g + 8 < ntok ? acc[3] : -INFINITY;
  float vs[1][2], vm[1][2];
  softmax_tiles<1, KT>(sc, scale2, st, o, vs, vm, false, scratch, lane);
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
#ifndef WQ_DEC_SUB
#define WQ_DEC_SUB 32                    // records of more tokens are consumed as parts of this many (0: off;
                                         // C4 S=128 185.4 -> 127.8 us, S=64 133.8 -> 127.9)
#endif
// FP16 items per window in reordered mode: 2 when a 64 KB record would leave a 2-stage ring
template <int S>
constexpr int stage_bytes() { return S >= 128 ? 32768 : WQ_DEC_STAGE; }
template <int D, int S>
constexpr int fsplit() { return 4 * S * D >= 2 * stage_bytes<S>() ? 2 : 1; }

template <int D, int S, int FS = 1>
struct DecodeSmem {
  // a stage must hold the largest item: an FP16 window (4*S*D bytes), or an FS-th of it and
  // the largest quantized record when FP16 windows are split (FS > 1, reordered mode only)
  static constexpr int REC8 = S * D * 2 + 4 * D + 4 * S;
  static constexpr int BIG = FS > 1 ? (4 * S * D / FS > REC8 ? 4 * S * D / FS : REC8) : 4 * S * D;
  static constexpr int STAGE = (BIG > stage_bytes<S>()) ? BIG : stage_bytes<S>();
  static constexpr int RING = WQ_DEC_RING;
  static constexpr int NST = (RING / STAGE) < 2 ? 2 : RING / STAGE;
  static constexpr int KT = D / 16;
  static constexpr int SCRATCH = 4 * 16 * 16;            // P' rows of up to 4 tiles per warp
  static constexpr int EPW = 8 * D + 24;                 // per warp: o [KT*32 groups][4], m[8], l[8], vb[8]
  static_assert(SCRATCH <= EPW * 4, "a warp's P' scratch lives in its own epilogue slot");
  static constexpr int PSLOT = 16 + 8 * D;               // floats of a CTA partial in the workspace
  static constexpr int NUS = 4;                          // entry ring published by the producer
  static constexpr size_t ring = (size_t)NST * STAGE;
  static constexpr size_t hw_off = ring;                                       // epilogue head weights
  static constexpr size_t q_off = hw_off + ((size_t)(NCW * 8 + 24) * 4 + 15) / 16 * 16;   // q fragments [KT][32][2]
  static constexpr size_t ep_off = q_off + (size_t)KT * 32 * 8;
  static constexpr size_t units_off = ep_off + (size_t)NCW * EPW * 4;
  static constexpr size_t ent_off = units_off + (size_t)(MAX_UNITS + 1) * 8;
  static constexpr size_t plan_off = ent_off + NUS * sizeof(Entry);
  static constexpr size_t misc_off = plan_off + sizeof(CtaPlan);
  static constexpr size_t bar_off = (misc_off + 16 + 15) / 16 * 16;
  // unreordered mode (UR): per ring slot the producer's item table {n, (offset, class) x n}
  static constexpr int MAXI = (int)(STAGE / (S * D / 2 + 4 * D + 4 * S));   // most records per stage
  static constexpr int TABN = 2 + 2 * MAXI;
  static constexpr size_t tab_off = bar_off + 2 * NST * 8;                    // full, empty barriers
  static constexpr size_t total = tab_off + (size_t)NST * TABN * 4;
  static_assert(total <= 232448, "decode shared memory exceeds the 227 KB opt-in limit");
};

// Producer of the unreordered image (UR): a unit's windows are
// streamed in ORIGINAL order; a stage is the longest run of consecutive records (mixed
// widths, contiguous bytes) that fits, one bulk copy, described to the consumers by a
// table {n, (byte offset, class) per record} written before the stage's full barrier
// arrive (release).  Split units give CTA k of n the windows [W k/n, W (k+1)/n) and the
// last CTA the FP16 rest tiles.
template <int D, int S, int STAGE, int NST, int NUS, int TABN>
WQ_DEV void produce_ur(const DecodeArgs &a, const CtaPlan &P, uint8_t *ring, uint64_t *full, uint64_t *empty,
                       Entry *ent, int *units_done, int *tab, int vc) {
  using IG = ItemGeo<D, S, false>;
  constexpr int MAXI = (TABN - 2) / 2;
  const int c = vc;
  const uint64_t pol = policy_evict_first();
  int sg = 0, uix = 0;
  auto publish = [&](int u, int n_u, int lo0, int len0, int rl, int nslots, int lo4, int len4, int nst4) {
    while (*reinterpret_cast<volatile int *>(units_done) < uix - (NUS - 1)) {
    }
    Entry &d = ent[uix % NUS];
    d.u = u; d.n_u = n_u;
    d.c0 = P.split ? P.c0 : c;
    d.c1 = P.split ? P.c1 : c + 1;
    d.rl = rl; d.nslots = nslots;
#pragma unroll
    for (int pp = 0; pp < 5; pp++) { d.lo[pp] = 0; d.len[pp] = 0; d.nst[pp] = 0; }
    d.lo[0] = lo0; d.len[0] = len0;
    d.lo[4] = lo4; d.len[4] = len4; d.nst[4] = nst4;
    __threadfence_block();
    *reinterpret_cast<volatile int *>(&d.tag) = uix;
    uix++;
  };
  for (int u = P.ua; u < P.ub; u++) {
    UnitGeo gg;
    unit_geo<D, S, false>(a, u, gg);
    const int W = gg.nslots;
    int w0 = 0, w1 = W, t0 = 0, t1 = gg.ntiles;
    if (P.split) {
      const int k = c - P.c0, n = P.c1 - P.c0;
      w0 = (int)((int64_t)W * k / n);
      w1 = (int)((int64_t)W * (k + 1) / n);
      if (k < n - 1) t1 = 0;
    }
    const int cap4 = STAGE / IG::sz(4);
    const int nst4 = (t1 - t0 + cap4 - 1) / cap4;
    publish(u, (w1 - w0) + (t1 - t0), w0, w1 - w0, gg.rl, W, W + t0, t1 - t0, nst4);
    const uint8_t *img = a.packed + a.offs[u];
    const int64_t *wo = a.woff + (int64_t)gg.b * (W + 1);
    for (int w = w0; w < w1;) {
      // the longest run [w, w + n) of records fitting one stage (offsets batch-loaded)
      int64_t o[MAXI + 1];
#pragma unroll
      for (int i = 0; i <= MAXI; i++) o[i] = (w + i <= w1) ? __ldg(wo + w + i) : INT64_MAX;
      int n = 0;
#pragma unroll
      for (int i = 1; i <= MAXI; i++) n += (o[i] - o[0] <= STAGE) ? 1 : 0;
      const int slot = sg % NST;
      mbar_wait_sleep(&empty[slot], ((uint32_t)(sg / NST) & 1u) ^ 1u, 64);
      int *tb = tab + slot * TABN;
      tb[0] = n;
#pragma unroll
      for (int i = 0; i < MAXI; i++) {
        if (i < n) {
          const int64_t rb = o[i + 1] - o[i];
          tb[2 + 2 * i] = (int)(o[i] - o[0]);
          tb[3 + 2 * i] = rb == IG::rb(0) ? 0 : rb == IG::rb(1) ? 1 : rb == IG::rb(2) ? 2 : 3;
        }
      }
      const uint32_t nb = (uint32_t)(o[n] - o[0]);
      WQ_CHECK(n >= 1 && nb <= (uint32_t)STAGE && a.offs[u] + o[n] <= a.offs[u + 1]);
      mbar_arrive_expect_tx(&full[slot], nb);
      bulk_g2s_evict_first(ring + (size_t)slot * STAGE, img + o[0], nb, &full[slot], pol);
      w += n;
      sg++;
    }
    const __half *kr = a.k_rest + gg.b * a.rs_b + gg.h * a.rs_h;
    const __half *vr = a.v_rest + gg.b * a.rs_b + gg.h * a.rs_h;
    for (int t = 0; t < nst4; t++, sg++) {
      const int slot = sg % NST;
      const int f0 = t0 + t * cap4, f1 = min(t1, f0 + cap4);
      mbar_wait_sleep(&empty[slot], ((uint32_t)(sg / NST) & 1u) ^ 1u, 64);
      uint8_t *dst = ring + (size_t)slot * STAGE;
      if (a.flags & WQ_DECODE_EARLY_) griddep_wait();
      const int r0 = 16 * f0, r1 = min(gg.rl, 16 * f1);
      const uint32_t nb = (uint32_t)(r1 - r0) * 2u * D;
      mbar_arrive_expect_tx(&full[slot], 2 * nb);
      bulk_g2s_evict_first(dst, kr + (int64_t)r0 * D, nb, &full[slot], pol);
      bulk_g2s_evict_first(dst + cap4 * 32 * D, vr + (int64_t)r0 * D, nb, &full[slot], pol);
    }
  }
  publish(-1, 0, 0, 0, 0, 0, 0, 0, 0);
}


// ---- fused cross-GPU log-sum-exp merge ----
// Symmetric buffer of every rank (peer_buffer_bytes): [2 parities][G ranks][B*Hq][d+2]
// fp32 partials, then one u32 arrival counter per unit (zero-filled once).  The CTA that
// holds the rank-local final partial of unit u (written to its own slot, a.partial)
// stores the unit's rows into slot [parity][rank] of every peer over NVLink (plain
// stores to IPC-mapped peer memory), releases them system-wide and bumps every peer's
// counter of u; it then waits for its own counter to reach G * epoch (every rank's
// rows of u have landed) and merges the G partials of u by log-sum-exp into out.
// Parity: a rank can run at most one call ahead of a peer (call e+1 of a rank needs
// every rank's rows of e+1), so two parities never collide.
WQ_DEV void red_release_sys_add(uint32_t *p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
WQ_DEV uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int D, int NT>
WQ_DEV void peer_exchange_merge(const DecodeArgs &a, int tid, int u, int b, int h) {
  const int grp = a.grp, G = a.peer_G, r = a.peer_rank;
  const int64_t slotf = (int64_t)a.B * a.Hq * (D + 2);            // floats per (parity, rank) slot
  const int par = (int)(a.peer_epoch & 1u);
  const int64_t row0 = (int64_t)b * a.Hq + h * grp;
  const int nrow = grp * (D + 2);
  named_bar_sync(1, NT);                          // the unit's rows in the own slot are complete
  const float *mine = a.partial + row0 * (D + 2);
  for (int p = 0; p < G; p++) {
    if (p == r) continue;
    float *dst = reinterpret_cast<float *>(a.peer_bufs[p]) + (par * G + r) * slotf + row0 * (D + 2);
    for (int i = tid; i < nrow; i += NT) dst[i] = mine[i];
  }
  __threadfence_system();
  named_bar_sync(1, NT);
  const int64_t ctr_off = 2LL * G * slotf * 4;                    // bytes: counters after the slots
  if (tid == 0) {
    for (int p = 0; p < G; p++) red_release_sys_add(reinterpret_cast<uint32_t *>(a.peer_bufs[p] + ctr_off) + u, 1u);
    const uint32_t *my = reinterpret_cast<const uint32_t *>(a.peer_bufs[r] + ctr_off) + u;
    const uint32_t want = (uint32_t)G * a.peer_epoch;
    // bounded wait (10 s of globaltimer): a peer that never arrives (a rank that skipped
    // the call, a broken mapping) must not hang the GPU; the result is then invalid.
    // The error word after the counters (wq_peer_error_offset) is polled too: once any
    // wait of this rank timed out, every later wait gives up at once instead of burning
    // another 10 s per unit and call.
    uint32_t *err = const_cast<uint32_t *>(my) - u + a.B * a.H;
    const uint64_t t0 = gtime();
    while ((int32_t)(ld_acquire_sys(my) - want) < 0) {
      __nanosleep(64);
      if (ld_acquire_sys(err) != 0u) break;
      if (gtime() - t0 > 10000000000ull) {
        atomicExch(err, 1u);
        break;
      }
    }
  }
  named_bar_sync(1, NT);
  const float *base = reinterpret_cast<const float *>(a.peer_bufs[r]) + par * G * slotf + row0 * (D + 2);
  for (int idx = tid; idx < grp * D; idx += NT) {
    const int j = idx / D, cc = idx - j * D;
    float M = -INFINITY;
    for (int p = 0; p < G; p++) {
      const float *pp = base + p * slotf + j * (D + 2);
      if (__ldcv(pp + 1) > 0.f) M = fmaxf(M, __ldcv(pp));
    }
    float L = 0.f, O = 0.f;
    for (int p = 0; p < G; p++) {
      const float *pp = base + p * slotf + j * (D + 2);
      const float l = __ldcv(pp + 1);
      if (!(l > 0.f)) continue;
      const float f = expf(__ldcv(pp) - M);
      L = fmaf(f, l, L);
      O = fmaf(f, __ldcv(pp + 2 + cc), O);
    }
    a.peer_out[(row0 + j) * D + cc] = __float2half_rn(L > 0.f ? O / L : 0.f);
  }
}

size_t peer_buffer_bytes(int B, int H, int Hq, int d, int G) {
  // slots, then B*H arrival counters and one error word (a timed-out wait sets it)
  return 2ull * G * B * Hq * (d + 2) * sizeof(float) + (((size_t)(B * H + 1) * sizeof(uint32_t) + 255) / 256) * 256;
}

// The kernel body; vc / vn = this CTA's index and the CTA count it plans with
// (blockIdx.x / gridDim.x, or a virtual rank's share of the grid under emulation).
template <int D, int S, bool UR, bool GRP = false>
WQ_DEV void decode_body(const DecodeArgs &a, const int vc, const int vn) {
  constexpr int FS = UR ? 1 : fsplit<D, S>();
  using SM = DecodeSmem<D, S, FS>;
  constexpr int KT = D / 16;
  constexpr int NST = SM::NST;
  constexpr int STAGE = SM::STAGE;
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t *ring = sm;
  int64_t *ustart = reinterpret_cast<int64_t *>(sm + SM::units_off);
  Entry *ent = reinterpret_cast<Entry *>(sm + SM::ent_off);
  int *s_flag = reinterpret_cast<int *>(sm + SM::misc_off);
  int *units_done = s_flag + 1;
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + SM::bar_off);
  uint64_t *empty = full + NST;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int U = a.B * a.H;
  // timestamps only in profiling builds (WQ_DEC_PROFILE=1, tools/dbg_decode_time.py)
  uint64_t *ts = (WQ_DEC_PROFILE && a.ws_ts) ? a.ws_ts + (size_t)vc * TS_PER_CTA : nullptr;
  if (ts && tid == 0) ts[0] = gtime();

  // ---- prologue (warp 0): unit cost prefix, then this CTA's share ----
  CtaPlan *cp = reinterpret_cast<CtaPlan *>(sm + SM::plan_off);
  if (warp == 0) plan_cta<D, S, false, (UR ? 0 : WQ_DEC_STREAM), GRP, FS>(a, ustart, cp, s_flag, lane, vc, vn);
  if (tid == 32) {
    for (int s = 0; s < NST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    *units_done = 0;
    for (int i = 0; i < SM::NUS; i++) ent[i].tag = -1;
    fence_mbar_init();
  }
  __syncthreads();
  const int G = *s_flag;
  const int c = vc;
  // the next launch on the stream may start its prologue and cache prefetch as soon
  // as SMs free up (it waits for this grid before touching q / outputs: PDL)
  if (tid == 0) griddep_launch_dependents();
  if (c >= G) return;
  if (ts && tid == 0) { ts[1] = gtime(); ts[70] = clock64(); }

  if (warp == NCW) {
    // =========================== producer ===========================
    if constexpr (UR) {
      if (lane == 0) produce_ur<D, S, STAGE, NST, SM::NUS, SM::TABN>(a, *cp, ring, full, empty, ent, units_done,
                                                                      reinterpret_cast<int *>(sm + SM::tab_off), vc);
    } else {
      if (lane == 0)
        produce<D, S, false, STAGE, NST, SM::NUS, GRP, FS>(a, *cp, ustart, ring, full, empty, ent, units_done, ts,
                                                           vc);
    }
    return;
  }

  // =========================== consumers ===========================
  float *ep = reinterpret_cast<float *>(sm + SM::ep_off);
  // the warp's P' scratch: the head of its own epilogue slot (dead until it parks there)
  uint8_t *scratch = reinterpret_cast<uint8_t *>(ep + warp * SM::EPW);
  const int g = lane >> 2, q = lane & 3;
  const int grp = a.grp;
  uint8_t *qs = sm + SM::q_off;
  uint32_t qf[KT][2];                             // warp 0: q of the next unit, staged to qs
  float o[KT][4];
  WarpState st;
  int uidx = 0, sg = 0;
  uint64_t acc_wait = 0, acc_comp = 0, t_ep = 0, t_loop = 0;
  // q fragments of a unit (B operand, heads x channels)
  auto load_q = [&](int uq) {
    const int bq = uq / a.H, hq = uq - bq * a.H;
    const __half *qrow = a.q + ((int64_t)bq * a.Hq + hq * grp + g) * D;
#pragma unroll
    for (int kt = 0; kt < KT; kt++) {
      qf[kt][0] = g < grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q) : 0u;
      qf[kt][1] = g < grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q + 8) : 0u;
    }
  };
  // warp 0 stages q of the first unit (cp->ua) while the producer plans and issues
  // the first copy; later entries restage at their start
  auto stage_q = [&](int uq) {
    load_q(uq);
#pragma unroll
    for (int kt = 0; kt < KT; kt++)
      *reinterpret_cast<uint2 *>(qs + (kt * 32 + lane) * 8) = make_uint2(qf[kt][0], qf[kt][1]);
  };
  if (warp == 0 && (a.flags & WQ_DECODE_EARLY_)) griddep_wait();   // q / outputs / workspace
  if (ts && tid == 0) ts[53] = gtime();
  if (warp == 0 && cp->ua < U) stage_q(cp->ua);
  if (ts && tid == 0) ts[54] = gtime();
  for (;;) {
    const Entry &E = ent[uidx % SM::NUS];
    while (*reinterpret_cast<const volatile int *>(&E.tag) != uidx) {
    }
    __threadfence_block();
    const int u = *reinterpret_cast<const volatile int *>(&E.u);
    if (u < 0) break;
    const int c0 = E.c0, c1 = E.c1, rl = E.rl, nslots = E.nslots;
    const int b = u / a.H, h = u % a.H;
    if (warp == 0 && uidx > 0) stage_q(u);        // (entries after the first: unit ua + uidx)
    named_bar_sync(2, NCW * 32);
    // GRP: sum_c q_c of the lane's heads 2q, 2q+1 (one MMA per k-tile with A = ones)
    float2 qsum = make_float2(0.f, 0.f);
    if constexpr (GRP) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const uint32_t ones[4] = {0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u};
#pragma unroll
      for (int kt = 0; kt < KT; kt++) {
        const uint2 qk = lds64(qs + (kt * 32 + lane) * 8);
        mma16816(acc, ones, qk.x, qk.y, acc);
      }
      qsum = make_float2(acc[0], acc[1]);
    }
#pragma unroll
    for (int mt = 0; mt < KT; mt++) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    st.m[0] = st.m[1] = -INFINITY;
    st.l[0] = st.l[1] = st.vb[0] = st.vb[1] = 0.f;

    const uint64_t t_ls = ts ? clock64() : 0;
    if (ts && tid == 0 && uidx == 0) {
      ts[61] = gtime();
      for (int pp = 0; pp < 5; pp++) ts[63 + pp] = (uint64_t)E.len[pp];
    }
    int nxt = warp;                                // next entry item of this warp
    int kbase = 0;                                 // entry item index of the stage's first item
    if constexpr (UR) {
      // windows in original order: item k of a stage at its table offset, own width
      const int *tabs = reinterpret_cast<const int *>(sm + SM::tab_off);
      for (int done = 0; done < E.len[0]; sg++) {
        const int slot = sg % NST;
        mbar_wait(&full[slot], (uint32_t)(sg / NST) & 1u);
        const int *tb = tabs + slot * SM::TABN;
        const int n = tb[0];
        const uint8_t *sbase = ring + (size_t)slot * STAGE;
        for (; nxt < kbase + n; nxt += NCW) {
          const int k = nxt - kbase;
          const uint8_t *rec = sbase + tb[2 + 2 * k];
          switch (tb[3 + 2 * k]) {
            case 0: do_window<D, S, 2>(rec, qs, a.scale_log2, st, o, scratch, lane); break;
            case 1: do_window<D, S, 4>(rec, qs, a.scale_log2, st, o, scratch, lane); break;
            case 2: do_window<D, S, 8>(rec, qs, a.scale_log2, st, o, scratch, lane); break;
            default: do_window<D, S, 16>(rec, qs, a.scale_log2, st, o, scratch, lane); break;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        kbase += n;
        done += n;
      }
    }
#pragma unroll
    for (int p = UR ? 4 : 0; p < 5; p++) {
      using IG = ItemGeo<D, S, false>;
      // item bytes of class p, computed (a table indexed by p would live in local memory)
      const int sz = p == 4 ? IG::REST_SZ : (p == 3 ? 4 * S * D / FS : S * D * (2 << p) / 4 + (GRP ? 16 : 4 * D + 4 * S));
      const int cap = STAGE / sz;
      const int len = E.len[p], nst = E.nst[p], lo = E.lo[p];
      // 2-bit stages (S <= 32) are consumed in PAIRS of windows (do_window2): a stage of n
      // records is ceil(n/2) work items, handed out round robin like single items
      constexpr bool PAIRS = WQ_DEC_PAIR && S <= 32 && !GRP;
      // records of more than WQ_DEC_SUB tokens are consumed as WQ_DEC_SUB-token parts, each
      // part one work item (a record of n parts keeps n warps busy)
      constexpr int SR16 = S / FS;                 // tokens of an FP16 item
      constexpr int SQ = S > WQ_DEC_SUB && WQ_DEC_SUB > 0 ? WQ_DEC_SUB : S;
      constexpr int SF = SR16 > WQ_DEC_SUB && WQ_DEC_SUB > 0 ? WQ_DEC_SUB : SR16;
      const int np = p == 4 ? 1 : (p == 3 ? SR16 / SF : S / SQ);
      for (int t = 0; t < nst; t++, sg++) {
        const int slot = sg % NST;
        const int nrec = min(cap, len - t * cap);
        const int n = (PAIRS && p == 0) ? (nrec + 1) / 2 : nrec * np;
        const uint64_t t0 = ts ? clock64() : 0;
        mbar_wait(&full[slot], (uint32_t)(sg / NST) & 1u);
        const uint64_t t1 = ts ? clock64() : 0;
        if (ts && sg < 64 && lane == 0 && warp == 0) ts[136 + sg] = clock64();
        const uint8_t *sbase = ring + (size_t)slot * STAGE;
        for (; nxt < kbase + n; nxt += NCW) {
          const int k = nxt - kbase;
          const int kr = np > 1 ? k / np : k, part = np > 1 ? k - kr * np : 0;
          WQ_CHECK(k < n && (kr + 1) * sz <= STAGE);
          const uint8_t *rec = sbase + (size_t)kr * sz;
          if (p == 0) {
            if constexpr (PAIRS) {
              const uint8_t *r0 = sbase + (size_t)(2 * k) * sz;
              if (2 * k + 1 < nrec) do_window2<D, S, 2>(r0, r0 + sz, qs, a.scale_log2, st, o, scratch, lane);
              else do_window<D, S, 2>(r0, qs, a.scale_log2, st, o, scratch, lane);
            } else {
              do_window<D, SQ, 2, GRP, S>(rec, qs, a.scale_log2, st, o, scratch, lane, qsum, part);
            }
          } else if (p == 1) {
            do_window<D, SQ, 4, GRP, S>(rec, qs, a.scale_log2, st, o, scratch, lane, qsum, part);
          } else if (p == 2) {
            do_window<D, SQ, 8, GRP, S>(rec, qs, a.scale_log2, st, o, scratch, lane, qsum, part);
          } else if (p == 3) {
            do_window<D, SF, 16, false, SR16>(rec, qs, a.scale_log2, st, o, scratch, lane, make_float2(0.f, 0.f),
                                              part);
          } else {
            const int ii = lo + t * cap + k;
            do_rest<D>(sbase + (size_t)k * 32 * D, sbase + (size_t)(cap + k) * 32 * D, min(16, rl - 16 * (ii - nslots)),
                       qs, a.scale_log2, st, o, scratch, lane);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        kbase += n;
        if (ts) { acc_wait += t1 - t0; acc_comp += clock64() - t1; }
      }
    }
    if (ts && tid == 0) ts[3] = gtime();
    const uint64_t t_e0 = ts ? clock64() : 0;
    if (ts) t_loop += t_e0 - t_ls;

    // ---------------- entry epilogue ----------------
    // (1) every warp parks its (m, l, vb) per head and its o fragments; o goes lane-
    // interleaved in 16-byte groups (group gi = mt*32 + lane: the lane's o[mt][0..3],
    // channels 16mt+g (+8), heads 2q, 2q+1), so parking and reading are conflict-free
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      st.l[0] += __shfl_xor_sync(0xffffffffu, st.l[0], off);
      st.l[1] += __shfl_xor_sync(0xffffffffu, st.l[1], off);
      st.vb[0] += __shfl_xor_sync(0xffffffffu, st.vb[0], off);
      st.vb[1] += __shfl_xor_sync(0xffffffffu, st.vb[1], off);
    }
    {
      float *mine = ep + warp * SM::EPW;
#pragma unroll
      for (int mt = 0; mt < KT; mt++)
        sts128(mine + (mt * 32 + lane) * 4, make_uint4(__float_as_uint(o[mt][0]), __float_as_uint(o[mt][1]),
                                                      __float_as_uint(o[mt][2]), __float_as_uint(o[mt][3])));
      if (g == 0) {
        float *stt = mine + 8 * D;                 // [3][8]: m, l, vb per head
        stt[2 * q] = st.m[0]; stt[2 * q + 1] = st.m[1];
        stt[8 + 2 * q] = st.l[0]; stt[8 + 2 * q + 1] = st.l[1];
        stt[16 + 2 * q] = st.vb[0]; stt[16 + 2 * q + 1] = st.vb[1];
      }
    }
    named_bar_sync(1, NCW * 32);
    uidx++;
    // (2) per head j (8 threads): M = max_w m_w, weights f_w = 2^(m_w - M), L = sum f_w l_w,
    // VB = sum f_w vb_w into hw = [NCW][8] f, then [8] M, [8] L, [8] VB
    const bool split = (c1 - c0) > 1;
    float *hw = reinterpret_cast<float *>(sm + SM::hw_off);
    if (tid < 8) {
      const int j = tid;
      float mw[NCW];
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NCW; w++) {
        mw[w] = ep[w * SM::EPW + 8 * D + j];
        M = fmaxf(M, mw[w]);
      }
      float L = 0.f, VB = 0.f;
#pragma unroll
      for (int w = 0; w < NCW; w++) {
        const float f = (M == -INFINITY) ? 0.f : ex2f(mw[w] - M);
        hw[w * 8 + j] = f;
        L = fmaf(f, ep[w * SM::EPW + 8 * D + 8 + j], L);
        VB = fmaf(f, ep[w * SM::EPW + 8 * D + 16 + j], VB);
      }
      hw[NCW * 8 + j] = M;
      hw[NCW * 8 + 8 + j] = L;
      hw[NCW * 8 + 16 + j] = VB;
    }
    named_bar_sync(1, NCW * 32);
    // (3) per 16-byte group: O = VB + sum_w f_w o_w; a split unit's CTA partial goes to
    // its workspace slot ([8] (M, L) pairs, then the groups), a whole unit's straight out
    float *wslot = a.ws_part + (int64_t)(c + u) * SM::PSLOT;
    for (int gi = tid; gi < KT * 32; gi += NCW * 32) {
      const int jq = 2 * (gi & 3);                 // heads jq, jq + 1
      float4 O = make_float4(hw[NCW * 8 + 16 + jq], hw[NCW * 8 + 17 + jq], hw[NCW * 8 + 16 + jq],
                             hw[NCW * 8 + 17 + jq]);
#pragma unroll
      for (int w = 0; w < NCW; w++) {
        const uint4 v = lds128(ep + w * SM::EPW + gi * 4);
        const uint2 f = lds64(hw + w * 8 + jq);
        O.x = fmaf(__uint_as_float(f.x), __uint_as_float(v.x), O.x);
        O.y = fmaf(__uint_as_float(f.y), __uint_as_float(v.y), O.y);
        O.z = fmaf(__uint_as_float(f.x), __uint_as_float(v.z), O.z);
        O.w = fmaf(__uint_as_float(f.y), __uint_as_float(v.w), O.w);
      }
      if (split) {
        *reinterpret_cast<float4 *>(wslot + 16 + gi * 4) = O;
      } else {
        const float2 M2 = make_float2(hw[NCW * 8 + jq], hw[NCW * 8 + jq + 1]);
        const float2 L2 = make_float2(hw[NCW * 8 + 8 + jq], hw[NCW * 8 + 9 + jq]);
        write_group<D>(a, b, h, gi, O, M2, L2);
      }
    }
    if (split && tid < 8) {
      wslot[2 * tid] = hw[NCW * 8 + tid];
      wslot[2 * tid + 1] = hw[NCW * 8 + 8 + tid];
    }
    const uint64_t t_e1 = ts ? clock64() : 0;
    if (split) {
      // (4) ticket: the last CTA of the unit merges all CTA partials by log-sum-exp
      named_bar_sync(1, NCW * 32);
      // one acq_rel ticket: releases this CTA's partial (written by all threads before
      // the barrier) and, for the last CTA, acquires every other CTA's partial
      if (tid == 0) *s_flag = (atom_add_acq_rel_gpu(a.ws_cnt + u, 1) == c1 - c0 - 1);
      named_bar_sync(1, NCW * 32);
      if (ts && tid == 0) { ts[6] = *s_flag; ts[7] = c - c0; }
      if (*s_flag) merge_unit<D, NCW * 32, SM::PSLOT>(a, tid, u, b, h, c0, c1);
    }
    if (a.peer_bufs && (!split || *s_flag)) peer_exchange_merge<D, NCW * 32>(a, tid, u, b, h);
    if (ts && tid == 0) {
      const uint64_t t_e2 = clock64();
      ts[68] += t_e1 - t_e0; ts[69] += t_e2 - t_e1;
      ts[4] = gtime(); ts[5] += (uint64_t)E.n_u;
    }
    named_bar_sync(1, NCW * 32);                  // ep is reused by the next entry
    if (tid == 0) atomicAdd(units_done, 1);
    if (ts) t_ep += clock64() - t_e0;
  }
  if (ts && lane == 0) {
    uint64_t *wt = ts + 8 + warp * 4;
    wt[0] = acc_wait; wt[1] = acc_comp; wt[2] = t_ep; wt[3] = t_loop;
  }
}

#ifndef WQ_DEC_LBT
#define WQ_DEC_LBT DT                    // launch-bounds thread count (> DT: a lower register cap; experiments)
#endif
template <int D, int S, bool UR, bool GRP>
__global__ void __launch_bounds__(WQ_DEC_LBT, 1) k_decode(DecodeArgs a) {
  decode_body<D, S, UR, GRP>(a, (int)blockIdx.x, (int)gridDim.x);
}

// Fused cross-GPU merge emulated on ONE device in ONE launch (tests): the grid is split
// into NR equal shares, share r plays rank r with its own arguments (image shard, rest,
// workspace, out) and exchanges its partials through the NR "peer" buffers exactly as
// wq_decode_attention_peer does across GPUs: peer stores, system-scope release/acquire
// counters, the bounded wait and the LSE merge.  All CTAs are co-resident (1 CTA/SM,
// grid <= SMs), so every wait is satisfied by CTAs of the same launch.
template <int NR>
struct DecodeArgsN {
  DecodeArgs r[NR];
};
template <int D, int S, int NR>
__global__ void __launch_bounds__(DT, 1) k_decode_emu(const __grid_constant__ DecodeArgsN<NR> s) {
  const int per = (int)gridDim.x / NR;
  const int rk = (int)blockIdx.x / per;
  if (rk >= NR) return;
  decode_body<D, S, false>(s.r[rk], (int)blockIdx.x - rk * per, per);
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

// Workspace layout (wq_decode_workspace): CTA partial slots of 16 + 8d floats (k_decode;
// >= grp * (d + 2), decode_tc's rows) for num_sms + B*H slots, then B*H ticket counters,
// then the profiling timestamps; each region 256-byte aligned.
DecodeWsLayout decode_ws_layout(int B, int H, int d, int num_sms) {
  DecodeWsLayout L;
  L.part = ((size_t)(num_sms + B * H) * (16 + 8 * (size_t)d) * sizeof(float) + 255) / 256 * 256;
  L.cnt = ((size_t)B * H * sizeof(int32_t) + 255) / 256 * 256;
  L.ts = (size_t)num_sms * TS_PER_CTA * sizeof(uint64_t);
  return L;
}
size_t decode_workspace_bytes(int B, int H, int Hq, int d, int num_sms) {
  (void)Hq;
  const DecodeWsLayout L = decode_ws_layout(B, H, d, num_sms);
  return L.part + L.cnt + L.ts;
}

template <int D, int S, bool UR, bool GRP = false>
static cudaError_t launch_decode_t(const DecodeArgs &a, int num_sms, cudaStream_t st) {
  using SM = DecodeSmem<D, S, UR ? 1 : fsplit<D, S>()>;
  static bool attr_set = false;                  // per instantiation (per process: one device)
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_decode<D, S, UR, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SM::total);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (a.peer_bufs) {
    // the exchange waits on partials written by other CTAs of this grid's peers: every CTA
    // must be resident at once (one per SM) or a waiting CTA could starve one not yet
    // scheduled on a peer
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode<D, S, UR, GRP>, DT, SM::total);
    if (e != cudaSuccess) return e;
    if (per_sm < 1 || num_sms > device_sm_count()) return cudaErrorCooperativeLaunchTooLarge;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms);
  cfg.blockDim = dim3(DT);
  cfg.dynamicSmemBytes = SM::total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (a.flags & WQ_DECODE_EARLY_) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, k_decode<D, S, UR, GRP>, a);
}

cudaError_t launch_decode(const DecodeArgs &a, int num_sms, cudaStream_t st) {
  // WQ_DECODE_TC=1 (head dim 128): the tcgen05/TMEM kernel of decode_tc.cu instead of
  // this file's mma.sync kernel.  Parity-clean but ~4x slower on C5 (its dequantization
  // warps are issue/latency bound), so it is opt-in.
  // (The tcgen05 kernel has no peer exchange: the fused-merge path always runs here.)
  static const bool use_tc = getenv("WQ_DECODE_TC") && atoi(getenv("WQ_DECODE_TC")) != 0;
  if (a.d == 128 && use_tc && !a.woff && !a.peer_bufs && !(a.flags & WQ_DECODE_GROUP_)) return launch_decode_tc(a, num_sms, st);
#define WQ_D(DD, SS)                                                                                      \
  if (a.d == DD && a.S == SS)                                                                             \
    return a.woff ? launch_decode_t<DD, SS, true>(a, num_sms, st)                                         \
                  : ((a.flags & WQ_DECODE_GROUP_) ? launch_decode_t<DD, SS, false, true>(a, num_sms, st)   \
                                                  : launch_decode_t<DD, SS, false>(a, num_sms, st));
  WQ_D(64, 16) WQ_D(64, 32) WQ_D(64, 64) WQ_D(64, 128)
  WQ_D(128, 16) WQ_D(128, 32) WQ_D(128, 64) WQ_D(128, 128)
#undef WQ_D
  return cudaErrorInvalidValue;
}

template <int D, int S>
static cudaError_t launch_emu_t(const DecodeArgs *ra, int nr, int num_sms, cudaStream_t st) {
  using SM = DecodeSmem<D, S, fsplit<D, S>()>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_decode_emu<D, S, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SM::total);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (nr != 2) return cudaErrorInvalidValue;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode_emu<D, S, 2>, DT, SM::total);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  DecodeArgsN<2> s;
  s.r[0] = ra[0];
  s.r[1] = ra[1];
  k_decode_emu<D, S, 2><<<(num_sms / 2) * 2, DT, SM::total, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_decode_emu(const DecodeArgs *ra, int nr, int num_sms, cudaStream_t st) {
  const DecodeArgs &a = ra[0];
  if (a.d == 128 && a.S == 32) return launch_emu_t<128, 32>(ra, nr, num_sms, st);
  if (a.d == 64 && a.S == 16) return launch_emu_t<64, 16>(ra, nr, num_sms, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_merge(const float *parts, int G, int BHq, int d, __half *out, cudaStream_t st) {
  k_merge<<<BHq, 128, 0, st>>>(parts, G, BHq, d, out);
  return cudaGetLastError();
}

}  // namespace wq
