// decode_tc.cu -- wq_decode_attention for head dim 128 on the 5th-generation tensor
// cores (tcgen05, accumulators and the dequantized operand in tensor memory).
// Computes Alg.2's decode branch: Eq.2-3 without mask over the
// reordered mixed-precision cache (reorder invariance Eq.12-13) with the
// dequantization fused into the operand path, split-KV with an online
// softmax and a log-sum-exp merge (reading Q24).
//
// Per CTA (persistent, one per SM, 14 warps):
//  * warp 12, producer: TMA 1-D bulk copies of the CTA's items (window records of one
//    width class per stage, FP16 rest rows) into a shared-memory ring (decode_common).
//  * warps 0-7, dequantizers: the items are consumed in GROUPS of 128 tokens (128/S
//    windows of one class, or 8 rest tiles).  For a group they write to TMEM
//      A_K = K codes  [128 tokens x 128 channels] fp16 (exact integers),
//      A_V = V codes^T [128 channels x 128 tokens] fp16, centered (code - 2^(b-1)),
//    straight from the D-1 fragment-order chunks (one LOP3 + one HSUB2 per pair, then
//    tcgen05.st 16x256b), and to shared memory the K-side B operand
//      B_q[w] = q_h * s_c (per window w, head h, channel c) as fp16 hi + lo,
//    plus the zero-point terms z[w][h] = sum_c q_h[c] mn_c (mma.sync on the param
//    quads) and the per-token V scale / zero point (s_t, mn_t + s_t 2^(b-1)).
//  * warp 13, MMA issuer (one thread): per group
//      S  = A_K x [B_q_hi | B_q_lo]   (M = 128 tokens, N = 8 x 128/S, 2 x 8 MMAs),
//      O += A_V x P'                  (M = 128 channels, N = 8 heads, 8 MMAs)
//    where P'[t][h] = p[t][h] * s_t comes from the softmax warps.
//  * warps 8-11, softmax (thread = token row): logits from TMEM (own window's 8
//    columns) + z, lazy running max shared by the warpgroup (rescale only when a
//    logit exceeds it by 2^8), p = 2^(x - m), row sums l and V zero-point sums in
//    registers, P' to shared memory (MN-major B operand); the unit epilogue reads
//    O from TMEM (thread = channel) and writes the CTA partial / output.
// Groups alternate between two buffer sets (TMEM A_K/A_V/S, shared B_q/P'/params),
// so group j+1 is dequantized while group j is in the MMA and softmax stages.
// The split-KV partition, producer and cross-CTA merge are decode_common.cuh's.
#include <type_traits>
#include "decode_common.cuh"

namespace wq {
namespace tcd {

constexpr int D = 128;
constexpr int KT = D / 16;              // k16 blocks over the head dim
constexpr int NDQ = 8;                  // dequant warps 0..7 (two per TMEM lane quarter)
constexpr int W_SMX = 8;                // softmax warps 8..11
constexpr int W_PROD = 12, W_MMA = 13;
constexpr int NT = 14 * 32;
constexpr float LAZY_TH = 8.0f;
constexpr int BAR_DQ = 1, BAR_SMX = 3, BAR_END = 5;
#ifndef WQ_TC_PROFILE
#define WQ_TC_PROFILE 0        // per-group clock64 stamps into the workspace (debug & 8; tools/dbg_tc_time.py)
#endif
constexpr int PROF_G = 38;     // groups stamped per CTA (5 events each)
#ifndef WQ_TC_PROF_W
#define WQ_TC_PROF_W -1        // >= 0: stamp the inside of dequant warp W instead of the pipeline
#endif

// TMEM columns (512 allocated): A_K[2] 64 each, A_V[2] 64 each, S[2] 8G each, O[2] 8 each
constexpr uint32_t TM_AK = 0, TM_AV = 128, TM_S = 256;

struct GMeta {
  int term, kind, n, nvalid, first, last, u, c0, c1, pad[3];
};

template <int S>
struct Cfg {
  static constexpr int G = 128 / S;          // windows per group
  static constexpr int NK = 8 * G;           // N of the K-side MMA (8 head columns per window)
  static constexpr int BW = NDQ / G;         // dequant warps per window when building B_q
  static constexpr int KB = KT / BW;         // k16 blocks per warp when building B_q
  static constexpr uint32_t TM_O = TM_S + 2 * NK;
  static constexpr int STAGE = (4 * S * D > 32768) ? 4 * S * D : 32768;
  static constexpr int BQ = NK * 256;        // bytes of one B_q (hi or lo): NK rows x 128 fp16
  // shared memory layout
  static constexpr size_t bq_off = 0;                              // [2 buf][2 hi/lo][BQ]
  static constexpr size_t bv_off = bq_off + 4 * (size_t)BQ;        // [2][128 tok][8 heads] fp16
  static constexpr size_t qs_off = bv_off + 2 * 2048;              // q fragments [KT][32][2]
  static constexpr size_t zp_off = qs_off + KT * 32 * 8;           // [2][BW][G][8] f32
  static constexpr size_t vp_off = zp_off + 2 * BW * G * 8 * 4;    // [2][128] float2
  static constexpr size_t meta_off = vp_off + 2 * 128 * 8;         // [2] GMeta
  static constexpr size_t xch_off = meta_off + 2 * sizeof(GMeta);  // [2][4] flags, [2][4][8] max, [4][16] sums
  static constexpr size_t units_off = xch_off + (8 + 64 + 64 + 8) * 4;
  static constexpr size_t ent_off = units_off + (size_t)(MAX_UNITS + 1) * 8;
  static constexpr int NUS = 4;
  static constexpr size_t plan_off = ent_off + NUS * sizeof(Entry);
  static constexpr size_t misc_off = plan_off + sizeof(CtaPlan);
  static constexpr size_t bar_off = (misc_off + 32 + 15) / 16 * 16;
  static constexpr int NBAR_FIXED = 10;                            // deq_full, s_full, p_full, o_done, ep_done x2
  static constexpr size_t small_end = bar_off + (size_t)NBAR_FIXED * 8 + 2 * 8 * 8;   // + full/empty (<= 8 stages)
  static constexpr size_t ring_off = (small_end + 1023) / 1024 * 1024;
  static constexpr size_t SMEM_MAX = 227 * 1024;
  static constexpr int NST_ = (int)((SMEM_MAX - ring_off) / STAGE);
  static constexpr int NST = NST_ > 6 ? 6 : NST_;
  static_assert(NST >= 2, "ring too small");
  static constexpr size_t total = ring_off + (size_t)NST * STAGE;
};

// token row r of a 16-row block -> K position of the tcgen05 operand written from
// mma.sync fragments (column pair p holds rows 2(p>>1) + 8(p&1) + {0,1})
WQ_DEV int kpos16(int r) { return 4 * ((r & 7) >> 1) + 2 * (r >> 3) + (r & 1); }

// Plain (non-volatile) shared-memory loads: the compiler may batch them ahead of the
// dequantization arithmetic (the asm volatile helpers of wq_device.cuh keep program order).
template <class T>
WQ_DEV T ldsp(const uint8_t *p) { return *reinterpret_cast<const T *>(p); }

// Raw code words of m-block mv (channels 16mv..16mv+15) of one 16-token V code tile
// (D-1 fragment order; a lane's chunk word w sits at (w/4)*512 + lane*16 + (w%4)*4).
template <int BITS>
WQ_DEV uint4 v_raw(const uint8_t *tile, int lane, int mv) {
  if constexpr (BITS == 2) {
    return make_uint4(ldsp<uint32_t>(tile + lane * 16 + 4 * (mv >> 1)), 0u, 0u, 0u);
  } else if constexpr (BITS == 4) {
    return make_uint4(ldsp<uint32_t>(tile + (mv >> 2) * 512 + lane * 16 + (mv & 3) * 4), 0u, 0u, 0u);
  } else if constexpr (BITS == 8) {
    const uint2 v = ldsp<uint2>(tile + (mv >> 1) * 512 + lane * 16 + (mv & 1) * 8);
    return make_uint4(v.x, v.y, 0u, 0u);
  } else {
    return ldsp<uint4>(tile + mv * 512 + lane * 16);
  }
}
// ... -> the A fragment a[0..3] = exact fp16 pairs of (code - 2^(BITS-1)); ODD = mv & 1
template <int BITS, int ODD>
WQ_DEV void v_deq(uint4 w, uint32_t (&a)[4]) {
  if constexpr (BITS == 2) {
    const uint32_t w8 = w.x >> 8;
    a[0] = dq_pair<2, 4 * ODD + 0, true>(w.x, w8); a[1] = dq_pair<2, 4 * ODD + 1, true>(w.x, w8);
    a[2] = dq_pair<2, 4 * ODD + 2, true>(w.x, w8); a[3] = dq_pair<2, 4 * ODD + 3, true>(w.x, w8);
  } else if constexpr (BITS == 4) {
    const uint32_t w8 = w.x >> 8;
    a[0] = dq_pair<4, 0, true>(w.x, w8); a[1] = dq_pair<4, 1, true>(w.x, w8);
    a[2] = dq_pair<4, 2, true>(w.x, w8); a[3] = dq_pair<4, 3, true>(w.x, w8);
  } else if constexpr (BITS == 8) {
    a[0] = dq_pair8<0, true>(w.x); a[1] = dq_pair8<1, true>(w.x);
    a[2] = dq_pair8<0, true>(w.y); a[3] = dq_pair8<1, true>(w.y);
  } else {
    a[0] = w.x; a[1] = w.y; a[2] = w.z; a[3] = w.w;
  }
}
// a lane's whole chunk of one 16-token K code tile (D*BITS/64 words)
template <int BITS>
WQ_DEV void k_chunk(uint32_t (&wd)[D * BITS / 64], const uint8_t *tile, int lane) {
  constexpr int WPL = D * BITS / 64;
#pragma unroll
  for (int i = 0; i < WPL / 4; i++) {
    const uint4 v = ldsp<uint4>(tile + 512 * i + lane * 16);
    wd[4 * i] = v.x; wd[4 * i + 1] = v.y; wd[4 * i + 2] = v.z; wd[4 * i + 3] = v.w;
  }
}

// Last-CTA merge of a split unit's CTA partials, thread = channel cc, heads in turn
// (few registers: it runs inside the softmax warps' loop).
WQ_DEV void merge_unit_rows(const DecodeArgs &a, int cc, int u, int b, int h, int c0, int c1) {
  const int grp = a.grp, np = c1 - c0;
  const int64_t stride = (int64_t)grp * (D + 2);
  const float *pb = a.ws_part + (int64_t)(c0 + u) * stride;
#pragma unroll 1
  for (int jj = 0; jj < grp; jj++) {
    const float *hb = pb + jj * (D + 2);
    float M = -INFINITY, L = 0.f, O = 0.f;
#pragma unroll 1
    for (int b0 = 0; b0 < np; b0 += 4) {
      float mv[4], lv[4], ov[4];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const bool ok = b0 + i < np;
        mv[i] = ok ? __ldcg(hb + (b0 + i) * stride) : -INFINITY;
        lv[i] = ok ? __ldcg(hb + (b0 + i) * stride + 1) : 0.f;
        ov[i] = ok ? __ldcg(hb + (b0 + i) * stride + 2 + cc) : 0.f;
      }
      float Mn = M;
#pragma unroll
      for (int i = 0; i < 4; i++) Mn = fmaxf(Mn, lv[i] > 0.f ? mv[i] : -INFINITY);
      if (Mn != -INFINITY) {
        const float rr = exp2f(M - Mn);
        L *= rr;
        O *= rr;
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const float f = lv[i] > 0.f ? exp2f(mv[i] - Mn) : 0.f;
          L = fmaf(f, lv[i], L);
          O = fmaf(f, ov[i], O);
        }
        M = Mn;
      }
    }
    const int64_t row = (int64_t)b * a.Hq + h * grp + jj;
    if (a.out) a.out[row * D + cc] = __float2half_rn(L > 0.f ? O / L : 0.f);
    if (a.partial) {
      float *pp = a.partial + row * (D + 2);
      if (cc == 0) { pp[0] = M * 0.69314718055994530942f; pp[1] = L; }
      pp[2 + cc] = O;
    }
  }
  if (cc == 0) a.ws_cnt[u] = 0;
}

template <int S>
__global__ void __launch_bounds__(NT, 1) k_decode_tc(DecodeArgs a) {
  using C = Cfg<S>;
  using IG = ItemGeo<D, S, true>;
  constexpr int G = C::G, NST = C::NST, STAGE = C::STAGE;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *ring = sm + C::ring_off;
  int64_t *ustart = reinterpret_cast<int64_t *>(sm + C::units_off);
  Entry *ent = reinterpret_cast<Entry *>(sm + C::ent_off);
  CtaPlan *cp = reinterpret_cast<CtaPlan *>(sm + C::plan_off);
  int *s_flag = reinterpret_cast<int *>(sm + C::misc_off);
  int *units_done = s_flag + 1;
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(s_flag + 2);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + C::bar_off);
  uint64_t *deq_full = bars, *s_full = bars + 2, *p_full = bars + 4, *o_done = bars + 6, *ep_done = bars + 8;
  uint64_t *full = bars + C::NBAR_FIXED, *empty = full + NST;
  GMeta *meta = reinterpret_cast<GMeta *>(sm + C::meta_off);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int U = a.B * a.H;
  uint64_t *ts = (WQ_TC_PROFILE && a.ws_ts) ? a.ws_ts + (size_t)blockIdx.x * TS_PER_CTA : nullptr;
  auto stamp = [&](int jj, int ev) { if (ts && jj < PROF_G) ts[10 + 5 * jj + ev] = clock64(); };
  if (ts && tid == 0) ts[0] = clock64();

  if (warp == 0) plan_cta<D, S, true>(a, ustart, cp, s_flag, lane, (int)blockIdx.x, (int)gridDim.x);
  if (tid == 32) {
    for (int s = 0; s < NST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NDQ);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(&deq_full[i], NDQ);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
      mbar_init(&ep_done[i], 1);
    }
    *units_done = 0;
    for (int i = 0; i < C::NUS; i++) ent[i].tag = -1;
    fence_mbar_init();
  }
  __syncthreads();
  const int Gc = *s_flag;
  const int c = blockIdx.x;
  if (tid == 0) griddep_launch_dependents();
  if (c >= Gc) return;
  if (warp == W_MMA) tmem_alloc(s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == W_PROD) {
    if (lane == 0) produce<D, S, true, STAGE, NST, C::NUS>(a, *cp, ustart, ring, full, empty, ent, units_done, nullptr,
                                                           (int)blockIdx.x);
    return;
  }

  if (warp == W_MMA) {
    // =========================== MMA issuer ===========================
    {
      // the whole warp runs the (warp-uniform) loop; one elected lane issues each
      // tcgen05.mma / commit, so descriptors stay in uniform registers
      constexpr uint32_t idK = tc_idesc_f16(128, C::NK, 0);
      constexpr uint32_t idV = tc_idesc_f16(128, 8, 1);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      // B descriptors of k-step 0; k-step ks adds ks * 256 B = ks * 16 to the address field
      const uint64_t dq0 = tc_sdesc(smem_u32(sm + C::bq_off), 128, 2048);
      const uint64_t dv0 = tc_sdesc(smem_u32(sm + C::bv_off), 128, 128);
      auto issue_k = [&](int bf) {
        const uint32_t dK = tm + TM_S + bf * C::NK, aK = tm + TM_AK + bf * 64;
        const uint64_t bhi = dq0 + (uint64_t)((2 * bf) * C::BQ >> 4), blo = bhi + (uint64_t)(C::BQ >> 4);
#pragma unroll
        for (int ks = 0; ks < KT; ks++) tc_mma_ts_elect(dK, aK + 8 * ks, bhi + 16 * ks, idK, ks > 0);
#pragma unroll
        for (int ks = 0; ks < KT; ks++) tc_mma_ts_elect(dK, aK + 8 * ks, blo + 16 * ks, idK, 1);
        tc_commit_elect(&s_full[bf]);
      };
      // event loop: K(nk) as soon as group nk is dequantized (and S[nk&1] was read by
      // the softmax of group nk-2, i.e. V(nk-2) issued), V(nv) as soon as P'(nv) is ready
      int nk = 0, nv = 0, ev = -1;
      bool term = false;
      int vfirst[2] = {0, 0};
      for (;;) {
        bool progressed = false;
        if (!term && nk <= nv + 1 && mbar_test(&deq_full[nk & 1], (uint32_t)(nk >> 1) & 1u)) {
          tc_fence_after();
          const GMeta &mm = meta[nk & 1];
          if (mm.term) {
            term = true;
          } else {
            vfirst[nk & 1] = mm.first;
            issue_k(nk & 1);
            progressed = true;
            if (WQ_TC_PROF_W < 0 && lane == 0) stamp(nk, 2);
            nk++;
          }
        }
        if (nv < nk && mbar_test(&p_full[nv & 1], (uint32_t)(nv >> 1) & 1u)) {
          tc_fence_after();
          const int bf = nv & 1, first = vfirst[bf];
          ev += first;
          if (first && ev >= 2) mbar_wait_hint(&ep_done[ev & 1], (uint32_t)((ev - 2) >> 1) & 1u);
          const uint32_t dO = tm + C::TM_O + (ev & 1) * 8, aV = tm + TM_AV + bf * 64;
          const uint64_t bv = dv0 + (uint64_t)(bf * (2048 >> 4));
#pragma unroll
          for (int ks = 0; ks < KT; ks++)
            tc_mma_ts_elect(dO, aV + 8 * ks, bv + 16 * ks, idV, (ks > 0 || !first) ? 1u : 0u);
          tc_commit_elect(&o_done[bf]);
          nv++;
          progressed = true;
        }
        if (term && nv == nk) break;
        if (!progressed) __nanosleep(32);
      }
    }
    __syncwarp();
  } else if (warp < NDQ) {
    // =========================== dequantizers ===========================
    const int wl = warp, qd = wl & 3, hf = wl >> 2;
    const int g = lane >> 2, q = lane & 3;
    uint8_t *qs = sm + C::qs_off;
    int uidx = 0, j = 0, sg = 0;
    if (wl == 0 && (a.flags & WQ_DECODE_EARLY_)) griddep_wait();     // q
    // wait until buffer set bf may be rewritten (group j - 2 fully consumed)
    // buffer set jj & 1 may be rewritten once group jj - 2 is fully consumed: warp 0
    // waits (with any stage waits it already did), the other warps block on a
    // hardware barrier instead of polling shared memory
    auto acquire = [&](int jj) {
      if (wl == 0 && jj >= 2) {
        const uint32_t par = (uint32_t)((jj - 2) >> 1) & 1u;
        mbar_wait_sleep(&s_full[jj & 1], par, 20);
        mbar_wait_sleep(&o_done[jj & 1], par, 20);
      }
      named_bar_sync(BAR_DQ, NDQ * 32);
      tc_fence_after();
    };
    auto publish = [&](int jj) {
      tc_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&deq_full[jj & 1]);
    };
    for (;;) {
      const Entry &E = ent[uidx % C::NUS];
      while (*reinterpret_cast<const volatile int *>(&E.tag) != uidx) {
      }
      __threadfence_block();
      const int u = *reinterpret_cast<const volatile int *>(&E.u);
      if (u < 0) {
        acquire(j);
        if (wl == 0 && lane == 0) meta[j & 1].term = 1;
        publish(j);
        break;
      }
      int len[5], nst[5], lo[5];
#pragma unroll
      for (int p = 0; p < 5; p++) { len[p] = E.len[p]; nst[p] = E.nst[p]; lo[p] = E.lo[p]; }
      const int c0 = E.c0, c1 = E.c1, rl = E.rl, nslots = E.nslots;
      named_bar_sync(BAR_DQ, NDQ * 32);            // everyone read the entry and finished the last one
      if (wl == 0) {
        const int bq_ = u / a.H, hq_ = u - bq_ * a.H;
        const __half *qrow = a.q + ((int64_t)bq_ * a.Hq + hq_ * a.grp + g) * D;
#pragma unroll
        for (int kt = 0; kt < KT; kt++) {
          const uint32_t x0 = g < a.grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q) : 0u;
          const uint32_t x1 = g < a.grp ? *reinterpret_cast<const uint32_t *>(qrow + 16 * kt + 2 * q + 8) : 0u;
          *reinterpret_cast<uint2 *>(qs + (kt * 32 + lane) * 8) = make_uint2(x0, x1);
        }
        if (lane == 0) atomicAdd(units_done, 1);   // entry slot may be reused
      }
      named_bar_sync(BAR_DQ, NDQ * 32);
      uidx++;

      // groups of the entry: pieces in order, GI items per group
      int ngroups = 0;
#pragma unroll
      for (int p = 0; p < 5; p++) ngroups += (len[p] + (p < 4 ? G : 8) - 1) / (p < 4 ? G : 8);
      int gi = 0;                                  // group index within the entry
      auto meta_write = [&](int kind, int n, int nvalid) {
        if (wl == 0 && lane == 0) {
          GMeta &m = meta[j & 1];
          m.term = 0; m.kind = kind; m.n = n; m.nvalid = nvalid;
          m.first = gi == 0; m.last = gi == (ngroups > 0 ? ngroups : 1) - 1;
          m.u = u; m.c0 = c0; m.c1 = c1;
        }
      };
      if (ngroups == 0) {
        // empty share: one all-masked group so the unit still gets this CTA's partial
        acquire(j);
        meta_write(0, 0, 0);
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; i++) z[i] = 0u;
        tmem_st_16x256b_x8(tmem + TM_AV + (j & 1) * 64 + ((uint32_t)(32 * qd + 16 * hf) << 16), z);
        publish(j);
        j++;
        continue;
      }
      auto piece = [&](auto pc) {
        constexpr int p = decltype(pc)::value;
        constexpr int sz = IG::sz(p);
        constexpr int cap = STAGE / sz;
        constexpr int GI = p < 4 ? G : 8;
        int waited = 0, released = 0;
        for (int k0 = 0; k0 < len[p]; k0 += GI, gi++, j++) {
          const int n = min(GI, len[p] - k0);
          const int tlast = (k0 + n - 1) / cap;
          for (; waited <= tlast; waited++) {
            const int s_ = sg + waited;
            if (wl == 0) mbar_wait_sleep(&full[s_ % NST], (uint32_t)(s_ / NST) & 1u, 20);
          }
          // item k0 + k of the piece: stage slot / offset of the group's first item once,
          // then cheap steps (cap, NST compile-time; a group spans at most two stages)
          const int s0 = sg + k0 / cap;
          const int slot0 = s0 % NST, off0 = k0 % cap;
          auto item = [&](int k) -> const uint8_t * {
            const int o = off0 + k;
            const int st = o / cap;
            int sl = slot0 + st;
            sl -= sl >= NST ? NST : 0;
            return ring + sl * STAGE + (o - st * cap) * sz;
          };
          acquire(j);
          if (WQ_TC_PROF_W != 99 && wl == (WQ_TC_PROF_W < 0 ? 0 : WQ_TC_PROF_W) && lane == 0) stamp(j, 0);
          const int bf = j & 1;
          const uint32_t tAK = tmem + TM_AK + bf * 64, tAV = tmem + TM_AV + bf * 64;
          float2 *vp = reinterpret_cast<float2 *>(sm + C::vp_off) + bf * 128;
          float *zp = reinterpret_cast<float *>(sm + C::zp_off) + bf * (C::BW * G * 8);
          uint8_t *bqh = sm + C::bq_off + (size_t)(2 * bf) * C::BQ, *bql = bqh + C::BQ;
          const int ts_ = 2 * qd + hf;             // 16-row tile of the group this warp writes (K side)
          auto bq_store = [&](int wi, int m, uint32_t h0, uint32_t h1, uint32_t l0, uint32_t l1) {
            const int off = g * 16 + wi * 2048 + (2 * m + (q >> 1)) * 128 + (q & 1) * 8;
            *reinterpret_cast<uint2 *>(bqh + off) = make_uint2(h0, h1);      // plain stores: may overlap
            *reinterpret_cast<uint2 *>(bql + off) = make_uint2(l0, l1);      // the loads around them
          };
          if constexpr (p < 4) {
            const int nvalid = n * S;
            meta_write(p, n, nvalid);
            auto run = [&](auto bits_c, auto full_c) {
              constexpr int BITS = decltype(bits_c)::value;
              constexpr bool FULL = decltype(full_c)::value;     // n == G: no absent windows
              auto present = [&](int w) { return FULL || w < n; };
              constexpr int TILE = 2 * D * BITS;
              // ---- K tile -> A_K ----
              {
                const int wi = (16 * ts_) / S, ti = ((16 * ts_) % S) / 16;
                if (present(wi)) {
                  uint32_t wd[D * BITS / 64];
                  k_chunk<BITS>(wd, item(wi) + ti * TILE, lane);
                  uint32_t r[32];
#pragma unroll
                  for (int kt = 0; kt < KT; kt++) {
                    r[4 * kt + 0] = deq_pair<BITS>(wd, 4 * kt + 0);
                    r[4 * kt + 1] = deq_pair<BITS>(wd, 4 * kt + 2);
                    r[4 * kt + 2] = deq_pair<BITS>(wd, 4 * kt + 1);
                    r[4 * kt + 3] = deq_pair<BITS>(wd, 4 * kt + 3);
                  }
                  tmem_st_16x256b_x8(tAK + ((uint32_t)(16 * ts_) << 16), r);
                  // V params of the tile's 16 tokens -> (s_t, mn_t + s_t 2^(BITS-1))
                  if (lane < 16) {
                    float2 v2 = make_float2(1.f, 0.f);
                    if constexpr (BITS < 16) {
                      const uint8_t *vpar = item(wi) + 2 * (S * D * BITS / 8) + 4 * D;
                      const int r16 = lane, qq = (r16 & 7) >> 1, hsel = 2 * (r16 >> 3) + (r16 & 1);
                      const __half *grp8 = reinterpret_cast<const __half *>(vpar + (4 * ti + qq) * 16);
                      const float s_ = __half2float(grp8[hsel]);
                      const float mn = __half2float(grp8[4 + hsel]);
                      v2 = make_float2(s_, fmaf(s_, (float)(1 << (BITS - 1)), mn));
                    }
                    vp[16 * ts_ + lane] = v2;
                  }
                }
              }
              if (wl == WQ_TC_PROF_W && lane == 0) stamp(j, 1);
              // ---- B_q (q * s_c, hi + lo) and z = q . mn for window wb, k-blocks [kb0, kb0 + KB) ----
              {
                const int wb = wl / C::BW, kb0 = (wl % C::BW) * C::KB;
                if (present(wb)) {
                  float zc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
                  const uint8_t *kp = item(wb) + 2 * (S * D * BITS / 8);
                  uint2 qk[C::KB];
                  uint4 pr[C::KB];
#pragma unroll
                  for (int i = 0; i < C::KB; i++) {        // all loads first
                    qk[i] = ldsp<uint2>(qs + ((kb0 + i) * 32 + lane) * 8);
                    if constexpr (BITS < 16) pr[i] = ldsp<uint4>(kp + (4 * (kb0 + i) + q) * 16);
                  }
#pragma unroll
                  for (int i = 0; i < C::KB; i++) {
                    const int m = kb0 + i;
                    if constexpr (BITS < 16) {
                      const uint32_t am[4] = {pr[i].x, pr[i].y, pr[i].z, pr[i].w};
                      mma16816(zc[i & 1], am, qk[i].x, qk[i].y, zc[i & 1]);
                      const uint32_t h0 = hmul2u(qk[i].x, pr[i].y), h1 = hmul2u(qk[i].y, pr[i].w);
                      const uint32_t l0 = h2u(__hfma2(u2h(qk[i].x), u2h(pr[i].y), __hneg2(u2h(h0))));
                      const uint32_t l1 = h2u(__hfma2(u2h(qk[i].y), u2h(pr[i].w), __hneg2(u2h(h1))));
                      bq_store(wb, m, h0, h1, l0, l1);
                    } else {
                      bq_store(wb, m, qk[i].x, qk[i].y, 0u, 0u);
                    }
                  }
                  if (lane < 4) {
                    float *zz = zp + ((wl % C::BW) * G + wb) * 8;
                    *reinterpret_cast<float2 *>(zz + 2 * q) = make_float2(zc[0][0] + zc[1][0], zc[0][1] + zc[1][1]);
                  }
                }
              }
              if (wl == WQ_TC_PROF_W && lane == 0) stamp(j, 2);
              // ---- V tiles -> A_V (channels 16*mv.., all 8 token tiles of the group) ----
              {
                const int mv = 2 * qd + hf;
                const uint8_t *ip[G];
#pragma unroll
                for (int wi = 0; wi < G; wi++) ip[wi] = item(wi);
                uint4 raw[8];
#pragma unroll
                for (int tt = 0; tt < 8; tt++) {          // all loads first
                  const int wi = (16 * tt) / S, ti = ((16 * tt) % S) / 16;
                  raw[tt] = make_uint4(0u, 0u, 0u, 0u);
                  if (present(wi)) raw[tt] = v_raw<BITS>(ip[wi] + S * D * BITS / 8 + ti * TILE, lane, mv);
                }
                uint32_t r[32];
#pragma unroll
                for (int tt = 0; tt < 8; tt++) {
                  const int wi = (16 * tt) / S;
                  uint32_t f[4];
                  if (hf) v_deq<BITS, 1>(raw[tt], f);
                  else v_deq<BITS, 0>(raw[tt], f);
                  if (!present(wi)) f[0] = f[1] = f[2] = f[3] = 0u;
                  r[4 * tt + 0] = f[0]; r[4 * tt + 1] = f[2]; r[4 * tt + 2] = f[1]; r[4 * tt + 3] = f[3];
                }
                tmem_st_16x256b_x8(tAV + ((uint32_t)(16 * mv) << 16), r);
                if (wl == WQ_TC_PROF_W && lane == 0) stamp(j, 3);
              }
            };
            using BC = std::integral_constant<int, (p == 0 ? 2 : p == 1 ? 4 : p == 2 ? 8 : 16)>;
            if (n == G) run(BC{}, std::true_type{});
            else run(BC{}, std::false_type{});
          } else {
            // ---- FP16 rest tiles (row-major [16][D] K and V rows as the bulk copies land them) ----
            const int t_first = lo[4] - nslots + k0;      // rest tile index of the group's first tile
            const int nvalid = min(16 * n, rl - 16 * t_first);
            meta_write(4, n, nvalid);
            const int mi = lane >> 3, rr = lane & 7;
            {
              if (ts_ < n) {
                const int kk = k0 + ts_;
                const uint8_t *sbase = ring + (size_t)((sg + kk / cap) % NST) * STAGE;
                const __half *Ks = reinterpret_cast<const __half *>(sbase + (size_t)(kk % cap) * 32 * D);
                uint32_t r[32];
#pragma unroll
                for (int kt = 0; kt < KT; kt++) {
                  uint32_t f[4];
                  ldsm_x4(f, Ks + ((mi & 1) * 8 + rr) * D + 16 * kt + (mi >> 1) * 8);
                  r[4 * kt + 0] = f[0]; r[4 * kt + 1] = f[2]; r[4 * kt + 2] = f[1]; r[4 * kt + 3] = f[3];
                }
                tmem_st_16x256b_x8(tAK + ((uint32_t)(16 * ts_) << 16), r);
                if (lane < 16) vp[16 * ts_ + lane] = make_float2(1.f, 0.f);
              }
            }
            {
              // B_q = q for every window slot of the group, z = 0
              const int wb = wl / C::BW, kb0 = (wl % C::BW) * C::KB;
#pragma unroll
              for (int i = 0; i < C::KB; i++) {
                const int m = kb0 + i;
                const uint2 qk = ldsp<uint2>(qs + (m * 32 + lane) * 8);
                bq_store(wb, m, qk.x, qk.y, 0u, 0u);
              }
              if (lane < 4) {
                float *zz = zp + ((wl % C::BW) * G + wb) * 8;
                zz[2 * q] = 0.f;
                zz[2 * q + 1] = 0.f;
              }
            }
            {
              const int mv = 2 * qd + hf;
              const int q2 = lane & 3;
              uint32_t r[32];
#pragma unroll
              for (int tt = 0; tt < 8; tt++) {
                uint32_t f[4] = {0u, 0u, 0u, 0u};
                if (tt < n) {
                  const int kk = k0 + tt;
                  const uint8_t *sbase = ring + (size_t)((sg + kk / cap) % NST) * STAGE;
                  const __half *Vs = reinterpret_cast<const __half *>(sbase + (size_t)(cap + kk % cap) * 32 * D);
                  ldsm_x4_t(f, Vs + ((mi >> 1) * 8 + rr) * D + 16 * mv + (mi & 1) * 8);
                  const int ntok = min(16, rl - 16 * (t_first + tt));
                  // zero masked token columns (stale shared memory may hold non-finite bits)
                  const uint32_t m01 = (2 * q2 < ntok ? 0xffffu : 0u) | (2 * q2 + 1 < ntok ? 0xffff0000u : 0u);
                  const uint32_t m89 = (2 * q2 + 8 < ntok ? 0xffffu : 0u) | (2 * q2 + 9 < ntok ? 0xffff0000u : 0u);
                  f[0] &= m01; f[1] &= m01; f[2] &= m89; f[3] &= m89;
                }
                r[4 * tt + 0] = f[0]; r[4 * tt + 1] = f[2]; r[4 * tt + 2] = f[1]; r[4 * tt + 3] = f[3];
              }
              tmem_st_16x256b_x8(tAV + ((uint32_t)(16 * mv) << 16), r);
            }
          }
          publish(j);
          if (WQ_TC_PROF_W != 99 && wl == (WQ_TC_PROF_W < 0 ? 0 : WQ_TC_PROF_W) && lane == 0) stamp(j, WQ_TC_PROF_W < 0 ? 1 : 4);
          if (WQ_TC_PROF_W == 99 && ts && lane == 0 && j < 23) ts[10 + 8 * j + wl] = clock64();
          // release the stages this piece no longer needs
          const int rel_end = (k0 + n == len[p]) ? nst[p] : (k0 + n) / cap;
          for (; released < rel_end; released++) {
            const int s_ = sg + released;
            if (lane == 0) mbar_arrive(&empty[s_ % NST]);
          }
        }
        sg += nst[p];
      };
      piece(std::integral_constant<int, 0>{});
      piece(std::integral_constant<int, 1>{});
      piece(std::integral_constant<int, 2>{});
      piece(std::integral_constant<int, 3>{});
      piece(std::integral_constant<int, 4>{});
    }
  } else {
    // =========================== softmax (warps 8..11) ===========================
    const int sq = warp - W_SMX;                   // TMEM lane quarter
    const int r = 32 * sq + lane;                  // token row (logits) / channel (epilogue)
    const int grp = a.grp;
    if (a.flags & WQ_DECODE_EARLY_) griddep_wait();   // outputs / workspace
    int *sflag = reinterpret_cast<int *>(sm + C::xch_off);           // [2][4]
    float *smax = reinterpret_cast<float *>(sflag + 8);              // [2][4][8]
    float *sred = smax + 64;                                         // [4][16]
    float m[8], ls[8], zs[8];
    int j = 0, e = -1;
    for (;;) {
      const int bf = j & 1;
      const uint32_t ph = (uint32_t)(j >> 1) & 1u;
      if (sq == 0) {
        mbar_wait_sleep(&deq_full[bf], ph, 32);
        if (!*reinterpret_cast<volatile int *>(&meta[bf].term)) {     // the terminator has no MMAs
          mbar_wait_sleep(&s_full[bf], ph, 20);
          if (j >= 2) mbar_wait_sleep(&o_done[bf], (uint32_t)((j - 2) >> 1) & 1u, 20);   // P' buffer free
        }
      }
      named_bar_sync(BAR_SMX, 128);
      tc_fence_after();
      const GMeta mt = meta[bf];
      if (mt.term) break;
      if (mt.first) {
        e++;
#pragma unroll
        for (int h = 0; h < 8; h++) { m[h] = -INFINITY; ls[h] = 0.f; zs[h] = 0.f; }
      }
      const int wi = r / S;
      const bool valid = r < mt.nvalid;
      // rows past nvalid (absent windows, masked rest tokens) read stale shared memory
      const float2 vs = valid ? reinterpret_cast<const float2 *>(sm + C::vp_off)[bf * 128 + r] : make_float2(0.f, 0.f);
      float z[8];
      {
        const float *zp = reinterpret_cast<const float *>(sm + C::zp_off) + bf * (C::BW * G * 8);
#pragma unroll
        for (int h = 0; h < 8; h++) z[h] = 0.f;
#pragma unroll
        for (int pp = 0; pp < C::BW; pp++) {
          const float4 z0 = *reinterpret_cast<const float4 *>(zp + (pp * G + wi) * 8);
          const float4 z1 = *reinterpret_cast<const float4 *>(zp + (pp * G + wi) * 8 + 4);
          z[0] += z0.x; z[1] += z0.y; z[2] += z0.z; z[3] += z0.w;
          z[4] += z1.x; z[5] += z1.y; z[6] += z1.z; z[7] += z1.w;
        }
      }
      if (r == 0 && WQ_TC_PROF_W < 0) stamp(j, 3);
      uint32_t sv[8];
      {
        const uint32_t tS = tmem + TM_S + bf * C::NK + ((uint32_t)(32 * sq) << 16);
        if constexpr (S >= 32) {
          tmem_ld_32x32b_x8(tS + 8 * ((32 * sq) / S), sv);
          tc_wait_ld();
        } else {
          uint32_t s16[16];
          tmem_ld_32x32b_x16(tS + 16 * sq, s16);
          tc_wait_ld();
#pragma unroll
          for (int h = 0; h < 8; h++) sv[h] = (lane < 16) ? s16[h] : s16[8 + h];
        }
      }
      float x[8];
      bool need = false;
#pragma unroll
      for (int h = 0; h < 8; h++) {
        x[h] = (valid && h < grp) ? (__uint_as_float(sv[h]) + z[h]) * a.scale_log2 : -INFINITY;
        need |= x[h] > m[h] + LAZY_TH || (m[h] == -INFINITY && x[h] > -INFINITY);
      }
      const int wneed = __any_sync(0xffffffffu, need);
      if (lane == 0) sflag[bf * 4 + sq] = wneed;
      named_bar_sync(BAR_SMX, 128);
      const int anyneed = sflag[bf * 4 + 0] | sflag[bf * 4 + 1] | sflag[bf * 4 + 2] | sflag[bf * 4 + 3];
      if (anyneed) {
        float mx[8];
#pragma unroll
        for (int h = 0; h < 8; h++) mx[h] = warp_max(x[h]);
        if (lane == 0) {
#pragma unroll
          for (int h = 0; h < 8; h++) smax[(bf * 4 + sq) * 8 + h] = mx[h];
        }
        named_bar_sync(BAR_SMX, 128);
        float al[8];
        bool resc = false;
#pragma unroll
        for (int h = 0; h < 8; h++) {
          float M = smax[(bf * 4) * 8 + h];
#pragma unroll
          for (int w = 1; w < 4; w++) M = fmaxf(M, smax[(bf * 4 + w) * 8 + h]);
          al[h] = 1.f;
          if (M > m[h] + LAZY_TH || (m[h] == -INFINITY && M > -INFINITY)) {
            al[h] = (m[h] == -INFINITY) ? 0.f : ex2f(m[h] - M);
            m[h] = M;
            resc = true;
          }
          ls[h] *= al[h];
          zs[h] *= al[h];
        }
        if (resc && !mt.first) {
          // O holds this entry's groups < j: wait for V(j - 1), rescale it in TMEM
          mbar_wait_hint(&o_done[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1u);
          tc_fence_after();
          const uint32_t tO = tmem + C::TM_O + (e & 1) * 8 + ((uint32_t)(32 * sq) << 16);
          uint32_t ov[8];
          tmem_ld_32x32b_x8(tO, ov);
          tc_wait_ld();
#pragma unroll
          for (int h = 0; h < 8; h++) ov[h] = __float_as_uint(__uint_as_float(ov[h]) * al[h]);
          tmem_st_32x32b_x8(tO, ov);
          tc_wait_st();
        }
      }
      uint32_t pk[4];
#pragma unroll
      for (int h = 0; h < 8; h += 2) {
        const float m0 = m[h] == -INFINITY ? 0.f : m[h], m1 = m[h + 1] == -INFINITY ? 0.f : m[h + 1];
        const float p0 = ex2f(x[h] - m0), p1 = ex2f(x[h + 1] - m1);
        ls[h] += p0; ls[h + 1] += p1;
        zs[h] = fmaf(p0, vs.y, zs[h]); zs[h + 1] = fmaf(p1, vs.y, zs[h + 1]);
        pk[h / 2] = pack_f2h2(p0 * vs.x, p1 * vs.x);
      }
      sts128(sm + C::bv_off + bf * 2048 + (16 * (r >> 4) + kpos16(r & 15)) * 16, make_uint4(pk[0], pk[1], pk[2], pk[3]));
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[bf]);
      if (r == 0 && WQ_TC_PROF_W < 0) stamp(j, 4);

      if (mt.last) {
        // ---------------- unit epilogue ----------------
        mbar_wait_hint(&o_done[bf], ph);
        tc_fence_after();
        uint32_t ov[8];
        tmem_ld_32x32b_x8(tmem + C::TM_O + (e & 1) * 8 + ((uint32_t)(32 * sq) << 16), ov);
        tc_wait_ld();
        tc_fence_before();
        // l and the V zero-point sums over the 128 token rows
        float rs[16];
#pragma unroll
        for (int h = 0; h < 8; h++) { rs[h] = ls[h]; rs[8 + h] = zs[h]; }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
          for (int i = 0; i < 16; i++) rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], off);
        if (lane == 0) {
#pragma unroll
          for (int i = 0; i < 16; i++) sred[sq * 16 + i] = rs[i];
        }
        named_bar_sync(BAR_SMX, 128);
        if (tid == W_SMX * 32) mbar_arrive(&ep_done[e & 1]);     // O buffer may be reused
        const int u = mt.u, c0 = mt.c0, c1 = mt.c1;
        const int b = u / a.H, h = u - b * a.H;
        const bool split = (c1 - c0) > 1;
        float *wslot = a.ws_part + (int64_t)(c + u) * grp * (D + 2);
        const int cc = r;                          // channel
        for (int jj = 0; jj < grp; jj++) {
          const float L = sred[jj] + sred[16 + jj] + sred[32 + jj] + sred[48 + jj];
          const float Z = sred[8 + jj] + sred[24 + jj] + sred[40 + jj] + sred[56 + jj];
          const float O = __uint_as_float(ov[jj]) + Z;
          const float M = m[jj];
          if (split) {
            if (cc == 0) { wslot[jj * (D + 2)] = M; wslot[jj * (D + 2) + 1] = L; }
            wslot[jj * (D + 2) + 2 + cc] = O;
          } else {
            const int64_t row = (int64_t)b * a.Hq + h * grp + jj;
            if (a.out) a.out[row * D + cc] = __float2half_rn(L > 0.f ? O / L : 0.f);
            if (a.partial) {
              float *pp = a.partial + row * (D + 2);
              if (cc == 0) { pp[0] = M * 0.69314718055994530942f; pp[1] = L; }
              pp[2 + cc] = O;
            }
          }
        }
        if (split) {
          named_bar_sync(BAR_SMX, 128);
          int *s_last = sflag + 8 + 64 + 64;       // spare word after sred (inside xch)
          if (r == 0) *s_last = (atom_add_acq_rel_gpu(a.ws_cnt + u, 1) == c1 - c0 - 1);
          named_bar_sync(BAR_SMX, 128);
          if (*s_last) merge_unit_rows(a, r, u, b, h, c0, c1);
        }
        named_bar_sync(BAR_SMX, 128);              // sred reused by the next entry
      }
      j++;
    }
  }
  // TMEM is released once every warp that touches it is done
  tc_fence_before();
  named_bar_sync(BAR_END, (NDQ + 4 + 1) * 32);
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc(tmem, 512);
  if (ts && tid == 0) ts[1] = clock64();
}

template <int S>
static cudaError_t launch_t(const DecodeArgs &a, int num_sms, cudaStream_t st) {
  using C = Cfg<S>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_decode_tc<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::total);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = C::total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (a.flags & WQ_DECODE_EARLY_) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, k_decode_tc<S>, a);
}

}  // namespace tcd

cudaError_t launch_decode_tc(const DecodeArgs &a, int num_sms, cudaStream_t st) {
  if (a.d != 128) return cudaErrorInvalidValue;
  switch (a.S) {
    case 16: return tcd::launch_t<16>(a, num_sms, st);
    case 32: return tcd::launch_t<32>(a, num_sms, st);
    case 64: return tcd::launch_t<64>(a, num_sms, st);
    case 128: return tcd::launch_t<128>(a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace wq
