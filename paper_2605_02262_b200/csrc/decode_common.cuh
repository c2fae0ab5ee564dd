// decode_common.cuh -- the split-KV work partition shared by the two decode kernels
// (decode.cu: mma.sync, the default for d = 64 and 128; decode_tc.cu: tcgen05/TMEM,
// d = 128, opt-in WQ_DECODE_TC=1): item geometry
// and cost model, the per-CTA plan computed in the prologue, the TMA producer that
// streams a CTA's items into the shared-memory ring, and the log-sum-exp merge of a
// split unit's CTA partials (Q24; Eq.12-13 P:462-473 make any split exact).
#pragma once
#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {

constexpr int MAX_UNITS = 1024;         // B * H
#ifndef WQ_DEC_MINCTA
#define WQ_DEC_MINCTA 98304   // A/B vs 49152: C2 9.43 -> 8.95 us (196608: 11.9, 393216: 20.3), C3/C5 unchanged
#endif
constexpr int64_t MIN_CTA_BYTES = WQ_DEC_MINCTA;   // least cost units per CTA (small calls use fewer CTAs)
constexpr uint32_t WQ_DECODE_EARLY_ = 1u;     // = WQ_DECODE_EARLY (include/wq.h)
constexpr uint32_t WQ_DECODE_GROUP_ = 2u;     // = WQ_DECODE_GROUP (include/wq.h)
constexpr int TS_PER_CTA = 200;        // debug & 8: per-CTA stamps + stage trace
#ifndef WQ_DEC_EOV
#define WQ_DEC_EOV 2000                // per-unit entry overhead in cost units of S*D/100
#endif
#ifndef WQ_DEC_C4
#define WQ_DEC_C4 174                  // 4-bit window cost, units of S*D/100 (2-bit: 156; r02 K2S refit 168 -> 174)
#endif
#ifndef WQ_DEC_C8
#define WQ_DEC_C8 204                  // 8-bit window cost (r02 refit: 233 -> 191, C5 -3.3 %, C3 -3.6 %; K2S refit -> 204)
#endif
#ifndef WQ_DEC_C16
#define WQ_DEC_C16 171                 // FP16 window cost, units of S*D/100 (r02 refit: 235 -> 171)
#endif
#ifndef WQ_DEC_CR
#define WQ_DEC_CR 40                   // FP16 rest tile (16 tokens) cost, units of D
#endif
#ifndef WQ_DEC_LOV
#define WQ_DEC_LOV 0                   // merge allowance of a split unit's last CTA, units of S*D/100
#endif
#ifndef WQ_DEC_SGAIN
#define WQ_DEC_SGAIN 8                 // least predicted makespan gain (%) for the stream split when units < CTAs
                                       // (with bit 0 of WQ_DEC_STREAM: A/B C3 37.8 -> 37.2 us, C5 33.75 -> 33.9,
                                       // C1 10.8 -> 11.1: left off)
#endif
#ifndef WQ_DEC_STREAM
#define WQ_DEC_STREAM 2                // cost-stream split: bit 0 when units < CTAs (measured slower,
                                       // DESIGN §5), bit 1 when units >= CTAs (C4, 256 units on 148
                                       // CTAs: whole units left 1.73 -> 2 units of makespan; C4 S=32
                                       // 121.6 -> 112.2 us, S=16 139.1 -> 127.0, S=128 127.8 -> 119.0)
#endif

// Compile-time item sizes and costs of a (D, S) instantiation.  Work is partitioned
// across CTAs in COST space, not bytes: every item costs its bytes plus a per-item
// compute term, so CTAs that get many narrow windows get fewer of them.
// TC selects the cost table of the tcgen05 kernel.
// FS > 1 (S = 128, d = 128: 64 KB FP16 records): an FP16 window is FS items of S/FS
// tokens each (its K tiles and V tiles of those tokens, copied as one (S/FS)-token FP16
// record), so a stage need not hold a whole 64 KB record and the ring keeps 4 stages.
template <int D, int S, bool TC = false, bool GRP = false, int FS = 1>
struct ItemGeo {
  // record bytes of class k (0..2 = 2/4/8-bit, 3 = FP16), D-1 contract (GRP: the 16-byte
  // parameter block of the paper-literal groups, reading Q37)
  static constexpr int64_t rb(int k) {
    return k == 3 ? 4LL * S * D : (int64_t)S * D * (2 << k) / 4 + (GRP ? 16LL : 4LL * D + 4LL * S);
  }
  static constexpr int REST_SZ = 64 * D;               // FP16 rest tile: 16 K rows + 16 V rows
  // item bytes: a record, an FS-th of an FP16 record, or a rest tile
  static constexpr int sz(int k) { return k == 4 ? REST_SZ : (k == 3 ? (int)(rb(3) / FS) : (int)rb(k)); }
  static constexpr int per_slot(int k) { return k == 3 ? FS : 1; }   // items per window slot
  // Cost of an item ~ its time on one SM inside a full decode launch.
  //  mma.sync kernel: measured per-class CTA-level item times on C5
  //   (tools/dbg_decode_time.py least-squares fit, round 2): 2-bit 0.136 us, 4-bit 0.147,
  //   8-bit 0.166, FP16 0.149 -> 156 : 168 : 191 : 171 in units of S*D/100 (round 1's
  //   156 : 170 : 233 : 235 left 8-bit-heavy CTAs idle ~7 us before the 2-bit ones);
  //   A/B over 4 tables: C5 34.96 -> 33.79 us, C3 38.81 -> 37.41 us, C4 unchanged.
  //   After the exact 2-bit K side (WQ_DEC_K2S: 2-bit windows 0.129 us, 4-bit 0.148, 8-bit
  //   0.176) 156 : 174 : 204 : 171 (A/B of 4 tables: C5 33.34 -> 32.84, C3 35.87 -> 35.71).
  //  tcgen05 kernel: the tensor work is asynchronous, an item costs its bytes plus
  //   a per-window dequantization term (same units).
  // fixed cost of one unit entry of a CTA (its epilogue, ~2 us: ~13 2-bit windows),
  // charged at the start of every unit in the cost-stream split
  static constexpr int64_t EOV = WQ_DEC_EOV * (int64_t)S * D / 100;
  static constexpr int64_t cost(int k) {
    if constexpr (TC) {
      return k == 4 ? 40LL * D
                    : (int64_t)(k == 0 ? 100 : k == 1 ? 140 : k == 2 ? 220 : 300) * S * D / 100;
    } else {
      return k == 4 ? (int64_t)WQ_DEC_CR * D
                    : (int64_t)(k == 0 ? 156 : k == 1 ? WQ_DEC_C4 : k == 2 ? WQ_DEC_C8 : WQ_DEC_C16) * S * D / 100 /
                          (k == 3 ? FS : 1);
    }
  }
};

// Geometry of one unit (request b, kv head h).
struct UnitGeo {
  int b, h, nslots, rl, ntiles;
  int so[5];
  int io[6];                            // item starts: classes 0-3 (FS items per FP16 slot), rest, end
  int64_t cs[5];                        // byte start of each class segment; cs[4] = image bytes
  int64_t cc[5];                        // cost start of each class segment; cc[4] = windows' cost
  double ccd[5];                        // cc as double (first_item: no int64 -> fp64 conversions)
};

template <int D, int S, bool TC, bool GRP = false, int FS = 1>
WQ_DEV void unit_geo(const DecodeArgs &a, int u, UnitGeo &g) {
  using IG = ItemGeo<D, S, TC, GRP, FS>;
  g.b = u / a.H;
  g.h = u - g.b * a.H;
  const int32_t *so = a.seg_off + 5 * g.b;
#pragma unroll
  for (int k = 0; k < 5; k++) g.so[k] = so[k];
  g.cs[0] = 0;
  g.cc[0] = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int64_t n = g.so[k + 1] - g.so[k];
    g.cs[k + 1] = g.cs[k] + n * IG::rb(k);
    g.cc[k + 1] = g.cc[k] + n * IG::per_slot(k) * IG::cost(k);
  }
  g.nslots = g.so[4];
  g.rl = a.rest_len ? a.rest_len[g.b] : 0;
  g.rl = g.rl < 0 ? 0 : (g.rl > a.R_max ? a.R_max : g.rl);     // contract: rest_len clamped to R_max
  g.ntiles = (g.rl + 15) / 16;
#pragma unroll
  for (int k = 0; k < 5; k++) g.ccd[k] = (double)g.cc[k];
#pragma unroll
  for (int k = 0; k < 4; k++) g.io[k] = g.so[k];
  g.io[4] = g.so[3] + FS * (g.so[4] - g.so[3]);
  g.io[5] = g.io[4] + g.ntiles;
}
template <int D, int S, bool TC, bool GRP = false, int FS = 1>
WQ_DEV int64_t unit_cost(const UnitGeo &g) {
  return g.cc[4] + (int64_t)g.ntiles * ItemGeo<D, S, TC, GRP, FS>::cost(4);
}

// first item whose start (in cost units, relative to the unit) is >= x.  Planning
// arithmetic runs in double (no 64-bit integer division on the producer's path);
// every CTA evaluates the same expressions, so neighbouring CTAs agree on the cut.
template <int D, int S, bool TC, bool GRP = false, int FS = 1>
WQ_DEV int first_item(const UnitGeo &g, double x) {
  using IG = ItemGeo<D, S, TC, GRP, FS>;
  if (x <= 0.0) return 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    if (x <= g.ccd[k]) return g.io[k];
    // (a multiply by the compile-time reciprocal: a DDIV is a long dependent sequence on
    // the producer's start-up path; every CTA evaluates the same expression)
    if (x < g.ccd[k + 1]) return g.io[k] + (int)ceil((x - g.ccd[k]) * (1.0 / (double)IG::cost(k)));
  }
  if (x <= g.ccd[4]) return g.io[4];
  const int t = (int)ceil((x - g.ccd[4]) * (1.0 / (double)IG::cost(4)));
  return g.io[4] + (t < g.ntiles ? t : g.ntiles);
}

// Stage plan of one unit's item range [i0, i1): five "pieces" (the width-class
// segments 2|4|8|16 and the FP16 rest tiles), each cut into stages of CAP(p)
// equal-size items.  Producer and consumers walk the same plan.
struct UnitPlan {
  int lo[5], hi[5], nst[5];
};
template <int D, int S, bool TC, int STAGE, bool GRP = false, int FS = 1>
WQ_DEV void plan_unit(const UnitGeo &g, int i0, int i1, UnitPlan &pl) {
  using IG = ItemGeo<D, S, TC, GRP, FS>;
#pragma unroll
  for (int p = 0; p < 5; p++) {
    const int a0 = g.io[p];
    const int a1 = g.io[p + 1];
    const int lo = i0 > a0 ? i0 : a0;
    const int hi = i1 < a1 ? i1 : a1;
    const int cap = STAGE / IG::sz(p);
    pl.lo[p] = lo;
    pl.hi[p] = hi > lo ? hi : lo;
    pl.nst[p] = (pl.hi[p] - pl.lo[p] + cap - 1) / cap;
  }
}

// A CTA's work is a list of "entries" (unit u, items [i0, i1) of it).  The producer
// lane publishes each entry's stage plan in a small shared ring and streams its
// stages; consumers walk the same stages in order.
struct Entry {
  int u, n_u, c0, c1, rl, nslots, tag;
  int lo[5], len[5], nst[5];
};
// This CTA's share, planned in the prologue by one warp (lane-parallel): units
// [ua, ub) whole, or one unit split over CTAs [c0, c1) of which this CTA takes
// items [i0, i1).
struct CtaPlan {
  int ua, ub, split, c0, c1, i0, i1;   // split: 0 whole units, 1 one unit over [c0, c1), 2 cost stream
  double lo, hi;                       // split 2: this CTA's range [lo, hi) of the units' cost stream
  int G;                               // CTAs that get work
  int geo_ok;                           // geo/img_off of unit ua valid (handed over by the planner)
  int64_t img_off;
  UnitGeo geo;
};

// ---- prologue (one warp): unit cost prefix ustart[U+1], then this CTA's share ----
// Writes *cp and *s_flag = G (number of CTAs that get work).
// STREAM (fewer units than CTAs): CTA c takes the cost range [T c/G, T (c+1)/G) of the
// units laid end to end, each unit's cost preceded by a fixed entry overhead EOV (its
// epilogue: a CTA that ends one unit and starts the next runs two), so every CTA gets
// the same cost; a unit-aligned split rounds each unit to a whole number of CTAs.
// vc / vn: this CTA's index and the CTA count of the grid it plans over (blockIdx.x /
// gridDim.x, or a virtual rank's share of one grid in the fused-merge emulation).
template <int D, int S, bool TC, int STREAM = 0, bool GRP = false, int FS = 1>
WQ_DEV void plan_cta(const DecodeArgs &a, int64_t *ustart, CtaPlan *cp, int *s_flag, int lane, int vc, int vn) {
  const int U = a.B * a.H;
  int64_t carry = 0;
  UnitGeo gg;                                   // this lane's unit of the last chunk
  int64_t ioff = 0;
  for (int base = 0; base < U; base += 32) {
    const int u = base + lane;
    int64_t v = 0;
    if (u < U) {
      ioff = a.offs[u];
      unit_geo<D, S, TC, GRP, FS>(a, u, gg);
      v = unit_cost<D, S, TC, GRP, FS>(gg) + (STREAM ? ItemGeo<D, S, TC, GRP, FS>::EOV : 0);
    }
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (u < U) ustart[u] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) ustart[U] = carry;
  __syncwarp();
  const int64_t T = carry;
  const double invT = T > 0 ? 1.0 / (double)T : 0.0;
  int G = (int)((double)T * (1.0 / (double)MIN_CTA_BYTES));
  G = G < 1 ? 1 : (G > vn ? vn : G);
  const int c = vc;
  bool stream = (STREAM & (U >= G ? 2 : 1)) != 0;
  if (stream && U < G && T > 0) {
    // units < CTAs: the unit-aligned split gives unit u n_u = c0(u+1) - c0(u) CTAs (below);
    // stream only if its makespan T/G beats max_u cost_u/n_u by the margin WQ_DEC_SGAIN %
    // (a CTA spanning two units runs two epilogues: C5, 9-10 CTAs per unit, stays aligned;
    // C3, 2-3 CTAs per unit, streams)
    const int64_t extra = G - U;
    double mk = 0.0;
    for (int base = 0; base < U; base += 32) {
      const int u = base + lane;
      if (u < U) {
        const int c0u = u + (int)rint((double)ustart[u] * extra * invT);
        const int c1u = (u + 1 < U) ? (u + 1) + (int)rint((double)ustart[u + 1] * extra * invT) : G;
        const double cu = (double)(ustart[u + 1] - ustart[u]);
        mk = fmax(mk, cu / (double)(c1u > c0u ? c1u - c0u : 1));
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mk = fmax(mk, __shfl_xor_sync(0xffffffffu, mk, o));
    stream = (double)T * (1.0 + WQ_DEC_SGAIN / 100.0) < mk * (double)G;
  }
  if ((U >= G && !stream) || T <= 0) {
    // whole units to the CTA owning their cost midpoint: a contiguous unit range
    int ua = 0, ub = 0;
    for (int base = 0; base < U; base += 32) {
      const int u = base + lane;
      int own = G;
      if (u < U) {
        const int64_t mid = ustart[u] + (ustart[u + 1] - ustart[u]) / 2;
        own = T > 0 ? (int)((double)mid * G * invT) : 0;
        own = own >= G ? G - 1 : own;
      }
      ua += __popc(__ballot_sync(0xffffffffu, own < c));
      ub += __popc(__ballot_sync(0xffffffffu, own <= c));
    }
    if (lane == 0) { cp->ua = ua; cp->ub = ub; cp->split = 0; cp->c0 = c; cp->c1 = c + 1; }
  } else if (stream) {
    const double Td = (double)T;
    const double lo = Td * c / G, hi = Td * (c + 1) / G;
    int ua = 0, ub = 0;
    for (int base = 0; base < U; base += 32) {
      const int u = base + lane;
      bool before = false, starts = false;
      if (u < U) {
        const double us = (double)ustart[u], ue = (double)ustart[u + 1];
        before = ue <= lo;                       // units have cost >= EOV > 0
        starts = us < hi;
      }
      ua += __popc(__ballot_sync(0xffffffffu, before));
      ub += __popc(__ballot_sync(0xffffffffu, starts));
    }
    if (lane == 0) { cp->ua = ua; cp->ub = ub; cp->split = 2; cp->c0 = c; cp->c1 = c + 1; cp->lo = lo; cp->hi = hi; }
  } else {
    // every unit gets 1 + its cost share of the G - U extra CTAs: unit u owns
    // CTAs [c0(u), c0(u+1)), c0(U) = G
    const int64_t extra = G - U;
    int cnt = 0;
    for (int base = 0; base < U; base += 32) {
      const int u = base + lane;
      const int c0u = u < U ? u + (int)rint((double)ustart[u] * extra * invT) : G;
      cnt += __popc(__ballot_sync(0xffffffffu, u < U && c0u <= c));
    }
    const int u = cnt - 1;                      // c0(0) = 0 <= c: u >= 0
    if (lane == 0) {
      const int c0 = u + (int)rint((double)ustart[u] * extra * invT);
      const int c1 = (u + 1 < U) ? (u + 1) + (int)rint((double)ustart[u + 1] * extra * invT) : G;
      cp->ua = u; cp->ub = u + 1; cp->split = c1 - c0 > 1; cp->c0 = c0; cp->c1 = c1;
    }
  }
  __syncwarp();
  const int ua = cp->ua;
  const int last_base = ((U - 1) / 32) * 32;
  if (lane == 0) cp->geo_ok = 0;
  __syncwarp();
  if (ua < U && ua >= last_base && lane == ua - last_base) {
    cp->geo = gg;
    cp->img_off = ioff;
    cp->geo_ok = 1;
  }
  if (lane == 0) { *s_flag = G; cp->G = G; }
  __syncwarp();
  // a unit split over CTAs [c0, c1): this CTA's item range, i0 by lane 0 and i1 by lane 1
  // in parallel (the producer's start-up path otherwise runs both searches back to back)
  if (cp->split == 1 && cp->geo_ok && lane < 2) {
    const UnitGeo &g0 = cp->geo;
    const int k = c - cp->c0, n = cp->c1 - cp->c0;
    const double lov = (double)WQ_DEC_LOV * S * D / 100;
    const double share = ((double)(ustart[ua + 1] - ustart[ua]) + lov) * (1.0 / (double)n);
    const int kk = k + lane;
    const int v = (lane == 1 && k == n - 1) ? g0.io[5] : first_item<D, S, TC, GRP, FS>(g0, share * kk);
    if (lane == 0) cp->i0 = v;
    else cp->i1 = v;
  }
}

// ---- producer (one lane): stream the CTA's entries into the ring ----
// Stages of NST x STAGE bytes, full[s] (1 arrival + tx bytes) / empty[s] barriers;
// entries published in a ring of NUS Entry slots, released via *units_done.
template <int D, int S, bool TC, int STAGE, int NST, int NUS, bool GRP = false, int FS = 1>
WQ_DEV void produce(const DecodeArgs &a, const CtaPlan &P, const int64_t *ustart, uint8_t *ring,
                    uint64_t *full, uint64_t *empty, Entry *ent, int *units_done, uint64_t *ts, int vc) {
  using IG = ItemGeo<D, S, TC, GRP, FS>;
  const int c = vc;
  const uint64_t pol = policy_evict_first();
  if (ts) { ts[62] = gtime(); ts[55] = clock64(); }
  int sg = 0;                                  // stage number of this CTA
  int uix = 0;                                 // entry number of this CTA
  auto publish = [&](int u, int n_u, const UnitGeo *gg, const UnitPlan *pl, int ec0, int ec1) {
    while (*reinterpret_cast<volatile int *>(units_done) < uix - (NUS - 1)) {
    }
    Entry &d = ent[uix % NUS];
    d.u = u;
    d.n_u = n_u;
    d.c0 = ec0;
    d.c1 = ec1;
    d.rl = gg ? gg->rl : 0;
    d.nslots = gg ? gg->io[4] : 0;               // items before the rest tiles
#pragma unroll
    for (int pp = 0; pp < 5; pp++) {
      d.lo[pp] = pl ? pl->lo[pp] : 0;
      d.len[pp] = pl ? pl->hi[pp] - pl->lo[pp] : 0;
      d.nst[pp] = pl ? pl->nst[pp] : 0;
    }
    __threadfence_block();
    *reinterpret_cast<volatile int *>(&d.tag) = uix;
    if (ts && uix == 0) ts[60] = gtime();
    uix++;
  };
  for (int u = P.ua; u < P.ub; u++) {
    int64_t img_off;
    UnitGeo gl;
    const bool first = u == P.ua && P.geo_ok;
    if (first) {
      img_off = P.img_off;                     // from the prologue: no global round trip
    } else {
      img_off = a.offs[u];
      unit_geo<D, S, TC, GRP, FS>(a, u, gl);
    }
    const UnitGeo &gg = first ? P.geo : gl;    // (the prologue's copy read in place)
    if (ts && u == P.ua) ts[57] = clock64();
    int i0 = 0, i1 = gg.io[5];
    int ec0 = P.split == 1 ? P.c0 : c, ec1 = P.split == 1 ? P.c1 : c + 1;
    if (P.split == 1 && first) {
      i0 = P.i0;                                 // planned in the prologue (plan_cta)
      i1 = P.i1;
    } else if (P.split == 1) {
      // the unit's cost plus the last CTA's merge allowance, cut into n equal shares: the
      // last CTA (the merger: it ends with the unit's FP16 windows and rest tiles, then
      // merges every partial) gets LOV less item cost than the others
      const double lov = (double)WQ_DEC_LOV * S * D / 100;
      const double ucost = (double)(ustart[u + 1] - ustart[u]) + lov;
      const int k = c - P.c0, n = P.c1 - P.c0;
      const double share = ucost * (1.0 / (double)n);
      i0 = first_item<D, S, TC, GRP, FS>(gg, share * k);
      if (k < n - 1) i1 = first_item<D, S, TC, GRP, FS>(gg, share * (k + 1));
    } else if (P.split == 2) {
      // this CTA's slice of unit u (items start EOV into the unit's cost range) and the
      // CTAs [ec0, ec1) sharing the unit; every CTA evaluates the same expressions
      const double us = (double)ustart[u], ue = (double)ustart[u + 1];
      const double eov = (double)ItemGeo<D, S, TC, GRP, FS>::EOV;
      const double Td = (double)ustart[a.B * a.H];
      const int Gp = P.G;
      auto Bk = [&](int k) { return Td * k / Gp; };
      if (P.lo > us) i0 = first_item<D, S, TC, GRP, FS>(gg, P.lo - us - eov);
      if (P.hi < ue) i1 = first_item<D, S, TC, GRP, FS>(gg, P.hi - us - eov);
      int k0 = (int)(us * Gp / Td);
      k0 = k0 < 0 ? 0 : (k0 > Gp - 1 ? Gp - 1 : k0);
      while (k0 + 1 < Gp && Bk(k0 + 1) <= us) k0++;
      while (k0 > 0 && Bk(k0) > us) k0--;
      int k1 = (int)(ue * Gp / Td);
      k1 = k1 < 0 ? 0 : (k1 > Gp - 1 ? Gp - 1 : k1);
      while (k1 > 0 && Bk(k1) >= ue) k1--;
      while (k1 + 1 < Gp && Bk(k1 + 1) < ue) k1++;
      ec0 = k0;
      ec1 = k1 + 1;
    }
    if (ts && u == P.ua) ts[58] = clock64();
    UnitPlan pl;
    plan_unit<D, S, TC, STAGE, GRP, FS>(gg, i0, i1, pl);
    if (ts && sg == 0) ts[56] = clock64();
    bool published = false;
    const uint8_t *img = a.packed + img_off;
    const __half *kr = a.k_rest + gg.b * a.rs_b + gg.h * a.rs_h;
    const __half *vr = a.v_rest + gg.b * a.rs_b + gg.h * a.rs_h;
#pragma unroll
    for (int p = 0; p < 5; p++) {
      const int cap = STAGE / IG::sz(p);
      for (int t = 0; t < pl.nst[p]; t++, sg++) {
        const int slot = sg % NST;
        const uint32_t fill = (uint32_t)(sg / NST);
        const int f0 = pl.lo[p] + t * cap;
        const int f1 = min(pl.hi[p], f0 + cap);
        mbar_wait_sleep(&empty[slot], (fill & 1) ^ 1, 64);
        if (ts && sg < 64) ts[72 + sg] = clock64();
        uint8_t *dst = ring + (size_t)slot * STAGE;
        if (p < 4 && (p < 3 || FS == 1)) {
          const uint32_t nb = (uint32_t)(f1 - f0) * IG::sz(p);
          WQ_CHECK(f0 >= gg.so[p] && f1 <= gg.so[p + 1] && nb <= (uint32_t)STAGE);
          WQ_CHECK(img_off + gg.cs[p] + (int64_t)(f1 - gg.so[p]) * IG::sz(p) <= a.offs[a.B * a.H]);
          WQ_CHECK(img_off + gg.cs[4] <= a.offs[u + 1]);
          mbar_arrive_expect_tx(&full[slot], nb);
          bulk_g2s_evict_first(dst, img + gg.cs[p] + (int64_t)(f0 - gg.so[p]) * IG::sz(p), nb, &full[slot], pol);
        } else if (p == 3) {
          // FP16 sub-items: item f = part (f - io[3]) % FS of window slot so[3] + (f - io[3]) / FS;
          // its K tiles and V tiles are copied back to back (an (S/FS)-token FP16 record)
          constexpr uint32_t HB = (uint32_t)(2 * S * D / FS);          // K (or V) bytes of a part
          mbar_arrive_expect_tx(&full[slot], (uint32_t)(f1 - f0) * 2u * HB);
          for (int f = f0; f < f1; f++) {
            const int wi = (f - gg.io[3]) / FS, part = (f - gg.io[3]) - wi * FS;
            const uint8_t *rec = img + gg.cs[3] + (int64_t)wi * IG::rb(3);
            WQ_CHECK(gg.so[3] + wi < gg.so[4] && (uint32_t)(f - f0 + 1) * 2u * HB <= (uint32_t)STAGE);
            uint8_t *di = dst + (size_t)(f - f0) * 2 * HB;
            bulk_g2s_evict_first(di, rec + (size_t)part * HB, HB, &full[slot], pol);
            bulk_g2s_evict_first(di + HB, rec + 2 * (size_t)S * D + (size_t)part * HB, HB, &full[slot], pol);
          }
        } else {
          // rest tiles [f0, f1) = rows [r0, r1): one bulk copy for K, one for V
          // (the rest buffers may be written by the preceding work: wait for it)
          if (a.flags & WQ_DECODE_EARLY_) griddep_wait();
          const int r0 = 16 * (f0 - gg.io[4]);
          const int r1 = min(gg.rl, 16 * (f1 - gg.io[4]));
          const uint32_t nb = (uint32_t)(r1 - r0) * 2u * D;
          WQ_CHECK(r0 >= 0 && r1 <= a.R_max && 2u * (uint32_t)cap * 32u * D <= (uint32_t)STAGE);
          mbar_arrive_expect_tx(&full[slot], 2 * nb);
          bulk_g2s_evict_first(dst, kr + (int64_t)r0 * D, nb, &full[slot], pol);
          bulk_g2s_evict_first(dst + cap * 32 * D, vr + (int64_t)r0 * D, nb, &full[slot], pol);
        }
        if (!published) { publish(u, i1 - i0, &gg, &pl, ec0, ec1); published = true; }
      }
    }
    if (!published) publish(u, i1 - i0, &gg, &pl, ec0, ec1);
  }
  publish(-1, 0, nullptr, nullptr, c, c + 1);   // terminator
  if (ts) ts[2] = gtime();
}

// ---- outputs of one 16-byte group of a unit's merged result ----
// Group gi = mt*32 + L (L = g*4 + q of the consumer fragment): channels 16mt + g, +8,
// heads 2q, 2q + 1: O = (ch0, j0), (ch0, j1), (ch1, j0), (ch1, j1); M, L per head (log2
// domain max, sum).  Writes out (fp16 O / L) and the ABI partial (m in natural log, l, o).
template <int D>
WQ_DEV void write_group(const DecodeArgs &a, int b, int h, int gi, float4 O, float2 M, float2 L) {
  const int mt = gi >> 5, ln = gi & 31, gg = ln >> 2, jq = 2 * (ln & 3);
  const int ch0 = 16 * mt + gg, ch1 = ch0 + 8;
  const float ov[4] = {O.x, O.y, O.z, O.w};
#pragma unroll
  for (int e = 0; e < 4; e++) {
    const int j = jq + (e & 1), ch = (e & 2) ? ch1 : ch0;
    if (j >= a.grp) continue;
    const float Lj = (e & 1) ? L.y : L.x, Mj = (e & 1) ? M.y : M.x;
    const int64_t row = (int64_t)b * a.Hq + h * a.grp + j;
    if (a.out) a.out[row * D + ch] = __float2half_rn(Lj > 0.f ? ov[e] / Lj : 0.f);
    if (a.partial) {
      float *pp = a.partial + row * (D + 2);
      if (ch == 0) { pp[0] = Mj * 0.69314718055994530942f; pp[1] = Lj; }
      pp[2 + ch] = ov[e];
    }
  }
}

// ---- last-CTA merge of a split unit (NT threads, thread index tid) ----
// CTA partial slot (PSLOT floats): [8 heads] (M, L) pairs, then the 16-byte o groups.
// One thread per group: the np partials' (M, L) of its two heads and its o group are
// loaded 8 partials at a time (every load of a batch in flight at once: one L2 round
// trip per batch), combined by log-sum-exp in registers, and written out.
#ifndef WQ_DEC_MB
#define WQ_DEC_MB 12                 // partials per load batch of the last-CTA merge (A/B: 12 > 8)
#endif
template <int D, int NT, int PSLOT>
WQ_DEV void merge_unit(const DecodeArgs &a, int tid, int u, int b, int h, int c0, int c1) {
  constexpr int NG = D * 2;                    // groups (KT * 32)
  constexpr int MB = WQ_DEC_MB;
  const int np = c1 - c0;
  const float *pb = a.ws_part + (int64_t)(c0 + u) * PSLOT;
  for (int gi = tid; gi < NG; gi += NT) {
    const int jq = 2 * (gi & 3);
    float2 M = make_float2(-INFINITY, -INFINITY), L = make_float2(0.f, 0.f);
    float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p0 = 0; p0 < np; p0 += MB) {
      float4 ml[MB], ov[MB];
#pragma unroll
      for (int i = 0; i < MB; i++) {
        if (p0 + i < np) {
          const float *ps = pb + (int64_t)(p0 + i) * PSLOT;
          ml[i] = __ldcg(reinterpret_cast<const float4 *>(ps + 2 * jq));       // (M, L) of jq, jq + 1
          ov[i] = __ldcg(reinterpret_cast<const float4 *>(ps + 16 + gi * 4));
        } else {
          ml[i] = make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
          ov[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      float2 Mn = M;
#pragma unroll
      for (int i = 0; i < MB; i++) {
        if (ml[i].y > 0.f) Mn.x = fmaxf(Mn.x, ml[i].x);
        if (ml[i].w > 0.f) Mn.y = fmaxf(Mn.y, ml[i].z);
      }
      const float r0 = Mn.x == -INFINITY ? 0.f : ex2f(M.x - Mn.x);
      const float r1 = Mn.y == -INFINITY ? 0.f : ex2f(M.y - Mn.y);
      L.x *= r0; O.x *= r0; O.z *= r0;
      L.y *= r1; O.y *= r1; O.w *= r1;
#pragma unroll
      for (int i = 0; i < MB; i++) {
        const float f0 = ml[i].y > 0.f ? ex2f(ml[i].x - Mn.x) : 0.f;
        const float f1 = ml[i].w > 0.f ? ex2f(ml[i].z - Mn.y) : 0.f;
        L.x = fmaf(f0, ml[i].y, L.x);
        L.y = fmaf(f1, ml[i].w, L.y);
        O.x = fmaf(f0, ov[i].x, O.x);
        O.y = fmaf(f1, ov[i].y, O.y);
        O.z = fmaf(f0, ov[i].z, O.z);
        O.w = fmaf(f1, ov[i].w, O.w);
      }
      M = Mn;
    }
    write_group<D>(a, b, h, gi, O, M, L);
  }
  if (tid == 0) a.ws_cnt[u] = 0;
}

// Exact fp16 value pair of pair-slot P (compile-time after unrolling) of a lane chunk
// (CENTER: code - 2^(BITS-1), the V side).
template <int BITS, bool CENTER = false>
WQ_DEV uint32_t deq_pair(const uint32_t *wd, int P) {
  constexpr int PPW = 16 / BITS;
  const uint32_t w = wd[P / PPW];
  if constexpr (BITS == 16) {
    return w;
  } else if constexpr (BITS == 8) {
    return (P % 2) == 0 ? dq_pair8<0, CENTER>(w) : dq_pair8<1, CENTER>(w);
  } else if constexpr (BITS == 4) {
    const uint32_t w8 = w >> 8;
    switch (P % 4) {
      case 0: return dq_pair<4, 0, CENTER>(w, w8);
      case 1: return dq_pair<4, 1, CENTER>(w, w8);
      case 2: return dq_pair<4, 2, CENTER>(w, w8);
      default: return dq_pair<4, 3, CENTER>(w, w8);
    }
  } else {
    const uint32_t w8 = w >> 8;
    switch (P % 8) {
      case 0: return dq_pair<2, 0, CENTER>(w, w8);
      case 1: return dq_pair<2, 1, CENTER>(w, w8);
      case 2: return dq_pair<2, 2, CENTER>(w, w8);
      case 3: return dq_pair<2, 3, CENTER>(w, w8);
      case 4: return dq_pair<2, 4, CENTER>(w, w8);
      case 5: return dq_pair<2, 5, CENTER>(w, w8);
      case 6: return dq_pair<2, 6, CENTER>(w, w8);
      default: return dq_pair<2, 7, CENTER>(w, w8);
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

}  // namespace wq
