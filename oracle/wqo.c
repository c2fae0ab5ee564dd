/*
 * wqo.c — CPU ORACLE (test infrastructure; see wqo.h for the rules).
 * Plain C99, fp64 unless the contract fixes fp32.  Build:
 *   gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC wqo.c -lm
 */
#include "wqo.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* fp16 <-> float, written out from the IEEE 754 binary16 definition          */
/* ------------------------------------------------------------------------ */
double wqo_f16_to_f64(uint16_t h) {
  int sign = (h >> 15) & 1;
  int e = (h >> 10) & 31;
  int m = h & 1023;
  double v;
  if (e == 0) v = ldexp((double)m, -24);                  /* subnormal / zero */
  else if (e == 31) v = (m == 0) ? INFINITY : NAN;
  else v = ldexp((double)(1024 + m), e - 25);            /* (1 + m/1024) * 2^(e-15) */
  return sign ? -v : v;
}

/* Encode a non-negative magnitude that is exactly representable in fp16
 * (or >= 65536, which becomes infinity). */
static uint16_t enc_mag(double a) {
  if (a == 0.0) return 0;
  if (a > 65504.0) return 0x7C00;
  if (a < ldexp(1.0, -14)) return (uint16_t)(a / ldexp(1.0, -24));   /* subnormal */
  int e2; frexp(a, &e2);                                 /* a = f * 2^e2, f in [0.5,1) */
  int e = e2 - 1;                                        /* a in [2^e, 2^(e+1)) */
  int mant = (int)(a / ldexp(1.0, e - 10)) - 1024;
  return (uint16_t)(((e + 15) << 10) | mant);
}

/* The fp16 quantum (ulp) at magnitude a (a > 0, a < 65536). */
static double quantum(double a) {
  if (a < ldexp(1.0, -14)) return ldexp(1.0, -24);
  int e2; frexp(a, &e2);
  return ldexp(1.0, (e2 - 1) - 10);
}

uint16_t wqo_f32_to_f16_ru(float xf) {
  double x = (double)xf;
  if (isnan(x)) return 0x7E00;
  uint16_t sign = (x < 0 || (x == 0 && signbit(x))) ? 0x8000 : 0;
  double a = fabs(x);
  if (isinf(x)) return sign | 0x7C00;
  if (a == 0.0) return sign;
  if (a >= 65536.0) return sign ? (uint16_t)(0x8000 | 0x7BFF) : 0x7C00;
  double qu = quantum(a);
  double t = floor(a / qu) * qu;                         /* magnitude truncated to fp16 */
  if (t != a && !sign) t += qu;                          /* round up (toward +inf) */
  uint16_t r = enc_mag(t);
  if (sign && (r & 0x7FFF) == 0) return 0x8000;          /* -0 */
  return sign | r;
}

uint16_t wqo_f32_to_f16_rn(float xf) {
  double x = (double)xf;
  if (isnan(x)) return 0x7E00;
  uint16_t sign = signbit(x) ? 0x8000 : 0;
  double a = fabs(x);
  if (isinf(x)) return sign | 0x7C00;
  if (a >= 65520.0) return sign | 0x7C00;                /* halfway to 2^16 rounds to inf */
  if (a == 0.0) return sign;
  double qu = quantum(a);
  double n = floor(a / qu);
  double rem = a / qu - n;                               /* exact: a/qu is a dyadic */
  if (rem > 0.5 || (rem == 0.5 && fmod(n, 2.0) == 1.0)) n += 1.0;
  return sign | enc_mag(n * qu);
}

uint16_t wqo_f64_to_f16_rn(double x) {
  if (isnan(x)) return 0x7E00;
  uint16_t sign = signbit(x) ? 0x8000 : 0;
  double a = fabs(x);
  if (isinf(x)) return sign | 0x7C00;
  if (a >= 65520.0) return sign | 0x7C00;                /* halfway to 2^16 rounds to inf */
  if (a == 0.0) return sign;
  double qu = quantum(a);
  double n = floor(a / qu);
  double rem = a / qu - n;                               /* exact for dyadic a */
  if (rem > 0.5 || (rem == 0.5 && fmod(n, 2.0) == 1.0)) n += 1.0;
  return sign | enc_mag(n * qu);
}

/* ------------------------------------------------------------------------ */
/* Eq.10-11, readings Q9 (n widths) and Q10 (clamp s, alpha > 0)  */
/* ------------------------------------------------------------------------ */
double wqo_f1(double s, double alpha) { return (exp(alpha * s) - 1.0) / (exp(alpha) - 1.0); }
double wqo_f2(double s, double alpha) { return (exp(-alpha * s) - 1.0) / (exp(-alpha) - 1.0); }

int wqo_thresholds(const double *s, int32_t L, double alpha, int32_t n, double *thr) {
  if (!(alpha > 0.0) || !isfinite(alpha) || n < 1 || n > 4 || L < 1) return 1;
  for (int l = 0; l < L; l++) {
    double sl = s[l];
    if (sl < 0.0) sl = 0.0;
    if (sl > 1.0) sl = 1.0;
    double lo = wqo_f1(sl, alpha), hi = wqo_f2(sl, alpha);
    double *t = thr + (int64_t)l * (n - 1);
    if (n == 2) t[0] = (lo + hi) / 2.0;
    if (n == 3) { t[0] = lo; t[1] = hi; }
    if (n == 4) { t[0] = lo; t[1] = (lo + hi) / 2.0; t[2] = hi; }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Eq.8: mean over the S*N (text, window) token pairs of cosine.  */
/* Zero-norm rows contribute 0 (Q5).  Literal double sum, j outer, k inner.   */
/* ------------------------------------------------------------------------ */
static double row_norm(const uint16_t *x, int32_t D) {
  double acc = 0.0;
  for (int c = 0; c < D; c++) { double v = wqo_f16_to_f64(x[c]); acc += v * v; }
  return sqrt(acc);
}

double wqo_window_score(const uint16_t *vis_b, int64_t vrs, const uint16_t *txt_b, int64_t trs,
                        int32_t N, int32_t D, int32_t S, int32_t w) {
  double sum = 0.0;
  for (int j = 0; j < N; j++) {
    const uint16_t *t = txt_b + (int64_t)j * trs;
    double nt = row_norm(t, D);
    for (int k = 0; k < S; k++) {
      const uint16_t *v = vis_b + (int64_t)(w * S + k) * vrs;
      double nv = row_norm(v, D);
      if (nt == 0.0 || nv == 0.0) continue;
      double dot = 0.0;
      for (int c = 0; c < D; c++) dot += wqo_f16_to_f64(t[c]) * wqo_f16_to_f64(v[c]);
      sum += dot / (nt * nv);
    }
  }
  return sum / ((double)S * (double)N);
}

void wqo_window_scores(const uint16_t *vis, int64_t vrs, int64_t vbs,
                       const uint16_t *txt, int64_t trs, int64_t tbs,
                       int32_t B, int32_t M, int32_t N, int32_t D, int32_t S, double *scores) {
  int32_t W = M / S;
#pragma omp parallel for schedule(dynamic)
  for (int64_t i = 0; i < (int64_t)B * W; i++) {
    int b = (int)(i / W), w = (int)(i % W);
    scores[i] = wqo_window_score(vis + b * vbs, vrs, txt + b * tbs, trs, N, D, S, w);
  }
}

/* ------------------------------------------------------------------------ */
/* Alg.1 lines 8-16 + P:322 pin + P:395 vote + Q13 budget; Alg.2 partition    */
/* ------------------------------------------------------------------------ */
static const int CLASS_BITS[4] = {2, 4, 8, 16};
static int class_of(int bits) { return bits == 2 ? 0 : bits == 4 ? 1 : bits == 8 ? 2 : 3; }

/* Q8: boundaries fall in the middle band(s). */
static int band_level(double x, const double *T, int n) {
  if (n == 1) return 0;
  if (n == 2) return x > T[0] ? 1 : 0;
  int level = 0;
  if (x >= T[0]) level++;
  for (int j = 1; j < n - 2; j++) if (x >= T[j]) level++;
  if (x > T[n - 2]) level++;
  return level;
}

static const double *g_sort_keys;
static int cmp_rank(const void *a, const void *b) {      /* (-score, index) order, Q7 */
  int i = *(const int *)a, j = *(const int *)b;
  double si = g_sort_keys[i], sj = g_sort_keys[j];
  if (si > sj) return -1;
  if (si < sj) return 1;
  return (i > j) - (i < j);
}

/* rank_of[w] for keys[0..W) */
static void rank_windows(const double *keys, int W, int *order, int *rank_of) {
  for (int w = 0; w < W; w++) order[w] = w;
  g_sort_keys = keys;
  qsort(order, W, sizeof(int), cmp_rank);
  for (int r = 0; r < W; r++) rank_of[order[r]] = r;
}

/* Q13: while over budget, demote the lowest-ranked non-pinned window whose
 * width is above the smallest width by one width step. */
static void apply_budget(uint8_t *bits, int W, const int *rank_of, const int *order,
                         const wqo_geom *g, double budget, int pin) {
  (void)rank_of;
  for (;;) {
    long sum = 0;
    for (int w = 0; w < W; w++) sum += bits[w];
    if (!((double)sum > budget * (double)W)) return;
    int victim = -1;
    for (int r = W - 1; r >= 0; r--) {                  /* lowest rank first */
      int w = order[r];
      if (pin && w == 0) continue;
      if (bits[w] > g->widths[0]) { victim = w; break; }
    }
    if (victim < 0) return;                              /* infeasible (checked by caller) */
    int k = 0;
    while (g->widths[k] != bits[victim]) k++;
    bits[victim] = (uint8_t)g->widths[k - 1];
  }
}

int wqo_assign_bits(const double *scores, const double *thr, int32_t L, const wqo_geom *g,
                    double budget, int32_t pin, int32_t vote,
                    uint8_t *bits, int32_t *rank, int32_t *perm, int32_t *seg_off) {
  int B = g->B, W = g->M / g->S, n = g->n_widths;
  int np = (pin && W > 0) ? 1 : 0;
  if (budget > 0.0 && (double)(16 * np + g->widths[0] * (W - np)) > budget * (double)W) return 3;
  int *order = (int *)malloc(sizeof(int) * (size_t)(W > 0 ? W : 1) * (size_t)B);
  int *rank_of = (int *)malloc(sizeof(int) * (size_t)(W > 0 ? W : 1) * (size_t)B);
  int *mord = (int *)malloc(sizeof(int) * (size_t)(W > 0 ? W : 1));
  int *mrank = (int *)malloc(sizeof(int) * (size_t)(W > 0 ? W : 1));
  double *mean = (double *)malloc(sizeof(double) * (size_t)(W > 0 ? W : 1));
  /* 1. ranks (layer independent: scores are computed once, Alg.1 line 8) */
  for (int b = 0; b < B; b++) {
    rank_windows(scores + (int64_t)b * W, W, order + (int64_t)b * W, rank_of + (int64_t)b * W);
    if (rank) for (int w = 0; w < W; w++) rank[(int64_t)b * W + w] = rank_of[(int64_t)b * W + w];
  }
  if (vote) {                                            /* batch-mean score for the budget rank */
    for (int w = 0; w < W; w++) {
      double s = 0.0;
      for (int b = 0; b < B; b++) s += scores[(int64_t)b * W + w];
      mean[w] = s / (double)B;
    }
    rank_windows(mean, W, mord, mrank);
  }
  for (int l = 0; l < L; l++) {
    const double *T = thr + (int64_t)l * (n - 1);
    uint8_t *bl = bits + (int64_t)l * B * W;
    /* 2. bands */
    for (int b = 0; b < B; b++)
      for (int w = 0; w < W; w++)
        bl[(int64_t)b * W + w] = (uint8_t)g->widths[band_level(scores[(int64_t)b * W + w], T, n)];
    /* 3. pin */
    if (np) for (int b = 0; b < B; b++) bl[(int64_t)b * W + 0] = 16;
    /* 4. vote: mode over the batch, ties -> higher width */
    if (vote) {
      for (int w = 0; w < W; w++) {
        int cnt[4] = {0, 0, 0, 0};
        for (int b = 0; b < B; b++) cnt[class_of(bl[(int64_t)b * W + w])]++;
        int best = 0;
        for (int k = 1; k < 4; k++) if (cnt[k] >= cnt[best]) best = k;
        for (int b = 0; b < B; b++) bl[(int64_t)b * W + w] = (uint8_t)CLASS_BITS[best];
      }
    }
    /* 5. budget (Q13) */
    if (budget > 0.0) {
      if (vote) {
        apply_budget(bl, W, mrank, mord, g, budget, np);
        for (int b = 1; b < B; b++) memcpy(bl + (int64_t)b * W, bl, (size_t)W);
      } else {
        for (int b = 0; b < B; b++)
          apply_budget(bl + (int64_t)b * W, W, rank_of + (int64_t)b * W, order + (int64_t)b * W,
                       g, budget, np);
      }
    }
    /* 6. stable partition into [2 | 4 | 8 | 16] (Alg.2, Q15) */
    for (int b = 0; b < B; b++) {
      int32_t *pl = perm + ((int64_t)l * B + b) * W;
      int32_t *so = seg_off + ((int64_t)l * B + b) * 5;
      int slot = 0;
      for (int k = 0; k < 4; k++) {
        so[k] = slot;
        for (int w = 0; w < W; w++)
          if (class_of(bl[(int64_t)b * W + w]) == k) pl[slot++] = w;
      }
      so[4] = slot;
    }
  }
  free(order); free(rank_of); free(mord); free(mrank); free(mean);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Byte accounting of the D-1 image                                           */
/* ------------------------------------------------------------------------ */
/* gran 0 (default, Q19): per-channel K / per-token V (s, mn) pairs, 4(d + S) bytes;
 * gran 1 (paper-literal P:508, reading Q37): one (s, mn) per (window, head, K|V) group,
 * a 16-byte block {mn_K, s_K, mn_V, s_V, 0, 0, 0, 0}. */
int64_t wqo_record_bytes_g(int32_t b, int32_t d, int32_t S, int32_t gran) {
  if (b == 16) return 2LL * S * d * 2;                   /* K and V fp16 */
  if (gran == 1) return 2LL * S * d * b / 8 + 16;
  return 2LL * S * d * b / 8 + 4LL * d + 4LL * S;        /* codes + (s, mn) fp16 pairs */
}
int64_t wqo_record_bytes(int32_t b, int32_t d, int32_t S) { return wqo_record_bytes_g(b, d, S, 0); }

int64_t wqo_packed_bytes(const wqo_geom *g, const int32_t n_per_class[4], int32_t code_only) {
  int64_t total = 0;
  for (int k = 0; k < 4; k++) {
    int64_t rec = code_only ? 2LL * g->S * g->d * CLASS_BITS[k] / 8
                            : wqo_record_bytes(CLASS_BITS[k], g->d, g->S);
    total += (int64_t)n_per_class[k] * rec;
  }
  return total;
}

/* KV bytes of a token mix (K and V, H heads, d channels), codes only */
int64_t wqo_kv_code_bytes(const int64_t tokens_per_class[4], int32_t d, int32_t H) {
  int64_t total = 0;
  for (int k = 0; k < 4; k++) total += tokens_per_class[k] * 2LL * H * d * CLASS_BITS[k] / 8;
  return total;
}

void wqo_layer_layout_g(const wqo_geom *g, const int32_t *seg_off_l, int64_t *offs, int32_t gran) {
  int64_t off = 0;
  for (int b = 0; b < g->B; b++) {
    const int32_t *so = seg_off_l + (int64_t)b * 5;
    int64_t img = 0;
    for (int k = 0; k < 4; k++) img += (int64_t)(so[k + 1] - so[k]) * wqo_record_bytes_g(CLASS_BITS[k], g->d, g->S, gran);
    for (int h = 0; h < g->H; h++) { offs[(int64_t)b * g->H + h] = off; off += img; }
  }
  offs[(int64_t)g->B * g->H] = off;
}
void wqo_layer_layout(const wqo_geom *g, const int32_t *seg_off_l, int64_t *offs) { wqo_layer_layout_g(g, seg_off_l, offs, 0); }

/* ------------------------------------------------------------------------ */
/* Eq.14-16 under Q17: fp32, one rounding per operation, RNE codes            */
/* ------------------------------------------------------------------------ */
static float f16f(uint16_t h) { return (float)wqo_f16_to_f64(h); }  /* exact */

/* Q17: mn / mx are the IEEE 754-2019 minimum / maximum operations (section 9.6),
 * which order -0 below +0: a group whose smallest value is a zero of either sign
 * stores mn = -0 (0x8000) iff a -0 is present, independent of element order. */
static float ieee_minimum(float a, float b) {
  if (a < b) return a;
  if (b < a) return b;
  return signbit(a) ? a : b;                             /* equal: -0 wins over +0 */
}
static float ieee_maximum(float a, float b) {
  if (a > b) return a;
  if (b > a) return b;
  return signbit(a) ? b : a;                             /* equal: +0 wins over -0 */
}

void wqo_quantize_group(const uint16_t *x, int32_t n, int64_t stride, int32_t bits,
                        uint16_t *s_out, uint16_t *mn_out, uint8_t *codes) {
  float mn = f16f(x[0]), mx = f16f(x[0]);
  for (int i = 1; i < n; i++) {
    float v = f16f(x[(int64_t)i * stride]);
    mn = ieee_minimum(mn, v);
    mx = ieee_maximum(mx, v);
  }
  float qmax = (float)((1 << bits) - 1);
  volatile float range = mx - mn;                        /* exact for fp16 operands */
  volatile float sq = range / qmax;                      /* IEEE division, RN */
  uint16_t s16 = wqo_f32_to_f16_ru(sq);                  /* round the scale UP */
  if (f16f(s16) < (float)ldexp(1.0, -24)) s16 = 0x0001;  /* floor 2^-24 (Q21) */
  volatile float s = f16f(s16);
  volatile float r = 1.0f / s;
  for (int i = 0; i < n; i++) {
    volatile float diff = f16f(x[(int64_t)i * stride]) - mn;
    volatile float prod = diff * r;
    float c = rintf(prod);                               /* ties to even (Q18) */
    if (c < 0.0f) c = 0.0f;
    if (c > qmax) c = qmax;
    codes[i] = (uint8_t)c;
  }
  *s_out = s16;
  *mn_out = wqo_f32_to_f16_rn(mn);                       /* exact: mn is an fp16 value */
}

/* ------------------------------------------------------------------------ */
/* D-1 fragment-order position of element (t, c) of a window tile            */
/*   K tile: t = token in window, c = channel; V tile: same (t, c) naming.     */
/* ------------------------------------------------------------------------ */
void wqo_code_pos(int32_t is_v, int32_t d, int32_t b, int32_t t, int32_t c,
                  int64_t *byte_off, int32_t *bit) {
  int tile = t / 16, tt = t % 16;
  int row, col;                                          /* row/col inside the 16 x (d) tile */
  int m, lane, r, e;
  if (!is_v) {                                           /* rows = tokens, cols = channels */
    row = tt; col = c;
    m = col / 16;
    int cc = col % 16;
    int hcol = cc / 8, q = (cc % 8) / 2;
    e = cc % 2;
    int g8 = row % 8, rhi = row / 8;
    r = rhi + 2 * hcol;
    lane = 4 * g8 + q;
  } else {                                               /* rows = channels, cols = tokens */
    row = c; col = tt;
    m = row / 16;
    int rr = row % 16;
    int g8 = rr % 8, rhi = rr / 8;
    int hcol = col / 8, q = (col % 8) / 2;
    e = col % 2;
    r = rhi + 2 * hcol;
    lane = 4 * g8 + q;
  }
  int P = 4 * m + r;
  int pairs_per_word = 16 / b;
  int word = P / pairs_per_word, j = P % pairs_per_word;
  int64_t tile_bytes = 2LL * d * b;                      /* 16 rows * d cols * b bits / 8 */
  int64_t chunk = (int64_t)d * b / 16;
  if (chunk >= 16)                                       /* 16-byte groups, lane-interleaved */
    *byte_off = tile * tile_bytes + (word / 4) * 512LL + lane * 16LL + 4LL * (word % 4);
  else
    *byte_off = tile * tile_bytes + lane * chunk + 4LL * word;
  *bit = 16 * e + b * j;
}

static void put_code(uint8_t *base, int64_t byte_off, int bit, int b, uint32_t code) {
  uint32_t w = (uint32_t)base[byte_off] | ((uint32_t)base[byte_off + 1] << 8) |
               ((uint32_t)base[byte_off + 2] << 16) | ((uint32_t)base[byte_off + 3] << 24);
  uint32_t mask = (b == 16 ? 0xFFFFu : ((1u << b) - 1u)) << bit;
  w = (w & ~mask) | ((code << bit) & mask);
  for (int i = 0; i < 4; i++) base[byte_off + i] = (uint8_t)(w >> (8 * i));
}

static uint32_t get_code(const uint8_t *base, int64_t byte_off, int bit, int b) {
  uint32_t w = (uint32_t)base[byte_off] | ((uint32_t)base[byte_off + 1] << 8) |
               ((uint32_t)base[byte_off + 2] << 16) | ((uint32_t)base[byte_off + 3] << 24);
  return (w >> bit) & (b == 16 ? 0xFFFFu : ((1u << b) - 1u));
}

static void put_u16(uint8_t *p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static uint16_t get_u16(const uint8_t *p) { return (uint16_t)(p[0] | (p[1] << 8)); }

/* byte offset of the (s, mn) of K channel c / V token t inside the params */
static int64_t kparam_off(int d, int c, int is_min) {
  int m = c / 16, q = (c % 8) / 2, h = (c % 16) / 8, e = c % 2;
  (void)d;
  return ((int64_t)4 * m + q) * 16 + 2 * (4 * h + (is_min ? 0 : 2) + e);
}
static int64_t vparam_off(int t, int is_min) {
  int i = t / 16, col = t % 16, q = (col % 8) / 2, h = col / 8, e = col % 2;
  return ((int64_t)4 * i + q) * 16 + 2 * ((is_min ? 4 : 0) + 2 * h + e);
}
int64_t wqo_param_pos(int32_t is_v, int32_t d, int32_t i, int32_t is_min) {
  return is_v ? vparam_off(i, is_min) : kparam_off(d, i, is_min);
}

static int64_t slot_offset(const wqo_geom *g, const int32_t *so, int slot, int *bits_out, int gran) {
  int64_t off = 0;
  for (int k = 0; k < 4; k++) {
    int n = so[k + 1] - so[k];
    if (slot < so[k + 1]) {
      *bits_out = CLASS_BITS[k];
      return off + (int64_t)(slot - so[k]) * wqo_record_bytes_g(CLASS_BITS[k], g->d, g->S, gran);
    }
    off += (int64_t)n * wqo_record_bytes_g(CLASS_BITS[k], g->d, g->S, gran);
  }
  *bits_out = 0;
  return -1;
}

/* Alg.2 prefill branch: window perm[slot] is quantized with its
 * segment's width and written at its slot (reorder + quant in one pass). */
void wqo_reorder_quantize_pack_g(const uint16_t *k, const uint16_t *v, const int64_t strides[3],
                                 int32_t vis_off, const wqo_geom *g,
                                 const int32_t *perm_l, int32_t perm_stride,
                                 const int32_t *seg_off_l, const int64_t *offs, uint8_t *packed, int32_t gran) {
  int d = g->d, S = g->S;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < g->B; b++) {
    for (int h = 0; h < g->H; h++) {
      const int32_t *so = seg_off_l + (int64_t)b * 5;
      uint16_t *grp = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)S * d);
      uint8_t *codes = (uint8_t *)malloc((size_t)S * d);
      for (int slot = 0; slot < so[4]; slot++) {
        int bits;
        int64_t roff = slot_offset(g, so, slot, &bits, gran);
        uint8_t *rec = packed + offs[(int64_t)b * g->H + h] + roff;
        int w = perm_l[(int64_t)b * perm_stride + slot];
        const uint16_t *K0 = k + b * strides[0] + h * strides[1] + (int64_t)(vis_off + w * S) * strides[2];
        const uint16_t *V0 = v + b * strides[0] + h * strides[1] + (int64_t)(vis_off + w * S) * strides[2];
        int64_t kbytes = (int64_t)S * d * bits / 8;          /* bytes of the K code/value tiles */
        memset(rec, 0, (size_t)wqo_record_bytes_g(bits, d, S, gran));
        if (bits == 16) {                                /* FP16 window: values in fragment order */
          for (int t = 0; t < S; t++)
            for (int c = 0; c < d; c++) {
              int64_t bo; int bit;
              wqo_code_pos(0, d, 16, t, c, &bo, &bit);
              put_code(rec, bo, bit, 16, K0[(int64_t)t * strides[2] + c]);
              wqo_code_pos(1, d, 16, t, c, &bo, &bit);
              put_code(rec + kbytes, bo, bit, 16, V0[(int64_t)t * strides[2] + c]);
            }
          continue;
        }
        if (gran == 1) {
          /* P:508 literal (Q37): ONE group per (window, head, K|V) -- all S*d values share
           * (s, mn); element (t, c) is group entry t*d + c */
          uint8_t *pb = rec + 2 * kbytes;
          uint16_t s16, mn16;
          for (int t = 0; t < S; t++)
            for (int c = 0; c < d; c++) grp[t * d + c] = K0[(int64_t)t * strides[2] + c];
          wqo_quantize_group(grp, S * d, 1, bits, &s16, &mn16, codes);
          put_u16(pb + 0, mn16);
          put_u16(pb + 2, s16);
          for (int t = 0; t < S; t++)
            for (int c = 0; c < d; c++) {
              int64_t bo; int bit;
              wqo_code_pos(0, d, bits, t, c, &bo, &bit);
              put_code(rec, bo, bit, bits, codes[t * d + c]);
            }
          for (int t = 0; t < S; t++)
            for (int c = 0; c < d; c++) grp[t * d + c] = V0[(int64_t)t * strides[2] + c];
          wqo_quantize_group(grp, S * d, 1, bits, &s16, &mn16, codes);
          put_u16(pb + 4, mn16);
          put_u16(pb + 6, s16);
          for (int t = 0; t < S; t++)
            for (int c = 0; c < d; c++) {
              int64_t bo; int bit;
              wqo_code_pos(1, d, bits, t, c, &bo, &bit);
              put_code(rec + kbytes, bo, bit, bits, codes[t * d + c]);
            }
          continue;
        }
        uint8_t *kp = rec + 2 * kbytes, *vp = kp + 4LL * d;
        for (int c = 0; c < d; c++) {                    /* K: one group per channel over S tokens */
          uint16_t s16, mn16;
          wqo_quantize_group(K0 + c, S, strides[2], bits, &s16, &mn16, codes);
          put_u16(kp + kparam_off(d, c, 0), s16);
          put_u16(kp + kparam_off(d, c, 1), mn16);
          for (int t = 0; t < S; t++) {
            int64_t bo; int bit;
            wqo_code_pos(0, d, bits, t, c, &bo, &bit);
            put_code(rec, bo, bit, bits, codes[t]);
          }
        }
        for (int t = 0; t < S; t++) {                    /* V: one group per token over d channels */
          uint16_t s16, mn16;
          for (int c = 0; c < d; c++) grp[c] = V0[(int64_t)t * strides[2] + c];
          wqo_quantize_group(grp, d, 1, bits, &s16, &mn16, codes);
          put_u16(vp + vparam_off(t, 0), s16);
          put_u16(vp + vparam_off(t, 1), mn16);
          for (int c = 0; c < d; c++) {
            int64_t bo; int bit;
            wqo_code_pos(1, d, bits, t, c, &bo, &bit);
            put_code(rec + kbytes, bo, bit, bits, codes[c]);
          }
        }
      }
      free(grp); free(codes);
    }
  }
}
void wqo_reorder_quantize_pack(const uint16_t *k, const uint16_t *v, const int64_t strides[3],
                               int32_t vis_off, const wqo_geom *g,
                               const int32_t *perm_l, int32_t perm_stride,
                               const int32_t *seg_off_l, const int64_t *offs, uint8_t *packed) {
  wqo_reorder_quantize_pack_g(k, v, strides, vis_off, g, perm_l, perm_stride, seg_off_l, offs, packed, 0);
}

/* x^ = mn + s * code (Eq.15 with z = -mn/s), exact in fp64; gran 1: the group's (s, mn) */
void wqo_dequant_record_g(const uint8_t *rec, int32_t bits, int32_t d, int32_t S, double *kh, double *vh,
                          int32_t gran) {
  int64_t kbytes = (int64_t)S * d * bits / 8;
  const uint8_t *kp = rec + 2 * kbytes, *vp = kp + 4LL * d;
  for (int t = 0; t < S; t++)
    for (int c = 0; c < d; c++) {
      int64_t bo; int bit;
      wqo_code_pos(0, d, bits, t, c, &bo, &bit);
      uint32_t kc = get_code(rec, bo, bit, bits);
      wqo_code_pos(1, d, bits, t, c, &bo, &bit);
      uint32_t vc = get_code(rec + kbytes, bo, bit, bits);
      if (bits == 16) {
        kh[(int64_t)t * d + c] = wqo_f16_to_f64((uint16_t)kc);
        vh[(int64_t)t * d + c] = wqo_f16_to_f64((uint16_t)vc);
      } else if (gran == 1) {
        double km = wqo_f16_to_f64(get_u16(kp + 0)), ks = wqo_f16_to_f64(get_u16(kp + 2));
        double vm = wqo_f16_to_f64(get_u16(kp + 4)), vs = wqo_f16_to_f64(get_u16(kp + 6));
        kh[(int64_t)t * d + c] = km + ks * (double)kc;
        vh[(int64_t)t * d + c] = vm + vs * (double)vc;
      } else {
        double ks = wqo_f16_to_f64(get_u16(kp + kparam_off(d, c, 0)));
        double km = wqo_f16_to_f64(get_u16(kp + kparam_off(d, c, 1)));
        double vs = wqo_f16_to_f64(get_u16(vp + vparam_off(t, 0)));
        double vm = wqo_f16_to_f64(get_u16(vp + vparam_off(t, 1)));
        kh[(int64_t)t * d + c] = km + ks * (double)kc;
        vh[(int64_t)t * d + c] = vm + vs * (double)vc;
      }
    }
}
void wqo_dequant_record(const uint8_t *rec, int32_t bits, int32_t d, int32_t S, double *kh, double *vh) {
  wqo_dequant_record_g(rec, bits, d, S, kh, vh, 0);
}

/* ------------------------------------------------------------------------ */
/* Eq.2-3 without mask: plain fp64 softmax attention of one query row */
/* over n tokens.  out[d]; part = (m, l, o[d]) if non-NULL.                    */
/* ------------------------------------------------------------------------ */
static void attend(const double *q, const double *K, const double *V, int64_t n, int d,
                   double scale, double *out, double *part) {
  double m = -INFINITY;
  double *logit = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int64_t t = 0; t < n; t++) {
    double s = 0.0;
    for (int c = 0; c < d; c++) s += q[c] * K[t * d + c];
    logit[t] = s * scale;
    if (logit[t] > m) m = logit[t];
  }
  double l = 0.0;
  for (int c = 0; c < d; c++) out[c] = 0.0;
  for (int64_t t = 0; t < n; t++) {
    double p = exp(logit[t] - m);
    l += p;
    for (int c = 0; c < d; c++) out[c] += p * V[t * d + c];
  }
  if (part) {
    part[0] = m; part[1] = l;
    for (int c = 0; c < d; c++) part[2 + c] = out[c];
  }
  for (int c = 0; c < d; c++) out[c] = (l > 0.0) ? out[c] / l : 0.0;
  free(logit);
}

/* Alg.2 decode branch evaluated as its definition: invert the
 * reorder (Eq.12-13), dequantize to fp64 and attend in original token order,
 * rest tokens (text/tail/generated, FP16) last. */
void wqo_decode_attention_g(const uint16_t *q, const uint8_t *packed, const int64_t *offs,
                            const int32_t *seg_off_l, const int32_t *perm_l, int32_t perm_stride,
                            const wqo_geom *g,
                            const uint16_t *k_rest, const uint16_t *v_rest,
                            const int64_t rest_strides[2], const int32_t *rest_len,
                            float sm_scale, double *out, double *partial, int32_t gran) {
  int d = g->d, S = g->S, grp = g->Hq / g->H;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < g->B; b++) {
    for (int h = 0; h < g->H; h++) {
      const int32_t *so = seg_off_l + (int64_t)b * 5;
      int nslot = so[4];
      int R = rest_len ? rest_len[b] : 0;
      int64_t n = (int64_t)nslot * S + R;
      double *K = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * d);
      double *V = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * d);
      /* original window order: visit windows by increasing window index */
      int64_t row = 0;
      int wmax = -1;
      for (int s = 0; s < nslot; s++) if (perm_l[(int64_t)b * perm_stride + s] > wmax) wmax = perm_l[(int64_t)b * perm_stride + s];
      for (int w = 0; w <= wmax; w++) {
        for (int s = 0; s < nslot; s++) {
          if (perm_l[(int64_t)b * perm_stride + s] != w) continue;
          int bits;
          int64_t roff = slot_offset(g, so, s, &bits, gran);
          wqo_dequant_record_g(packed + offs[(int64_t)b * g->H + h] + roff, bits, d, S,
                               K + row * d, V + row * d, gran);
          row += S;
        }
      }
      for (int t = 0; t < R; t++) {
        const uint16_t *kr = k_rest + b * rest_strides[0] + h * rest_strides[1] + (int64_t)t * d;
        const uint16_t *vr = v_rest + b * rest_strides[0] + h * rest_strides[1] + (int64_t)t * d;
        for (int c = 0; c < d; c++) {
          K[row * d + c] = wqo_f16_to_f64(kr[c]);
          V[row * d + c] = wqo_f16_to_f64(vr[c]);
        }
        row++;
      }
      double *qq = (double *)malloc(sizeof(double) * (size_t)d);
      for (int j = 0; j < grp; j++) {
        int hq = h * grp + j;
        for (int c = 0; c < d; c++) qq[c] = wqo_f16_to_f64(q[((int64_t)b * g->Hq + hq) * d + c]);
        attend(qq, K, V, row, d, (double)sm_scale, out + ((int64_t)b * g->Hq + hq) * d,
               partial ? partial + ((int64_t)b * g->Hq + hq) * (d + 2) : NULL);
      }
      free(qq); free(K); free(V);
    }
  }
}
void wqo_decode_attention(const uint16_t *q, const uint8_t *packed, const int64_t *offs,
                          const int32_t *seg_off_l, const int32_t *perm_l, int32_t perm_stride,
                          const wqo_geom *g,
                          const uint16_t *k_rest, const uint16_t *v_rest,
                          const int64_t rest_strides[2], const int32_t *rest_len,
                          float sm_scale, double *out, double *partial) {
  wqo_decode_attention_g(q, packed, offs, seg_off_l, perm_l, perm_stride, g, k_rest, v_rest, rest_strides, rest_len,
                         sm_scale, out, partial, 0);
}

void wqo_bruteforce_attention(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                              const int64_t strides[3], int32_t vis_off, const wqo_geom *g,
                              const int32_t *win_l, int32_t win_stride, const int32_t *n_win,
                              const uint16_t *k_rest, const uint16_t *v_rest,
                              const int64_t rest_strides[2], const int32_t *rest_len,
                              float sm_scale, double *out) {
  int d = g->d, S = g->S, grp = g->Hq / g->H;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < g->B; b++) {
    for (int h = 0; h < g->H; h++) {
      int nw = n_win[b];
      int R = rest_len ? rest_len[b] : 0;
      int64_t n = (int64_t)nw * S + R;
      double *K = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * d);
      double *V = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * d);
      int64_t row = 0;
      for (int i = 0; i < nw; i++) {
        int w = win_l[(int64_t)b * win_stride + i];
        for (int t = 0; t < S; t++) {
          const uint16_t *kr = k + b * strides[0] + h * strides[1] + (int64_t)(vis_off + w * S + t) * strides[2];
          const uint16_t *vr = v + b * strides[0] + h * strides[1] + (int64_t)(vis_off + w * S + t) * strides[2];
          for (int c = 0; c < d; c++) { K[row * d + c] = wqo_f16_to_f64(kr[c]); V[row * d + c] = wqo_f16_to_f64(vr[c]); }
          row++;
        }
      }
      for (int t = 0; t < R; t++) {
        const uint16_t *kr = k_rest + b * rest_strides[0] + h * rest_strides[1] + (int64_t)t * d;
        const uint16_t *vr = v_rest + b * rest_strides[0] + h * rest_strides[1] + (int64_t)t * d;
        for (int c = 0; c < d; c++) { K[row * d + c] = wqo_f16_to_f64(kr[c]); V[row * d + c] = wqo_f16_to_f64(vr[c]); }
        row++;
      }
      double *qq = (double *)malloc(sizeof(double) * (size_t)d);
      for (int j = 0; j < grp; j++) {
        int hq = h * grp + j;
        for (int c = 0; c < d; c++) qq[c] = wqo_f16_to_f64(q[((int64_t)b * g->Hq + hq) * d + c]);
        attend(qq, K, V, row, d, (double)sm_scale, out + ((int64_t)b * g->Hq + hq) * d, NULL);
      }
      free(qq); free(K); free(V);
    }
  }
}

/* o = sum_g e^{m_g - m*} o_g / sum_g e^{m_g - m*} l_g */
void wqo_merge(const double *parts, int32_t G, int32_t BHq, int32_t d, double *out) {
  for (int64_t i = 0; i < BHq; i++) {
    double mstar = -INFINITY;
    for (int gg = 0; gg < G; gg++) {
      const double *p = parts + ((int64_t)gg * BHq + i) * (d + 2);
      if (p[1] > 0.0 && p[0] > mstar) mstar = p[0];
    }
    double l = 0.0;
    for (int c = 0; c < d; c++) out[i * d + c] = 0.0;
    for (int gg = 0; gg < G; gg++) {
      const double *p = parts + ((int64_t)gg * BHq + i) * (d + 2);
      if (!(p[1] > 0.0)) continue;
      double f = exp(p[0] - mstar);
      l += f * p[1];
      for (int c = 0; c < d; c++) out[i * d + c] += f * p[2 + c];
    }
    for (int c = 0; c < d; c++) out[i * d + c] = (l > 0.0) ? out[i * d + c] / l : 0.0;
  }
}

/* ------------------------------------------------------------------------ */
/* T9 unfused baseline: dequantize the whole image to FP16.      */
/* ------------------------------------------------------------------------ */
void wqo_dequantize_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off_l,
                          const wqo_geom *g, const int64_t *offs16, uint8_t *img16) {
  int d = g->d, S = g->S;
  int64_t rec16 = wqo_record_bytes(16, d, S), kbytes16 = (int64_t)S * d * 2;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < g->B; b++) {
    for (int h = 0; h < g->H; h++) {
      const int32_t *so = seg_off_l + (int64_t)b * 5;
      double *kh = (double *)malloc(sizeof(double) * (size_t)S * d);
      double *vh = (double *)malloc(sizeof(double) * (size_t)S * d);
      for (int slot = 0; slot < so[4]; slot++) {
        int bits;
        int64_t roff = slot_offset(g, so, slot, &bits, 0);
        const uint8_t *rec = packed + offs[(int64_t)b * g->H + h] + roff;
        uint8_t *dst = img16 + offs16[(int64_t)b * g->H + h] + (int64_t)slot * rec16;
        wqo_dequant_record(rec, bits, d, S, kh, vh);       /* exact x^ = mn + s*code (fp16 values if 16) */
        for (int t = 0; t < S; t++)
          for (int c = 0; c < d; c++) {
            int64_t bo; int bit;
            wqo_code_pos(0, d, 16, t, c, &bo, &bit);
            put_code(dst, bo, bit, 16, wqo_f64_to_f16_rn(kh[(int64_t)t * d + c]));
            wqo_code_pos(1, d, 16, t, c, &bo, &bit);
            put_code(dst + kbytes16, bo, bit, 16, wqo_f64_to_f16_rn(vh[(int64_t)t * d + c]));
          }
      }
      free(kh); free(vh);
    }
  }
}

/* T11 similarity variant: Pearson correlation instead of cosine in Eq.8,
 * the mean over the S*N pairs of corr(t_j, v_k); a zero-variance row contributes 0.
 * Literal double sum, every pair's correlation from its own means and variances. */
static double pearson(const uint16_t *x, const uint16_t *y, int32_t D) {
  double mx = 0.0, my = 0.0;
  for (int c = 0; c < D; c++) { mx += wqo_f16_to_f64(x[c]); my += wqo_f16_to_f64(y[c]); }
  mx /= D; my /= D;
  double sxy = 0.0, sxx = 0.0, syy = 0.0;
  for (int c = 0; c < D; c++) {
    double a = wqo_f16_to_f64(x[c]) - mx, b = wqo_f16_to_f64(y[c]) - my;
    sxy += a * b; sxx += a * a; syy += b * b;
  }
  if (sxx == 0.0 || syy == 0.0) return 0.0;
  return sxy / (sqrt(sxx) * sqrt(syy));
}

void wqo_window_scores_pearson(const uint16_t *vis, int64_t vrs, int64_t vbs,
                               const uint16_t *txt, int64_t trs, int64_t tbs,
                               int32_t B, int32_t M, int32_t N, int32_t D, int32_t S, double *scores) {
  int W = M / S;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < B; b++)
    for (int w = 0; w < W; w++) {
      double sum = 0.0;
      for (int j = 0; j < N; j++)
        for (int k = 0; k < S; k++)
          sum += pearson(txt + b * tbs + (int64_t)j * trs, vis + b * vbs + (int64_t)(w * S + k) * vrs, D);
      scores[(int64_t)b * W + w] = sum / ((double)S * (double)N);
    }
}

/* Per-layer scorer (reading Q36): Eq.8 where the visual vector of
 * token t is the concatenation over the H kv heads of its post-RoPE key, K[b][h][vis_off+t][:],
 * and the text vector of text token j the concatenation over h of the mean of the GQA
 * group's queries, (1/g) sum_{g'} Q[b][h g + g'][j][:].  Literal double sum over the S*N
 * pairs, every vector built in fp64, zero-norm vectors contribute 0 (Q5). */
void wqo_window_scores_layer(const uint16_t *k, const int64_t ks[3], int32_t vis_off, const uint16_t *qt,
                             const int64_t qs[3], int32_t B, int32_t H, int32_t Hq, int32_t d, int32_t M,
                             int32_t N, int32_t S, double *scores) {
  int W = M / S, D = H * d, grp = Hq / H;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < B; b++)
    for (int w = 0; w < W; w++) {
      double *tv = (double *)malloc(sizeof(double) * (size_t)D);
      double *vv = (double *)malloc(sizeof(double) * (size_t)D);
      double sum = 0.0;
      for (int j = 0; j < N; j++) {
        for (int c = 0; c < D; c++) {
          int h = c / d, cc = c % d;
          double acc = 0.0;
          for (int gq = 0; gq < grp; gq++)
            acc += wqo_f16_to_f64(qt[b * qs[0] + (int64_t)(h * grp + gq) * qs[1] + (int64_t)j * qs[2] + cc]);
          tv[c] = acc / (double)grp;
        }
        double nt = 0.0;
        for (int c = 0; c < D; c++) nt += tv[c] * tv[c];
        nt = sqrt(nt);
        for (int kk = 0; kk < S; kk++) {
          int t = vis_off + w * S + kk;
          for (int c = 0; c < D; c++)
            vv[c] = wqo_f16_to_f64(k[b * ks[0] + (int64_t)(c / d) * ks[1] + (int64_t)t * ks[2] + c % d]);
          double nv = 0.0, dot = 0.0;
          for (int c = 0; c < D; c++) { nv += vv[c] * vv[c]; dot += tv[c] * vv[c]; }
          nv = sqrt(nv);
          if (nt == 0.0 || nv == 0.0) continue;
          sum += dot / (nt * nv);
        }
      }
      scores[(int64_t)b * W + w] = sum / ((double)S * (double)N);
      free(tv); free(vv);
    }
}
