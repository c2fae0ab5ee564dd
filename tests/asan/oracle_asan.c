/* oracle_asan.c -- drives every oracle function once on small inputs so the build
 * with -fsanitize=address,undefined (tests/test_oracle_sanitize.py) checks the oracle
 * for out-of-bounds accesses and undefined behaviour ("ASan/UBSan build of
 * the oracle"; the oracle once read past rest buffers, commit 0fe15d7).  Inputs are a
 * fixed LCG stream; the exit code is 0 when every call returned. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../oracle/wqo.h"

static uint32_t st = 12345u;
static double urand(void) { st = st * 1664525u + 1013904223u; return (st >> 8) / 16777216.0; }
static uint16_t h16(double x) { return wqo_f64_to_f16_rn(x); }

int main(void) {
  const int B = 2, H = 2, Hq = 4, d = 64, S = 16, W = 5, tail = 3, N = 3, D = 24, R = 7;
  const int M = W * S + tail;
  uint16_t *vis = malloc(sizeof(uint16_t) * B * M * D), *txt = malloc(sizeof(uint16_t) * B * N * D);
  for (int i = 0; i < B * M * D; i++) vis[i] = h16(urand() - 0.4);
  for (int i = 0; i < B * N * D; i++) txt[i] = h16(urand() - 0.3);
  for (int c = 0; c < D; c++) vis[2 * D + c] = 0;                   /* zero-norm row */
  double *scores = malloc(sizeof(double) * B * W);
  wqo_window_scores(vis, D, (int64_t)M * D, txt, D, (int64_t)N * D, B, M, N, D, S, scores);
  wqo_window_scores_pearson(vis, D, (int64_t)M * D, txt, D, (int64_t)N * D, B, M, N, D, S, scores);
  double s_l[2] = {0.5, 1.3}, thr[6];
  if (wqo_thresholds(s_l, 2, 2.0, 4, thr)) return 1;
  wqo_geom g = {B, H, Hq, d, M, S, 4, {2, 4, 8, 16}};
  uint8_t *bits = malloc(2 * B * W);
  int32_t *rank = malloc(sizeof(int32_t) * B * W), *perm = malloc(sizeof(int32_t) * 2 * B * W);
  int32_t *seg = malloc(sizeof(int32_t) * 2 * B * 5);
  if (wqo_assign_bits(scores, thr, 2, &g, 5.0, 1, 1, bits, rank, perm, seg)) return 2;
  if (wqo_assign_bits(scores, thr, 2, &g, 0.0, 1, 0, bits, rank, perm, seg)) return 3;
  int32_t cnt[4] = {1, 2, 3, 4};
  if (wqo_packed_bytes(&g, cnt, 0) <= 0 || wqo_packed_bytes(&g, cnt, 1) <= 0) return 4;
  int64_t tok[4] = {10, 20, 30, 40};
  if (wqo_kv_code_bytes(tok, d, H) <= 0) return 5;
  int64_t *offs = malloc(sizeof(int64_t) * (B * H + 1));
  wqo_layer_layout(&g, seg, offs);
  uint16_t *k = malloc(sizeof(uint16_t) * B * H * M * d), *v = malloc(sizeof(uint16_t) * B * H * M * d);
  for (int i = 0; i < B * H * M * d; i++) { k[i] = h16(4 * urand() - 2); v[i] = h16(2 * urand() - 1); }
  int64_t strides[3] = {(int64_t)H * M * d, (int64_t)M * d, d};
  uint8_t *packed = calloc((size_t)offs[B * H] + 16, 1);
  wqo_reorder_quantize_pack(k, v, strides, 0, &g, perm, W, seg, offs, packed);
  uint16_t q[B * Hq * d], kr[B * H * R * d], vr[B * H * R * d];
  for (int i = 0; i < B * Hq * d; i++) q[i] = h16(urand() - 0.5);
  for (int i = 0; i < B * H * R * d; i++) { kr[i] = h16(urand() - 0.5); vr[i] = h16(urand() - 0.5); }
  int64_t rs[2] = {(int64_t)H * R * d, (int64_t)R * d};
  int32_t rest_len[2] = {R, 0};
  double *out = malloc(sizeof(double) * B * Hq * d), *part = malloc(sizeof(double) * 2 * B * Hq * (d + 2));
  wqo_decode_attention(q, packed, offs, seg, perm, W, &g, kr, vr, rs, rest_len, 0.125f, out, part);
  memcpy(part + B * Hq * (d + 2), part, sizeof(double) * B * Hq * (d + 2));
  wqo_merge(part, 2, B * Hq, d, out);
  int32_t nwin[2] = {W, W};
  int32_t win[2 * W];
  for (int i = 0; i < 2 * W; i++) win[i] = i % W;
  wqo_bruteforce_attention(q, k, v, strides, 0, &g, win, W, nwin, kr, vr, rs, rest_len, 0.125f, out);
  int32_t seg16[2 * 5] = {0, 0, 0, 0, seg[4], 0, 0, 0, 0, seg[9]};
  int64_t *offs16 = malloc(sizeof(int64_t) * (B * H + 1));
  wqo_layer_layout(&g, seg16, offs16);
  uint8_t *img16 = calloc((size_t)offs16[B * H] + 16, 1);
  wqo_dequantize_image(packed, offs, seg, &g, offs16, img16);
  double kh[S * d], vh[S * d];
  wqo_dequant_record(packed, 2, d, S, kh, vh);
  uint16_t grp[5] = {0x0000, 0x8000, 0x3C00, 0x7BFF, 0xFBFF}, s16, mn16;
  uint8_t codes[5];
  wqo_quantize_group(grp, 5, 1, 8, &s16, &mn16, codes);
  for (uint32_t x = 0; x < 65536; x += 7) {
    (void)wqo_f16_to_f64((uint16_t)x);
    (void)wqo_f32_to_f16_ru((float)wqo_f16_to_f64((uint16_t)x) * 1.001f);
    (void)wqo_f32_to_f16_rn((float)wqo_f16_to_f64((uint16_t)x) * 0.999f);
  }
  for (int t = 0; t < S; t++)
    for (int c = 0; c < d; c++) {
      int64_t bo; int32_t bit;
      wqo_code_pos(t & 1, d, 4, t, c, &bo, &bit);
    }
  (void)wqo_param_pos(1, d, 3, 1);
  /* paper-literal group granularity (gran 1) and the per-layer scorer */
  int64_t *offs_g = malloc(sizeof(int64_t) * (B * H + 1));
  wqo_layer_layout_g(&g, seg, offs_g, 1);
  uint8_t *packed_g = calloc((size_t)offs_g[B * H] + 16, 1);
  wqo_reorder_quantize_pack_g(k, v, strides, 0, &g, perm, W, seg, offs_g, packed_g, 1);
  wqo_decode_attention_g(q, packed_g, offs_g, seg, perm, W, &g, kr, vr, rs, rest_len, 0.125f, out, part, 1);
  wqo_dequant_record_g(packed_g, 4, d, S, kh, vh, 1);
  if (wqo_record_bytes_g(2, d, S, 1) != (int64_t)S * d * 2 / 4 + 16) return 6;
  uint16_t qt[B * Hq * N * d];
  for (int i = 0; i < B * Hq * N * d; i++) qt[i] = h16(urand() - 0.5);
  int64_t qs[3] = {(int64_t)Hq * N * d, (int64_t)N * d, d};
  wqo_window_scores_layer(k, strides, 0, qt, qs, B, H, Hq, d, M, N, S, scores);
  free(offs_g); free(packed_g);
  printf("oracle_asan: ok %.6f\n", out[0]);
  free(vis); free(txt); free(scores); free(bits); free(rank); free(perm); free(seg); free(offs);
  free(k); free(v); free(packed); free(out); free(part); free(offs16); free(img16);
  return 0;
}
