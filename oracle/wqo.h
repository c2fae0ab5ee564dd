/*
 * wqo.h — CPU ORACLE for the WindowQuant hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_2605_02262_b200/csrc); it re-derives
 * everything from the paper (PAPER.md, "P:n" = line n) and the readings Qn
 * listed in DESIGN.md §3.  Arithmetic is fp64 except where the contract fixes
 * fp32 (the quantizer, Q17).  Compiled with -O2 -ffp-contract=off -fno-fast-math.
 *
 * Every function is the slow literal form of the definition it cites:
 *   wqo_window_score      Eq.8 double sum over (text token, window token) pairs
 *   wqo_thresholds        Eq.10-11
 *   wqo_assign_bits       P:313 bands, P:322 pin, P:395 vote, Q13 budget loop,
 *                         Alg.2 P:420-444 stable partition
 *   wqo_quantize_group    Eq.14-16 under reading Q17
 *   wqo_reorder_quantize_pack   Alg.2 prefill branch -> the D-1 byte image
 *   wqo_decode_attention  Eq.2-3 (no mask) over the dequantized cache
 *                         rebuilt in ORIGINAL token order (Eq.12-13)
 *   wqo_bruteforce_attention    Eq.2-3 on the unquantized fp16 K/V
 *   wqo_merge             LSE merge of shard partials
 *   wqo_dequantize_image  T9 unfused baseline: every record
 *                         rewritten as FP16, x^16 = RN_fp16(mn + s*code)
 */
#ifndef WQO_H_
#define WQO_H_
#include <stdint.h>

typedef struct {
  int32_t B, H, Hq, d, M, S, n_widths;
  int32_t widths[4];
} wqo_geom;

/* fp16 <-> float conversions written out bit by bit */
double   wqo_f16_to_f64(uint16_t h);
uint16_t wqo_f32_to_f16_ru(float x);   /* round toward +infinity */
uint16_t wqo_f32_to_f16_rn(float x);   /* round to nearest, ties to even */
uint16_t wqo_f64_to_f16_rn(double x);  /* round to nearest, ties to even */

/* Eq.10-11 */
double wqo_f1(double s, double alpha);
double wqo_f2(double s, double alpha);
int    wqo_thresholds(const double *s, int32_t L, double alpha, int32_t n, double *thr);

/* Eq.8 for one window / all windows (OpenMP over (b, w)) */
double wqo_window_score(const uint16_t *vis_b, int64_t vis_row_stride,
                        const uint16_t *txt_b, int64_t txt_row_stride,
                        int32_t N, int32_t D, int32_t S, int32_t w);
void   wqo_window_scores(const uint16_t *vis, int64_t vrs, int64_t vbs,
                         const uint16_t *txt, int64_t trs, int64_t tbs,
                         int32_t B, int32_t M, int32_t N, int32_t D, int32_t S,
                         double *scores);

/* T11 variant: Eq.8 with Pearson correlation per pair */
void   wqo_window_scores_pearson(const uint16_t *vis, int64_t vrs, int64_t vbs,
                                 const uint16_t *txt, int64_t trs, int64_t tbs,
                                 int32_t B, int32_t M, int32_t N, int32_t D, int32_t S,
                                 double *scores);

/* Per-layer scorer (reading Q36): Eq.8 on the layer's post-RoPE
 * visual keys (kv heads concatenated) against the text tokens' queries averaged over each
 * GQA group; k [B][H][T][d] and q_text [B][Hq][N][d] with element strides ks / qs (b, h, t). */
void wqo_window_scores_layer(const uint16_t *k, const int64_t ks[3], int32_t vis_off, const uint16_t *qt,
                             const int64_t qs[3], int32_t B, int32_t H, int32_t Hq, int32_t d, int32_t M,
                             int32_t N, int32_t S, double *scores);

/* Alg.1 band/pin/vote + budget + Alg.2 partition.  Returns 0, or 3 if the
 * budget is infeasible. */
int wqo_assign_bits(const double *scores, const double *thr, int32_t L,
                    const wqo_geom *g, double budget, int32_t pin, int32_t vote,
                    uint8_t *bits, int32_t *rank, int32_t *perm, int32_t *seg_off);

/* Byte accounting (D-1) */
int64_t wqo_record_bytes(int32_t b, int32_t d, int32_t S);
int64_t wqo_packed_bytes(const wqo_geom *g, const int32_t n_per_class[4], int32_t code_only);
int64_t wqo_kv_code_bytes(const int64_t tokens_per_class[4], int32_t d, int32_t H);
void    wqo_layer_layout(const wqo_geom *g, const int32_t *seg_off_l, int64_t *offs);

/* Eq.14-16 (Q17) for one group of n fp16 values x[i*stride] */
void wqo_quantize_group(const uint16_t *x, int32_t n, int64_t stride, int32_t bits,
                        uint16_t *s_out, uint16_t *mn_out, uint8_t *codes);

/* Position of element (row, col) of a code tile (D-1): byte offset of its
 * 32-bit word inside the tile and its bit offset inside that word. */
/* Byte offset of the fp16 scale (is_min = 0) or zero point (is_min = 1) of K
 * channel i (is_v = 0) or V token i (is_v = 1) inside a record's params (D-1). */
int64_t wqo_param_pos(int32_t is_v, int32_t d, int32_t i, int32_t is_min);
void wqo_code_pos(int32_t is_v, int32_t d, int32_t b, int32_t t, int32_t c,
                  int64_t *byte_off, int32_t *bit);

void wqo_reorder_quantize_pack(const uint16_t *k, const uint16_t *v, const int64_t strides[3],
                               int32_t vis_off, const wqo_geom *g,
                               const int32_t *perm_l, int32_t perm_stride,
                               const int32_t *seg_off_l, const int64_t *offs,
                               uint8_t *packed);

/* Dequantize the record of one (b, h, slot) into fp64 K^[S][d], V^[S][d]. */
void wqo_dequant_record(const uint8_t *rec, int32_t bits, int32_t d, int32_t S,
                        double *kh, double *vh);

/* out: fp64 [B][Hq][d]; partial: fp64 [B][Hq][d+2] or NULL. */
void wqo_decode_attention(const uint16_t *q, const uint8_t *packed, const int64_t *offs,
                          const int32_t *seg_off_l, const int32_t *perm_l, int32_t perm_stride,
                          const wqo_geom *g,
                          const uint16_t *k_rest, const uint16_t *v_rest,
                          const int64_t rest_strides[2], const int32_t *rest_len,
                          float sm_scale, double *out, double *partial);

/* Attention of each (b, hq) over the unquantized fp16 tokens of the windows
 * listed in win_l[b][0..n_win[b]) (window order as listed) plus the rest. */
void wqo_bruteforce_attention(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                              const int64_t strides[3], int32_t vis_off, const wqo_geom *g,
                              const int32_t *win_l, int32_t win_stride, const int32_t *n_win,
                              const uint16_t *k_rest, const uint16_t *v_rest,
                              const int64_t rest_strides[2], const int32_t *rest_len,
                              float sm_scale, double *out);

/* parts [G][B*Hq][d+2] (m, l, o) -> out [B*Hq][d] */
void wqo_merge(const double *parts, int32_t G, int32_t BHq, int32_t d, double *out);

/* T9's unfused baseline: every slot of the
 * packed layer image rewritten as an FP16 record (D-1 width-16 layout) in the same
 * slot order at img16 + offs16[b*H+h] + slot * 4*S*d; b-bit values become
 * RN_fp16(mn + s*code) (Eq.15, exact sum, one rounding), FP16 values are copied.
 * offs16 = wqo_layer_layout of seg16 = {0,0,0,0,nslots}. */
void wqo_dequantize_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off_l,
                          const wqo_geom *g, const int64_t *offs16, uint8_t *img16);

/* Paper-literal group quantization (reading Q37): gran = 1
 * stores ONE (s, mn) per (window, head, K|V) group -- all S*d values of the window's K
 * (resp. V) for that head -- in a 16-byte block {mn_K, s_K, mn_V, s_V, 0,0,0,0} after the
 * codes (code layout D-1 unchanged); gran = 0 is the default per-channel K / per-token V. */
int64_t wqo_record_bytes_g(int32_t b, int32_t d, int32_t S, int32_t gran);
void wqo_layer_layout_g(const wqo_geom *g, const int32_t *seg_off_l, int64_t *offs, int32_t gran);
void wqo_reorder_quantize_pack_g(const uint16_t *k, const uint16_t *v, const int64_t strides[3],
                                 int32_t vis_off, const wqo_geom *g,
                                 const int32_t *perm_l, int32_t perm_stride,
                                 const int32_t *seg_off_l, const int64_t *offs, uint8_t *packed, int32_t gran);
void wqo_dequant_record_g(const uint8_t *rec, int32_t bits, int32_t d, int32_t S, double *kh, double *vh,
                          int32_t gran);
void wqo_decode_attention_g(const uint16_t *q, const uint8_t *packed, const int64_t *offs,
                            const int32_t *seg_off_l, const int32_t *perm_l, int32_t perm_stride,
                            const wqo_geom *g,
                            const uint16_t *k_rest, const uint16_t *v_rest,
                            const int64_t rest_strides[2], const int32_t *rest_len,
                            float sm_scale, double *out, double *partial, int32_t gran);

#endif
