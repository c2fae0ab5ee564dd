/*
 * wq.h — C ABI of the B200-native WindowQuant hot path (libwq.so).
 *
 * WindowQuant = "Mixed-Precision KV Cache Quantization based on Window-Level
 * Similarity for VLMs Inference Optimization" (arxiv 2605.02262).  Citations:
 * "P:n" = /root/reference/PAPER.md line n (LaTeX source), Eq.k in LaTeX order,
 * Alg.1 = window-level quantization search, Alg.2 = window-level KV
 * cache computation.  Readings where the paper is silent are named
 * Qn and listed in DESIGN.md §3 (same numbering as SURVEY.md §8(c)).
 *
 * Conventions (all calls)
 *  - Pointers are DEVICE pointers unless the parameter name ends in `_host`.
 *  - The caller owns every buffer.  The library never allocates, frees or keeps
 *    a pointer after the call returns.  Scratch space comes from an explicit
 *    `workspace` argument whose size is returned by the matching *_workspace()
 *    query; workspaces must be zero-filled once after allocation: the kernels
 *    leave the synchronization counters in them zeroed again on exit (the rest
 *    is scratch whose contents do not matter between calls).
 *  - Device calls are asynchronous on `stream` (a cudaStream_t passed as void*,
 *    NULL = legacy default stream).  Argument validation is synchronous: a call
 *    that returns anything but WQ_OK launched nothing, and wq_last_error()
 *    names the offending argument and shape.
 *  - fp16 tensors are IEEE binary16 (the paper's KV precision).  KV,
 *    queries and outputs are fp16 ONLY: there is no bf16 entry point (Q40).
 *  - No floating-point atomics anywhere: every output is bit-reproducible run
 *    to run and GPU to GPU.
 *  - There is no CPU fallback: every device call launches CUDA kernels.
 */
#ifndef WQ_H_
#define WQ_H_
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WQ_OK = 0,
  WQ_EINVAL = 1,        /* bad scalar argument (NULL pointer, alpha <= 0, ...) */
  WQ_ESHAPE = 2,        /* inconsistent or unsupported shape               */
  WQ_EBUDGET = 3,       /* average-bit budget infeasible (data independent) */
  WQ_EUNSUPPORTED = 4,  /* valid but not built (e.g. head dim 96)           */
  WQ_ECUDA = 5          /* a CUDA launch/runtime error                      */
} wq_status;

/* Geometry of one layer call.  W = M / S full windows (Eq.7); the
 * M mod S tail tokens are not a window and stay FP16 (reading Q2). */
typedef struct {
  int32_t B;            /* requests in the batch                            */
  int32_t H;            /* KV heads                                        */
  int32_t Hq;           /* query heads, Hq % H == 0; group g = Hq / H (Q26) */
  int32_t d;            /* head dim, 64 or 128                             */
  int32_t M;            /* visual tokens per request (Eq.4-5)   */
  int32_t S;            /* window size: 16, 32, 64 or 128 (Eq.7)           */
  int32_t n_widths;     /* 1..4 */
  int32_t widths[4];    /* strictly ascending subset of {2,4,8,16} (Q9)    */
} wq_geom;

typedef struct {
  double  budget_avg_bits; /* <= 0: no budget.  Else sum_w bits_w <= budget*W (Q13) */
  int32_t pin_first;       /* 1 (default): window 0 is FP16 in every layer */
  int32_t batch_vote;      /* 0 (default); 1: per-(layer, window) mode over the batch (Q14) */
} wq_assign_opts;

/* The canonical width classes; segment k of a packed image holds width
 * WQ_CLASS_BITS[k].  (Alg.2 concatenates INT2, INT4, FP16 in that order,
 * P:451-453; 8-bit is the north-star extension, Q9.) */
#define WQ_N_CLASSES 4
/* class k <-> bits {2, 4, 8, 16}[k] */

/* ---------------------------------------------------------------------------
 * Packed KV image (contract D-1; the oracle writes the same bytes).
 *
 * One image per layer: for each (b, h) in b-major order a contiguous byte
 * range starting at offs[b*H + h] (offs from wq_layer_layout); inside it the
 * window records of request b in SLOT order.  Slots [seg_off[b][k],
 * seg_off[b][k+1]) form segment k and have width {2,4,8,16}[k]; segments are
 * precision-contiguous as in Alg.2.  All K/V heads of a
 * request share its slot list (bits are per (layer, request, window)).
 *
 * Window record, width b < 16 (head dim d, window S, T16 = 16-token tile):
 *   [K codes: S/16 tiles x 2*d*b bytes][V codes: S/16 tiles x 2*d*b bytes]
 *   [K params: 4*d bytes][V params: 4*S bytes]           size S*d*b/4 + 4d + 4S
 * Width 16: [K values: S/16 x 32*d bytes][V values: S/16 x 32*d bytes]  size 4*S*d
 *
 * Code tiles are in "fragment order": a tile holds 32 lane chunks of d*b/16
 * bytes, chunk L belongs to lane L (g = L/4, q = L%4).  Chunks of >= 16 bytes
 * are interleaved in 16-byte groups so a warp's 16-byte loads are contiguous:
 * word w of chunk L is at byte (w/4)*512 + L*16 + (w%4)*4 of the tile; an
 * 8-byte chunk (d = 64, b = 2) is at byte L*8.  A chunk holds d/4
 * element PAIRS P = 0..d/4-1 with m = P/4, r = P%4:
 *   K tile (tokens x channels): row = g + 8*(r&1) (token in tile),
 *                               col = 16*m + 2*q + 8*(r>>1) (channel)
 *   V tile (channels x tokens): row = 16*m + g + 8*(r&1) (channel),
 *                               col = 2*q + 8*(r>>1) (token in tile)
 *   element e in {0,1} of a pair is (row, col + e).
 * Pairs are packed into little-endian 32-bit words: word P / (16/b), slot
 * j = P % (16/b); element e occupies bits [16*e + b*j, 16*e + b*j + b).
 * (For b = 16 a pair is one word holding two raw fp16 values.)
 *
 * K params (per channel c over the window's S tokens, Q19): 4 x d/16 groups
 * of 16 bytes, group (q, m) at byte (4*m + q)*16 holds fp16
 *   { mn(c0), mn(c0+1), s(c0), s(c0+1), mn(c0+8), mn(c0+9), s(c0+8), s(c0+9) },
 *   c0 = 16*m + 2*q  (one 16-byte load is directly the mma A fragment of the
 *   zero-point term: rows g hold mn, rows g+8 are ignored).
 * V params (per token t over the d channels, Q19): S/16 x 4 groups of 16 B,
 * group (i, q) at byte (4*i + q)*16 holds fp16
 *   { s(t0), s(t0+1), s(t0+8), s(t0+9), mn(t0), mn(t0+1), mn(t0+8), mn(t0+9) },
 *   t0 = 16*i + 2*q (token index within the window).
 *
 * Quantizer (Eq.14-16, reading Q17/Q18/Q21).  Per group x[0..n),
 * q_max = 2^b - 1, all arithmetic IEEE fp32 with one rounding per operation:
 *   mn = minimum x, mx = maximum x   (IEEE 754-2019 minimum/maximum, sec. 9.6:
 *        -0 < +0, so mn is -0 iff the smallest value is a zero and a -0 is present)
 *   s  = max(RoundUp_fp16(fl(mx - mn) / q_max), 2^-24)        (stored fp16)
 *   r  = fl(1 / s)
 *   code_i = clamp(rint_half_even(fl(fl(x_i - mn) * r)), 0, q_max)
 *   dequantized x^_i = mn + s * code_i      (error <= s*(1/2 + 2^-14))
 * -------------------------------------------------------------------------*/

/* Thresholds of Eq.10-11 (Alg.1 lines 4-7).  HOST call.
 * s_host[L]: layer sensitivities s_l (Eq.9; calibration is out of scope), clamped
 * to [0, 1] (Q10).  alpha > 0 (default 2).  thr_host[L][n_widths-1]:
 *   n=3: (f1, f2); n=4: (f1, (f1+f2)/2, f2); n=2: ((f1+f2)/2); n=1: none (Q9).
 * Errors: WQ_EINVAL (NULL, L < 1, alpha <= 0 or not finite, n_widths outside 1..4). */
wq_status wq_thresholds(const double *s_host, int32_t L, double alpha,
                        int32_t n_widths, double *thr_host);

/* Window-prompt similarity, Eq.8 (Alg.1 lines 9-12):
 *   scores[b][w] = 1/(S*N) * sum_{j<N} sum_{k<S} cos(t_j, v_{w*S+k}),  w < W = M/S
 * computed through the exact identity sum_j sum_k t^_j . v^_k = (sum_k v^_k).(sum_j t^_j)
 * with x^ = x/||x|| (Q3), fp64 accumulation and output (Q6).  A zero-norm row
 * contributes 0 (Q5).
 * vis: fp16, element (b, m, c) at vis[b*vis_batch_stride + m*vis_row_stride + c];
 * txt: fp16, element (b, j, c) at txt[b*txt_batch_stride + j*txt_row_stride + c]
 * (strides in elements, rows 16-byte aligned).  scores: fp64 [B][W].
 * workspace: wq_window_scores_workspace(B, D) bytes.
 * Errors: WQ_ESHAPE if M < S, D % 8 != 0, N < 1, S not in {16,32,64,128}. */
wq_status wq_window_scores_workspace(int32_t B, int32_t D, size_t *bytes_host);
wq_status wq_window_scores(const void *vis, int64_t vis_row_stride, int64_t vis_batch_stride,
                           const void *txt, int64_t txt_row_stride, int64_t txt_batch_stride,
                           int32_t B, int32_t M, int32_t N, int32_t D, int32_t S,
                           double *scores, void *workspace, size_t workspace_bytes,
                           void *stream);

/* Similarity-function variants of the scorer (T11: the paper compares
 * cosine, Pearson correlation and Euclidean distance and keeps cosine).
 *   WQ_SIM_COSINE  Eq.8 as above.
 *   WQ_SIM_PEARSON scores[b][w] = 1/(S*N) sum_j sum_k pearson(t_j, v_k), pearson(x, y) =
 *                  cos(x - mean(x), y - mean(y)) (means over the D channels); the pooled
 *                  identity holds for the centred normalized rows; a constant row
 *                  (zero variance) contributes 0.
 * (Euclidean distance is not a similarity in [0, 1] the thresholds of Eq.10-11 could
 * band, and the paper does not say how it maps one; not provided.) */
enum { WQ_SIM_COSINE = 0, WQ_SIM_PEARSON = 1 };
wq_status wq_window_scores_ex(const void *vis, int64_t vis_row_stride, int64_t vis_batch_stride,
                              const void *txt, int64_t txt_row_stride, int64_t txt_batch_stride,
                              int32_t B, int32_t M, int32_t N, int32_t D, int32_t S, int32_t metric,
                              double *scores, void *workspace, size_t workspace_bytes, void *stream);

/* Per-layer scorer (the "visual keys x text queries" wording of
 * P:274 and Alg.1 line 11's E_w^i with a layer index; reading Q36).  For layer i:
 *   scores[b][w] = 1/(S*N) * sum_{j<N} sum_{k<S} cos(t_j, v_{w*S+k})
 * with v_t = concat over kv heads h of K[b][h][vis_off + t][:] (post-RoPE keys, D = H*d)
 * and t_j = concat over h of (1/g) sum_{g'<g} Q[b][h*g + g'][j][:] (the text tokens'
 * queries averaged over each GQA group, g = Hq/H), evaluated like wq_window_scores (pooled
 * identity, fp64).  k: fp16, element (b, h, t, c) at k[b*k_strides[0] + h*k_strides[1] +
 * t*k_strides[2] + c] (rows 16-byte aligned); q_text: fp16, element (b, hq, j, c) at
 * q_text[b*q_strides[0] + hq*q_strides[1] + j*q_strides[2] + c].  scores fp64 [B][W].
 * workspace: wq_window_scores_workspace(B, H*d) bytes.  k and q_text rows 16-byte aligned.
 * Errors: WQ_ESHAPE (S, M < S, H*d > 1024, Hq % H, Hq/H > 8), WQ_EUNSUPPORTED (d not 64/128),
 * WQ_EINVAL (alignment). */
wq_status wq_window_scores_layer(const void *k, const int64_t k_strides[3], int32_t vis_off, const void *q_text,
                                 const int64_t q_strides[3], int32_t B, int32_t H, int32_t Hq, int32_t d,
                                 int32_t M, int32_t N, int32_t S, double *scores, void *workspace,
                                 size_t workspace_bytes, void *stream);

/* Bit assignment + permutation (Alg.1 lines 8-16, P:313, P:316-322, P:395;
 * Alg.2 lines 2-13).  For each layer l and request b:
 *   1. rank[b][w]: position of window w in (-score, w) order (0 = most similar, Q7)
 *   2. band: level = [x >= T_1] + sum_{1<j<n-1} [x >= T_j] + [x > T_{n-1}]
 *      (n >= 3; n = 2: [x > T_1]; n = 1: 0), bits = widths[level] (Q8)
 *   3. pin: window 0 -> 16 if opts->pin_first (Q12)
 *   4. vote (opts->batch_vote): per (l, w) the mode over b, ties -> higher
 *      width (Q14); the budget then ranks by the batch-mean score
 *   5. budget: while sum_w bits > budget*W, demote the lowest-ranked
 *      non-pinned window with bits > widths[0] one width step (Q13)
 *   6. stable partition of windows by width class -> perm (slot -> window),
 *      seg_off[5] (class boundaries in slots).  The pinned window is in the
 *      16 class even if 16 is not in widths (Q9, Q15).
 * scores: fp64 [B][W] (device).  thr_host: [L][n_widths-1] HOST (copied into
 * kernel parameters; L <= 64).  Outputs (device): bits u8 [L][B][W],
 * rank i32 [B][W] (may be NULL), perm i32 [L][B][W], seg_off i32 [L][B][5].
 * Errors: WQ_EBUDGET if 16*pin + widths[0]*(W-pin) > budget*W (checked on host). */
wq_status wq_assign_bits(const double *scores, const double *thr_host, int32_t L,
                         const wq_geom *g, const wq_assign_opts *opts,
                         uint8_t *bits, int32_t *rank, int32_t *perm, int32_t *seg_off,
                         void *stream);

/* The whole search module in ONE launch (the fused scorer -> assign
 * kernel): wq_window_scores_ex (metric WQ_SIM_COSINE / WQ_SIM_PEARSON) over vis/txt of
 * request geometry g (B, M, S; widths), then wq_assign_bits for L layers -- the same
 * results (scores within rounding order: identical code, identical fixed reduction trees;
 * ranks, bits, perms, seg_off bit-identical).  A cooperative persistent grid: phases
 * (text pool, window scores, one rank sort per request, assignment) separated by grid-wide
 * barriers; the per-(layer, request) assignment reuses its request's single sort.
 * vis: fp16 rows as wq_window_scores (D channels, row/batch strides), txt likewise with N
 * rows.  Outputs as wq_window_scores / wq_assign_bits (rank may be NULL).
 * workspace: wq_search_workspace(B, D, W = M/S) bytes (pooled text + rank orders).
 * Errors: as wq_window_scores and wq_assign_bits; WQ_ECUDA if the cooperative grid cannot
 * be made co-resident. */
wq_status wq_search_workspace(int32_t B, int32_t D, int32_t W, size_t *bytes_host);
wq_status wq_search(const void *vis, int64_t vis_row_stride, int64_t vis_batch_stride, const void *txt,
                    int64_t txt_row_stride, int64_t txt_batch_stride, int32_t N, int32_t D, int32_t metric,
                    const double *thr_host, int32_t L, const wq_geom *g, const wq_assign_opts *opts,
                    double *scores, uint8_t *bits, int32_t *rank, int32_t *perm, int32_t *seg_off,
                    void *workspace, size_t workspace_bytes, void *stream);

/* Quantization granularity of the packed image (the *_ex entries; the plain entries
 * use WQ_GRAN_CHANNEL_TOKEN).
 *   WQ_GRAN_CHANNEL_TOKEN: per-channel K / per-token V parameters inside each window
 *     (reading Q19, KIVI-style; record = K codes, V codes, 2 fp16 per K channel,
 *     2 fp16 per V token: S*d*b/4 + 4d + 4S bytes).
 *   WQ_GRAN_GROUP: the paper-literal groups of P:508 ("grouped by sliding windows"):
 *     one (s, mn) per (window, KV head, K|V) over all S*d values (Eq.14-16 applied to
 *     the group; reading Q37); record = K codes, V codes, then a 16-byte block
 *     {mn_K, s_K, mn_V, s_V, 0, 0, 0, 0} (fp16): S*d*b/4 + 16 bytes.
 * FP16 windows (b = 16) are stored raw under both. */
enum { WQ_GRAN_CHANNEL_TOKEN = 0, WQ_GRAN_GROUP = 1 };

/* Bytes of one (b, h) image holding n_per_class_host[k] windows of class k
 * ({2,4,8,16}[k]) under contract D-1.  HOST.  With code_bytes_only = 1 the
 * params are not counted and the result is the paper's accounting.
 * Errors: WQ_EINVAL (NULL pointer, unknown granularity). */
wq_status wq_packed_bytes(const wq_geom *g, const int32_t n_per_class_host[4],
                          int32_t code_bytes_only, int64_t *bytes_host);
wq_status wq_packed_bytes_ex(const wq_geom *g, const int32_t n_per_class_host[4],
                             int32_t code_bytes_only, int32_t granularity, int64_t *bytes_host);

/* Byte offsets of the (b, h) images of one layer: offs[B*H + 1] (i64, device),
 * offs[0] = 0, offs[B*H] = total bytes.  seg_off_l: i32 [B][5] (device).
 * The _ex form takes the granularity (WQ_GRAN_*) of the image it lays out. */
wq_status wq_layer_layout(const wq_geom *g, const int32_t *seg_off_l, int64_t *offs,
                          void *stream);
wq_status wq_layer_layout_ex(const wq_geom *g, const int32_t *seg_off_l, int32_t granularity,
                             int64_t *offs, void *stream);

/* Reorder + group-quantize + pack one layer (Alg.2 lines 2-15, Eq.14-16,
 * group = window P:508; per-channel K / per-token V parameters, Q19).
 * k, v: fp16, element (b, h, t, c) at x[b*strides[0] + h*strides[1] + t*strides[2] + c]
 *   (strides in elements; rows 16-byte aligned).  Window w of request b covers
 *   tokens vis_off + w*S .. vis_off + w*S + S-1 (Q1).
 * perm_l: i32 [B][perm_stride]: slot -> window (any subset of windows; the
 *   multi-GPU sequence split passes each rank its own slot list).
 * seg_off_l: i32 [B][5]: slot boundaries of the width classes.
 * offs: i64 [B*H+1] from wq_layer_layout.  packed: u8 image (>= offs[B*H] bytes,
 *   16-byte aligned).  Output bytes are bit-exact with the oracle.
 * Errors: WQ_ESHAPE (d not 64/128, S not 16/32/64/128), WQ_EINVAL. */
wq_status wq_reorder_quantize_pack(const void *k, const void *v, const int64_t strides[3],
                                   int32_t vis_off, const wq_geom *g,
                                   const int32_t *perm_l, int32_t perm_stride,
                                   const int32_t *seg_off_l, const int64_t *offs,
                                   uint8_t *packed, void *stream);
/* The same with the granularity (WQ_GRAN_*); offs must come from wq_layer_layout_ex with
 * the same granularity.  WQ_GRAN_GROUP: Q17's quantizer over the S*d values of each
 * (window, head, K|V) group; bit-exact with the oracle's gran = 1.
 * Errors: as above, WQ_EINVAL for an unknown granularity. */
wq_status wq_reorder_quantize_pack_ex(const void *k, const void *v, const int64_t strides[3],
                                      int32_t vis_off, const wq_geom *g,
                                      const int32_t *perm_l, int32_t perm_stride,
                                      const int32_t *seg_off_l, const int64_t *offs,
                                      int32_t granularity, uint8_t *packed, void *stream);

/* Decode attention over the reordered mixed-precision cache (Alg.2 decode
 * branch P:450-458, Eq.2-3 without mask P:214, reorder invariance Eq.12-13
 * P:462-473, fused dequantization P:510).  For each request b and query head
 * hq (KV head h = hq / (Hq/H)):
 *   out[b][hq] = sum_t softmax_t(sm_scale * q[b][hq] . k^_t) v^_t
 * over every slot of the (b, h) image (dequantized on load) and the FP16 rest
 * tokens t < rest_len[b] (text, tail, generated: P:257, Q29).  Split-KV
 * online softmax with a log-sum-exp merge (Q24).
 * q: fp16 [B][Hq][d] contiguous.  packed/offs/seg_off_l: as produced above.
 * k_rest, v_rest: fp16, element (b, h, t, c) at x[b*rest_strides[0] + h*rest_strides[1] + t*d + c];
 *   rest_len: i32 [B] (device), each in [0, R_max] (values outside are clamped).
 * out: fp16 [B][Hq][d] (may be NULL).  partial: fp32 [B][Hq][d+2] =
 *   (m, l, o[d]) with m = max logit, l = sum exp(logit - m), o = sum exp(logit - m) v
 *   (unnormalized; m = -inf, l = 0 for an empty cache), may be NULL.
 * workspace: wq_decode_workspace(g) bytes, zero-filled once.
 * Numerical domain (fp16 intermediates of the fused dequantization): for every K
 *   channel group |q_c| * s_c < 2^15 (q*s is carried as an fp16 hi + lo pair; 2-bit
 *   windows carry (code - 2) * s_c in fp16 instead, which needs s_c <= 32752) and for
 *   every V token group s_t < 255 (p * s_t is an fp16 MMA operand with p <= 2^8, the
 *   lazy-rescale headroom).  Outside it results are undefined.  For b = 2 this allows V
 *   ranges up to 765 and, with |q| <= 8, K channel ranges up to 12288.  Inside it the
 *   output error is within 2e-3 of the row's largest |output| plus an absolute 2^-16: a
 *   V group with a subnormal scale (s = 2^-24..2^-14: zero, constant or subnormal-range
 *   values) makes p * s an fp16 subnormal, worth up to 2^(b-1) * 2^-24 absolute.
 * Errors: WQ_ESHAPE (unsupported d/S, Hq/H > 8), WQ_EINVAL (both outputs NULL). */
wq_status wq_decode_workspace(const wq_geom *g, size_t *bytes_host);

/* wq_decode_attention_ex flags. */
enum {
  /* WQ_DECODE_EARLY: the caller guarantees that packed, offs, seg_off_l and
   * rest_len are NOT written by the work enqueued immediately before this call
   * on `stream` (e.g. the previous layer's decode).  The kernel is then launched
   * as a programmatic dependent of that work (PDL): it plans the split-KV
   * partition and starts streaming the packed cache into shared memory while
   * that work drains, and touches q, k_rest/v_rest, out, partial and the
   * workspace only after it has completed.  Without the guarantee, pass 0. */
  WQ_DECODE_EARLY = 1,
  /* WQ_DECODE_GROUP: the image is WQ_GRAN_GROUP (one (s, mn) per window and tensor):
   * logit = s_K * sum_c code_c q_c + mn_K * sum_c q_c, V weight p * s_V.  Numerical
   * domain: s_V < 255 (as the per-token V scale above); no K-side bound beyond fp32.
   * Not accepted by the unreordered entry (WQ_EINVAL). */
  WQ_DECODE_GROUP = 2
};
/* wq_decode_attention with flags (WQ_DECODE_*); flags = 0 is wq_decode_attention. */
wq_status wq_decode_attention_ex(const void *q, const uint8_t *packed, const int64_t *offs,
                                 const int32_t *seg_off_l, const wq_geom *g,
                                 const void *k_rest, const void *v_rest,
                                 const int64_t rest_strides[2], const int32_t *rest_len,
                                 int32_t R_max, float sm_scale,
                                 void *out, float *partial,
                                 void *workspace, size_t workspace_bytes, uint32_t flags, void *stream);
wq_status wq_decode_attention(const void *q, const uint8_t *packed, const int64_t *offs,
                              const int32_t *seg_off_l, const wq_geom *g,
                              const void *k_rest, const void *v_rest,
                              const int64_t rest_strides[2], const int32_t *rest_len,
                              int32_t R_max, float sm_scale,
                              void *out, float *partial,
                              void *workspace, size_t workspace_bytes, void *stream);

/* LSE merge of G partials (the cross-GPU step of the sequence split, §8(e)):
 * parts fp32 [G][B][Hq][d+2] as written by wq_decode_attention;
 * out[b][hq] = sum_g e^{m_g - m*} o_g / sum_g e^{m_g - m*} l_g, m* = max_g m_g.
 * out: fp16 [B][Hq][d]. */
wq_status wq_merge_partials(const float *parts, int32_t G, const wq_geom *g,
                            void *out, void *stream);

/* Sequence split of the long-video case (§8(e)): rank r of G keeps, in every
 * width segment k of request b, the contiguous slot chunk
 *   [seg[k] + n_k*r/G, seg[k] + n_k*(r+1)/G),  n_k = seg[k+1] - seg[k]
 * (integer division), so every rank holds the same precision mix and bytes.
 * perm_l/seg_off_l: i32 [B][W] / [B][5] (device) as from wq_assign_bits;
 * outputs perm_r i32 [B][W] (first seg_off_r[b][4] entries valid), seg_off_r
 * i32 [B][5].  The rank's image is then built and decoded with perm_r/seg_off_r
 * and its (m, l, o) partials merged with wq_merge_partials after an all-gather. */
wq_status wq_shard_slots(const int32_t *perm_l, const int32_t *seg_off_l, int32_t B, int32_t W,
                         int32_t G, int32_t r, int32_t *perm_r, int32_t *seg_off_r, void *stream);

/* ---------------------------------------------------------------------------
 * Unfused baseline of the fusion ablation (T9).
 * The paper fuses dequantization into attention; the ablation first writes
 * the whole cache back to FP16 in HBM and then runs FP16 attention.
 *
 * wq_dequant_layout: seg16 i32 [B][5] = {0,0,0,0,nslots_b} (every slot of the FP16
 *   image is in class 16) and offs16 i64 [B*H+1], the FP16 image's (b, h) offsets.
 * wq_dequantize_image: img16 (>= offs16[B*H] bytes, 16-byte aligned) receives, for
 *   every slot of the packed layer image, an FP16 record (D-1 width-16 layout, same
 *   slot order, so perm_l still maps slots to windows) holding
 *     x^16 = RN_fp16(mn + s * code)    (the exact Eq.15 value, one rounding to fp16)
 *   for b-bit records and the stored values for FP16 records.  Bit-exact with the
 *   oracle.  Decode the result with wq_decode_attention(..., img16, offs16, seg16, ...).
 *   Input images of WQ_GRAN_CHANNEL_TOKEN granularity only (the default).
 * Errors: WQ_EINVAL (NULL, misaligned), WQ_ESHAPE (geometry). */
wq_status wq_dequant_layout(const wq_geom *g, const int32_t *seg_off_l, int32_t *seg16, int64_t *offs16,
                            void *stream);
wq_status wq_dequantize_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off_l,
                              const wq_geom *g, const int64_t *offs16, uint8_t *img16, void *stream);

/* ---------------------------------------------------------------------------
 * "Module III off" baseline of the reordering ablation (T8; P:401:
 * without reordering, windows of different precision stay interleaved in the cache).
 * SURVEY.md §8(f) row 1.
 *
 * wq_unreordered_layout: woff i64 [B][W+1], woff[b][w] = sum_{w'<w} record bytes of
 *   width bits_l[b][w'] (bits_l u8 [B][W] of the layer, from wq_assign_bits).
 * wq_unreorder_image: uimg (>= offs[B*H] bytes, 16-byte aligned) receives the records of
 *   the packed image in ORIGINAL window order: window w of (b, h) at
 *   offs[b*H+h] + woff[b][w] (records are quantized independently, so this is the byte
 *   image a quantizer without the reordering step writes).
 * wq_decode_attention_unreordered: wq_decode_attention over uimg; windows are visited
 *   in original order, each dispatched on its own width.  Same outputs/workspace/errors
 *   as wq_decode_attention (the result equals the reordered decode, Eq.12-13).
 *   WQ_GRAN_CHANNEL_TOKEN images only (record sizes of the default granularity). */
wq_status wq_unreordered_layout(const wq_geom *g, const uint8_t *bits_l, int64_t *woff, void *stream);
wq_status wq_unreorder_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off_l,
                             const int32_t *perm_l, const wq_geom *g, const int64_t *woff, uint8_t *uimg,
                             void *stream);
wq_status wq_decode_attention_unreordered(const void *q, const uint8_t *uimg, const int64_t *offs,
                                          const int32_t *seg_off_l, const int64_t *woff, const wq_geom *g,
                                          const void *k_rest, const void *v_rest,
                                          const int64_t rest_strides[2], const int32_t *rest_len,
                                          int32_t R_max, float sm_scale, void *out, float *partial,
                                          void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Fused cross-GPU log-sum-exp merge of the long-video sequence split (§8(e) P2,
 * SURVEY.md §8(f) row 2): the decode kernel itself exchanges the per-rank (m, l, o)
 * partials over NVLink peer memory and merges them, instead of partial -> NCCL
 * all-gather -> wq_merge_partials.
 *
 * wq_peer_buffer_bytes: bytes of the symmetric per-rank buffer
 *   [2 parities][G][B][Hq][d+2] fp32 + one u32 counter per (b, h) + one u32 error
 *   word (set when a wait for the peers timed out after 10 s: the output of that call
 *   and of every later call is invalid, later waits give up at once; its byte offset is
 *   wq_peer_error_offset), 256-B aligned.
 *   Every rank allocates one (cudaMalloc, zero-filled ONCE), maps the peers' buffers
 *   (CUDA IPC, peer access over NVLink) and keeps a device array of the G pointers.
 * wq_decode_attention_peer: wq_decode_attention of rank `rank` over its shard
 *   (wq_shard_slots) that writes the MERGED fp16 out [B][Hq][d] of all G ranks.
 *   `epoch` = 1, 2, 3, ... on every call (the same on all ranks); all G ranks must make
 *   the same sequence of calls (the kernel waits on its peers' contributions).
 *   peer_bufs: device array [G] of device pointers (entry `rank` = local_buf).
 *   No PDL flag, WQ_GRAN_CHANNEL_TOKEN images only.  With G = 1 it is the ordinary decode
 *   through the exchange path.
 *   Every CTA of the launch must be resident at once (one per SM, grid = SM count):
 *   the call returns WQ_ECUDA if the occupancy query says otherwise.  The tcgen05
 *   variant (WQ_DECODE_TC) is never used for this call.
 * Errors: as wq_decode_attention, WQ_EINVAL for rank/G/epoch/NULL. */
wq_status wq_peer_buffer_bytes(const wq_geom *g, int32_t G, size_t *bytes_host);
/* Byte offset of the error word inside the symmetric buffer (u32; 0 = no timeout). */
wq_status wq_peer_error_offset(const wq_geom *g, int32_t G, size_t *offset_host);
wq_status wq_decode_attention_peer(const void *q, const uint8_t *packed, const int64_t *offs,
                                   const int32_t *seg_off_l, const wq_geom *g, const void *k_rest,
                                   const void *v_rest, const int64_t rest_strides[2],
                                   const int32_t *rest_len, int32_t R_max, float sm_scale, void *out,
                                   void *workspace, size_t workspace_bytes, void *const *peer_bufs,
                                   void *local_buf, int32_t G, int32_t rank, uint32_t epoch, void *stream);

/* Test entry of the fused merge without a second GPU: G = 2 virtual ranks of
 * wq_decode_attention_peer run in ONE launch on this device, each on half of the SMs,
 * rank r with its own q/packed/offs/seg_off/rest/out/workspace (HOST arrays of G device
 * pointers: q_host[r] etc.) and the symmetric buffer local_bufs_host[r]; peer_bufs is the
 * device array of the G buffers.  Every exchange step of the cross-GPU protocol runs
 * (peer stores, system-scope release counters, acquire wait, LSE merge); since all CTAs
 * of the launch are co-resident, no kernel waits on another launch.
 * Errors: WQ_EUNSUPPORTED unless G = 2 and (d, S) in {(128, 32), (64, 16)}; as
 * wq_decode_attention_peer otherwise. */
wq_status wq_decode_attention_peer_emulated(int32_t G, const void *const *q_host, const uint8_t *const *packed_host,
                                            const int64_t *const *offs_host, const int32_t *const *seg_off_host,
                                            const wq_geom *g, const void *const *k_rest_host,
                                            const void *const *v_rest_host, const int64_t rest_strides[2],
                                            const int32_t *const *rest_len_host, int32_t R_max, float sm_scale,
                                            void *const *out_host, void *const *workspace_host,
                                            size_t workspace_bytes, void *const *peer_bufs,
                                            void *const *local_bufs_host, uint32_t epoch, void *stream);

/* Thread-local message of the last non-OK status of this thread. */
const char *wq_last_error(void);

/* Library build id (git describe at build time) and the SM arch it targets. */
const char *wq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WQ_H_ */
