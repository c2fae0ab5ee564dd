// abi.cu -- the extern "C" boundary of libwq.so (include/wq.h).  Host-side argument
// validation (synchronous, status + wq_last_error) and kernel launches; no compute
// happens here and there is no CPU fallback.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/wq.h"
#include "wq_device.cuh"
#include "wq_internal.h"

#ifndef WQ_BUILD_ID
#define WQ_BUILD_ID "dev"
#endif

namespace {
thread_local char g_err[512] = "";

wq_status fail(wq_status s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

wq_status cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return WQ_OK;
  return fail(WQ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

wq_status check_geom(const wq_geom *g, bool need_heads) {
  if (!g) return fail(WQ_EINVAL, "geom is NULL");
  if (g->B < 1 || g->M < 0) return fail(WQ_ESHAPE, "B=%d M=%d", g->B, g->M);
  if (!(g->S == 16 || g->S == 32 || g->S == 64 || g->S == 128))
    return fail(WQ_ESHAPE, "window S=%d not in {16,32,64,128}", g->S);
  if (g->n_widths < 1 || g->n_widths > 4) return fail(WQ_ESHAPE, "n_widths=%d not in 1..4", g->n_widths);
  for (int i = 0; i < g->n_widths; i++) {
    int w = g->widths[i];
    if (!(w == 2 || w == 4 || w == 8 || w == 16)) return fail(WQ_ESHAPE, "widths[%d]=%d not in {2,4,8,16}", i, w);
    if (i && w <= g->widths[i - 1]) return fail(WQ_ESHAPE, "widths must be strictly ascending");
  }
  if (need_heads) {
    if (!(g->d == 64 || g->d == 128)) return fail(WQ_EUNSUPPORTED, "head dim d=%d not in {64,128}", g->d);
    if (g->H < 1 || g->Hq < g->H || g->Hq % g->H) return fail(WQ_ESHAPE, "Hq=%d not a multiple of H=%d", g->Hq, g->H);
    if (g->Hq / g->H > 8) return fail(WQ_EUNSUPPORTED, "GQA group Hq/H=%d > 8", g->Hq / g->H);
    if ((int64_t)g->B * g->H > 1024) return fail(WQ_EUNSUPPORTED, "B*H=%lld > 1024", (long long)g->B * g->H);
  }
  return WQ_OK;
}

cudaStream_t S_(void *s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace

namespace wq {
int device_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}
}  // namespace wq

extern "C" {

const char *wq_last_error(void) { return g_err; }
const char *wq_version(void) { return WQ_BUILD_ID " sm_100a"; }

wq_status wq_thresholds(const double *s_host, int32_t L, double alpha, int32_t n_widths, double *thr_host) {
  if (!s_host || (n_widths > 1 && !thr_host)) return fail(WQ_EINVAL, "NULL pointer");
  if (L < 1) return fail(WQ_EINVAL, "L=%d < 1", L);
  if (!(alpha > 0.0) || !std::isfinite(alpha)) return fail(WQ_EINVAL, "alpha=%g must be > 0 (P:358)", alpha);
  if (n_widths < 1 || n_widths > 4) return fail(WQ_EINVAL, "n_widths=%d not in 1..4", n_widths);
  for (int l = 0; l < L; l++) {
    double s = s_host[l];
    s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);                       // Q10
    double f1 = (std::exp(alpha * s) - 1.0) / (std::exp(alpha) - 1.0);    // Eq.10
    double f2 = (std::exp(-alpha * s) - 1.0) / (std::exp(-alpha) - 1.0);  // Eq.11
    double *t = thr_host + (int64_t)l * (n_widths - 1);
    if (n_widths == 2) t[0] = (f1 + f2) / 2.0;
    if (n_widths == 3) { t[0] = f1; t[1] = f2; }
    if (n_widths == 4) { t[0] = f1; t[1] = (f1 + f2) / 2.0; t[2] = f2; }
  }
  return WQ_OK;
}

wq_status wq_window_scores_workspace(int32_t B, int32_t D, size_t *bytes_host) {
  if (!bytes_host) return fail(WQ_EINVAL, "bytes_host is NULL");
  if (B < 1 || D < 8) return fail(WQ_ESHAPE, "B=%d D=%d", B, D);
  *bytes_host = (size_t)B * D * sizeof(double);
  return WQ_OK;
}

wq_status wq_window_scores_ex(const void *vis, int64_t vrs, int64_t vbs, const void *txt, int64_t trs,
                              int64_t tbs, int32_t B, int32_t M, int32_t N, int32_t D, int32_t S,
                              int32_t metric, double *scores, void *workspace, size_t workspace_bytes,
                              void *stream) {
  if (!vis || !txt || !scores || !workspace) return fail(WQ_EINVAL, "NULL pointer");
  if (metric != WQ_SIM_COSINE && metric != WQ_SIM_PEARSON) return fail(WQ_EINVAL, "metric=%d", metric);
  if (!(S == 16 || S == 32 || S == 64 || S == 128)) return fail(WQ_ESHAPE, "S=%d not in {16,32,64,128}", S);
  if (B < 1 || N < 1 || M < S) return fail(WQ_ESHAPE, "B=%d N=%d M=%d (need M >= S=%d)", B, N, M, S);
  if (D % 8 || D < 8 || D > 4096) return fail(WQ_ESHAPE, "D=%d must be a multiple of 8 in [8, 4096]", D);
  if (vrs % 8 || vbs % 8 || trs % 8 || tbs % 8 || !aligned16(vis) || !aligned16(txt))
    return fail(WQ_EINVAL, "rows must be 16-byte aligned (strides multiple of 8 elements)");
  if (workspace_bytes < (size_t)B * D * sizeof(double)) return fail(WQ_EINVAL, "workspace too small");
  double *tbar = reinterpret_cast<double *>(workspace);
  wq_status s = cuda_status(wq::launch_text_pool((const __half *)txt, trs, tbs, B, N, D, tbar, metric, S_(stream)),
                            "text pool");
  if (s != WQ_OK) return s;
  return cuda_status(
      wq::launch_window_scores((const __half *)vis, vrs, vbs, B, M, N, D, S, tbar, scores, metric, S_(stream)),
      "window scores");
}

wq_status wq_window_scores(const void *vis, int64_t vrs, int64_t vbs, const void *txt, int64_t trs,
                           int64_t tbs, int32_t B, int32_t M, int32_t N, int32_t D, int32_t S,
                           double *scores, void *workspace, size_t workspace_bytes, void *stream) {
  return wq_window_scores_ex(vis, vrs, vbs, txt, trs, tbs, B, M, N, D, S, WQ_SIM_COSINE, scores, workspace,
                             workspace_bytes, stream);
}

wq_status wq_window_scores_layer(const void *k, const int64_t k_strides[3], int32_t vis_off, const void *q_text,
                                 const int64_t q_strides[3], int32_t B, int32_t H, int32_t Hq, int32_t d, int32_t M,
                                 int32_t N, int32_t S, double *scores, void *workspace, size_t workspace_bytes,
                                 void *stream) {
  if (!k || !k_strides || !q_text || !q_strides || !scores || !workspace) return fail(WQ_EINVAL, "NULL pointer");
  if (!(S == 16 || S == 32 || S == 64 || S == 128)) return fail(WQ_ESHAPE, "S=%d not in {16,32,64,128}", S);
  if (B < 1 || N < 1 || M < S || vis_off < 0) return fail(WQ_ESHAPE, "B=%d N=%d M=%d vis_off=%d (need M >= S=%d)",
                                                       B, N, M, vis_off, S);
  if (!(d == 64 || d == 128)) return fail(WQ_EUNSUPPORTED, "head dim d=%d not in {64,128}", d);
  if (H < 1 || Hq < H || Hq % H) return fail(WQ_ESHAPE, "Hq=%d not a multiple of H=%d", Hq, H);
  const int D = H * d;
  if (D > 1024) return fail(WQ_ESHAPE, "H*d=%d > 1024", D);
  if (Hq / H > 8) return fail(WQ_ESHAPE, "GQA group Hq/H=%d > 8", Hq / H);
  if (k_strides[0] % 8 || k_strides[1] % 8 || k_strides[2] % 8 || !aligned16(k))
    return fail(WQ_EINVAL, "K rows must be 16-byte aligned (strides multiple of 8 elements)");
  if (q_strides[0] % 8 || q_strides[1] % 8 || q_strides[2] % 8 || !aligned16(q_text))
    return fail(WQ_EINVAL, "q_text rows must be 16-byte aligned (strides multiple of 8 elements)");
  if (workspace_bytes < (size_t)B * D * sizeof(double)) return fail(WQ_EINVAL, "workspace too small");
  double *tbar = reinterpret_cast<double *>(workspace);
  wq_status s = cuda_status(wq::launch_text_pool_q((const __half *)q_text, q_strides[0], q_strides[1], q_strides[2],
                                                   B, N, H, Hq / H, d, tbar, S_(stream)),
                            "text query pool");
  if (s != WQ_OK) return s;
  const __half *vis = (const __half *)k + (int64_t)vis_off * k_strides[2];
  return cuda_status(wq::launch_window_scores(vis, k_strides[2], k_strides[0], B, M, N, D, S, tbar, scores, 0,
                                              S_(stream), d, k_strides[1]),
                     "layer window scores");
}

wq_status wq_assign_bits(const double *scores, const double *thr_host, int32_t L, const wq_geom *g,
                         const wq_assign_opts *opts, uint8_t *bits, int32_t *rank, int32_t *perm,
                         int32_t *seg_off, void *stream) {
  wq_status s = check_geom(g, false);
  if (s != WQ_OK) return s;
  if (!scores || !bits || !perm || !seg_off || (g->n_widths > 1 && !thr_host))
    return fail(WQ_EINVAL, "NULL pointer");
  if (L < 1 || L > wq::MAX_LAYERS) return fail(WQ_EINVAL, "L=%d not in 1..%d", L, wq::MAX_LAYERS);
  const int W = g->M / g->S;
  if (W < 1 || W > 4096) return fail(WQ_ESHAPE, "W=M/S=%d not in 1..4096", W);
  wq::AssignParams p{};
  p.L = L; p.B = g->B; p.W = W; p.n_widths = g->n_widths;
  for (int i = 0; i < 4; i++) p.widths[i] = i < g->n_widths ? g->widths[i] : 0;
  p.pin = opts ? opts->pin_first : 1;
  p.vote = opts ? opts->batch_vote : 0;
  p.budget = opts ? opts->budget_avg_bits : 0.0;
  const int np = p.pin ? 1 : 0;
  if (p.budget > 0.0 && (double)(16 * np + g->widths[0] * (W - np)) > p.budget * (double)W)
    return fail(WQ_EBUDGET, "budget %.4f bits infeasible: pinned window + %d x %d-bit windows exceed it",
                p.budget, W - np, g->widths[0]);
  for (int l = 0; l < L; l++)
    for (int j = 0; j < g->n_widths - 1; j++) p.thr[l * 3 + j] = thr_host[(int64_t)l * (g->n_widths - 1) + j];
  if (rank) {
    s = cuda_status(wq::launch_rank(scores, g->B, W, rank, S_(stream)), "rank");
    if (s != WQ_OK) return s;
  }
  return cuda_status(wq::launch_assign(scores, p, bits, perm, seg_off, S_(stream)), "assign");
}

wq_status wq_search_workspace(int32_t B, int32_t D, int32_t W, size_t *bytes_host) {
  if (!bytes_host) return fail(WQ_EINVAL, "bytes_host is NULL");
  if (B < 1 || D < 8 || W < 1) return fail(WQ_ESHAPE, "B=%d D=%d W=%d", B, D, W);
  const size_t tb = ((size_t)B * D * sizeof(double) + 255) / 256 * 256;
  *bytes_host = tb + (size_t)(B + 1) * W * sizeof(int32_t);
  return WQ_OK;
}

wq_status wq_search(const void *vis, int64_t vrs, int64_t vbs, const void *txt, int64_t trs, int64_t tbs, int32_t N,
                    int32_t D, int32_t metric, const double *thr_host, int32_t L, const wq_geom *g,
                    const wq_assign_opts *opts, double *scores, uint8_t *bits, int32_t *rank, int32_t *perm,
                    int32_t *seg_off, void *workspace, size_t workspace_bytes, void *stream) {
  wq_status s = check_geom(g, false);
  if (s != WQ_OK) return s;
  if (!vis || !txt || !scores || !bits || !perm || !seg_off || !workspace || (g->n_widths > 1 && !thr_host))
    return fail(WQ_EINVAL, "NULL pointer");
  if (metric != WQ_SIM_COSINE && metric != WQ_SIM_PEARSON) return fail(WQ_EINVAL, "metric=%d", metric);
  if (L < 1 || L > wq::MAX_LAYERS) return fail(WQ_EINVAL, "L=%d not in 1..%d", L, wq::MAX_LAYERS);
  const int W = g->M / g->S;
  if (W < 1 || W > 4096) return fail(WQ_ESHAPE, "W=M/S=%d not in 1..4096", W);
  if (N < 1) return fail(WQ_ESHAPE, "N=%d", N);
  if (D % 8 || D < 8 || D > 4096) return fail(WQ_ESHAPE, "D=%d must be a multiple of 8 in [8, 4096]", D);
  if (vrs % 8 || vbs % 8 || trs % 8 || tbs % 8 || !aligned16(vis) || !aligned16(txt))
    return fail(WQ_EINVAL, "rows must be 16-byte aligned (strides multiple of 8 elements)");
  size_t need = 0;
  wq_search_workspace(g->B, D, W, &need);
  if (workspace_bytes < need) return fail(WQ_EINVAL, "workspace too small (see wq_search_workspace)");
  wq::AssignParams p{};
  p.L = L; p.B = g->B; p.W = W; p.n_widths = g->n_widths;
  for (int i = 0; i < 4; i++) p.widths[i] = i < g->n_widths ? g->widths[i] : 0;
  p.pin = opts ? opts->pin_first : 1;
  p.vote = opts ? opts->batch_vote : 0;
  p.budget = opts ? opts->budget_avg_bits : 0.0;
  const int np = p.pin ? 1 : 0;
  if (p.budget > 0.0 && (double)(16 * np + g->widths[0] * (W - np)) > p.budget * (double)W)
    return fail(WQ_EBUDGET, "budget %.4f bits infeasible: pinned window + %d x %d-bit windows exceed it",
                p.budget, W - np, g->widths[0]);
  for (int l = 0; l < L; l++)
    for (int j = 0; j < g->n_widths - 1; j++) p.thr[l * 3 + j] = thr_host[(int64_t)l * (g->n_widths - 1) + j];
  double *tbar = reinterpret_cast<double *>(workspace);
  int32_t *order = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(workspace) +
                                               ((size_t)g->B * D * sizeof(double) + 255) / 256 * 256);
  return cuda_status(wq::launch_search((const __half *)vis, vrs, vbs, (const __half *)txt, trs, tbs, g->B, g->M, N, D,
                                       g->S, metric, p, tbar, scores, order, bits, rank, perm, seg_off, S_(stream)),
                     "search");
}

static bool gran_ok(int32_t gran) { return gran == WQ_GRAN_CHANNEL_TOKEN || gran == WQ_GRAN_GROUP; }

wq_status wq_packed_bytes_ex(const wq_geom *g, const int32_t n_per_class_host[4], int32_t code_bytes_only,
                             int32_t granularity, int64_t *bytes_host) {
  if (!g || !n_per_class_host || !bytes_host) return fail(WQ_EINVAL, "NULL pointer");
  if (!gran_ok(granularity)) return fail(WQ_EINVAL, "granularity=%d", granularity);
  static const int cb[4] = {2, 4, 8, 16};
  int64_t t = 0;
  for (int k = 0; k < 4; k++) {
    int64_t rec = code_bytes_only ? (int64_t)g->S * g->d * cb[k] / 4
                                  : wq::record_bytes(cb[k], g->d, g->S, granularity);
    t += (int64_t)n_per_class_host[k] * rec;
  }
  *bytes_host = t;
  return WQ_OK;
}

wq_status wq_packed_bytes(const wq_geom *g, const int32_t n_per_class_host[4], int32_t code_bytes_only,
                          int64_t *bytes_host) {
  return wq_packed_bytes_ex(g, n_per_class_host, code_bytes_only, WQ_GRAN_CHANNEL_TOKEN, bytes_host);
}

wq_status wq_layer_layout_ex(const wq_geom *g, const int32_t *seg_off_l, int32_t granularity, int64_t *offs,
                             void *stream) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!seg_off_l || !offs) return fail(WQ_EINVAL, "NULL pointer");
  if (!gran_ok(granularity)) return fail(WQ_EINVAL, "granularity=%d", granularity);
  if (g->B > 4096) return fail(WQ_ESHAPE, "B=%d > 4096", g->B);
  return cuda_status(wq::launch_layer_layout(seg_off_l, g->B, g->H, g->d, g->S, granularity, offs, S_(stream)),
                     "layout");
}

wq_status wq_layer_layout(const wq_geom *g, const int32_t *seg_off_l, int64_t *offs, void *stream) {
  return wq_layer_layout_ex(g, seg_off_l, WQ_GRAN_CHANNEL_TOKEN, offs, stream);
}

wq_status wq_reorder_quantize_pack(const void *k, const void *v, const int64_t strides[3], int32_t vis_off,
                                   const wq_geom *g, const int32_t *perm_l, int32_t perm_stride,
                                   const int32_t *seg_off_l, const int64_t *offs, uint8_t *packed,
                                   void *stream) {
  return wq_reorder_quantize_pack_ex(k, v, strides, vis_off, g, perm_l, perm_stride, seg_off_l, offs,
                                     WQ_GRAN_CHANNEL_TOKEN, packed, stream);
}

wq_status wq_reorder_quantize_pack_ex(const void *k, const void *v, const int64_t strides[3], int32_t vis_off,
                                      const wq_geom *g, const int32_t *perm_l, int32_t perm_stride,
                                      const int32_t *seg_off_l, const int64_t *offs, int32_t granularity,
                                      uint8_t *packed, void *stream) {
  if (!gran_ok(granularity)) return fail(WQ_EINVAL, "granularity=%d", granularity);
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!k || !v || !strides || !perm_l || !seg_off_l || !offs || !packed) return fail(WQ_EINVAL, "NULL pointer");
  if (perm_stride < 1) return fail(WQ_EINVAL, "perm_stride=%d", perm_stride);
  if (strides[0] % 8 || strides[1] % 8 || strides[2] % 8 || !aligned16(k) || !aligned16(v) || !aligned16(packed))
    return fail(WQ_EINVAL, "K/V rows and the packed image must be 16-byte aligned");
  if (strides[2] < g->d) return fail(WQ_ESHAPE, "token stride %lld < d=%d", (long long)strides[2], g->d);
  if (vis_off < 0) return fail(WQ_EINVAL, "vis_off=%d", vis_off);
  return cuda_status(wq::launch_quant((const __half *)k, (const __half *)v, strides, vis_off, g->B, g->H, g->d,
                                      g->S, g->M, perm_l, perm_stride, seg_off_l, offs, packed, granularity,
                                      S_(stream)),
                     "quantize");
}

wq_status wq_decode_workspace(const wq_geom *g, size_t *bytes_host) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!bytes_host) return fail(WQ_EINVAL, "bytes_host is NULL");
  *bytes_host = wq::decode_workspace_bytes(g->B, g->H, g->Hq, g->d, wq::device_sm_count());
  return WQ_OK;
}

wq_status wq_decode_attention(const void *q, const uint8_t *packed, const int64_t *offs, const int32_t *seg_off_l,
                              const wq_geom *g, const void *k_rest, const void *v_rest,
                              const int64_t rest_strides[2], const int32_t *rest_len, int32_t R_max,
                              float sm_scale, void *out, float *partial, void *workspace,
                              size_t workspace_bytes, void *stream) {
  return wq_decode_attention_ex(q, packed, offs, seg_off_l, g, k_rest, v_rest, rest_strides, rest_len, R_max,
                                sm_scale, out, partial, workspace, workspace_bytes, 0u, stream);
}

struct PeerCfg {
  uint8_t *const *bufs;      // device array [G]
  void *local;               // this rank's buffer (host-known device pointer)
  int32_t G, rank;
  uint32_t epoch;
};

// validated kernel arguments of one decode call (no launch)
static wq_status decode_args(const void *q, const uint8_t *packed, const int64_t *offs,
                             const int32_t *seg_off_l, const wq_geom *g, const void *k_rest,
                             const void *v_rest, const int64_t rest_strides[2], const int32_t *rest_len,
                             int32_t R_max, float sm_scale, void *out, float *partial, void *workspace,
                             size_t workspace_bytes, uint32_t flags, const int64_t *woff, const PeerCfg *pc,
                             wq::DecodeArgs &a) {
  if (flags & ~(uint32_t)(WQ_DECODE_EARLY | WQ_DECODE_GROUP)) return fail(WQ_EINVAL, "unknown decode flags 0x%x", flags);
  if ((flags & WQ_DECODE_GROUP) && woff) return fail(WQ_EINVAL, "WQ_DECODE_GROUP needs a reordered image");
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!q || !packed || !offs || !seg_off_l || !workspace) return fail(WQ_EINVAL, "NULL pointer");
  if (!out && !partial) return fail(WQ_EINVAL, "both out and partial are NULL");
  if (R_max < 0) return fail(WQ_EINVAL, "R_max=%d", R_max);
  if (R_max > 0 && (!k_rest || !v_rest || !rest_len || !rest_strides))
    return fail(WQ_EINVAL, "rest buffers NULL with R_max=%d", R_max);
  if (R_max > 0 && (rest_strides[0] % 8 || rest_strides[1] % 8 || !aligned16(k_rest) || !aligned16(v_rest)))
    return fail(WQ_EINVAL, "rest rows must be 16-byte aligned");
  if (!aligned16(packed) || !aligned16(q)) return fail(WQ_EINVAL, "packed / q must be 16-byte aligned");
  if (!(sm_scale > 0.f) || !std::isfinite(sm_scale)) return fail(WQ_EINVAL, "sm_scale=%g", (double)sm_scale);
  const int sms = wq::device_sm_count();
  if (workspace_bytes < wq::decode_workspace_bytes(g->B, g->H, g->Hq, g->d, sms))
    return fail(WQ_EINVAL, "workspace too small (see wq_decode_workspace)");
  a = wq::DecodeArgs{};
  a.q = (const __half *)q; a.packed = packed; a.offs = offs; a.seg_off = seg_off_l;
  a.k_rest = (const __half *)k_rest; a.v_rest = (const __half *)v_rest;
  a.rs_b = R_max > 0 ? rest_strides[0] : 0; a.rs_h = R_max > 0 ? rest_strides[1] : 0;
  a.rest_len = R_max > 0 ? rest_len : nullptr; a.R_max = R_max;
  a.B = g->B; a.H = g->H; a.Hq = g->Hq; a.grp = g->Hq / g->H; a.d = g->d; a.S = g->S;
  a.scale_log2 = sm_scale * 1.4426950408889634f;
  a.out = (__half *)out; a.partial = partial;
  a.flags = flags;
  a.woff = woff;
  if (pc) {
    // the rank-local unit results go to this rank's slot of the current parity; the
    // kernel exchanges them with the peers and writes the merged result to out
    const int64_t slotf = (int64_t)g->B * g->Hq * (g->d + 2);
    a.peer_bufs = pc->bufs; a.peer_G = pc->G; a.peer_rank = pc->rank; a.peer_epoch = pc->epoch;
    a.peer_out = (__half *)out;
    a.out = nullptr;
    a.partial = reinterpret_cast<float *>(pc->local) + ((int64_t)(pc->epoch & 1u) * pc->G + pc->rank) * slotf;
  }
  const wq::DecodeWsLayout wl = wq::decode_ws_layout(g->B, g->H, g->d, sms);
  a.ws_part = reinterpret_cast<float *>(workspace);
  a.ws_cnt = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(workspace) + wl.part);
  // profiling builds only (WQ_DEC_PROFILE / WQ_TC_PROFILE): per-CTA timestamps when
  // WQ_DECODE_DEBUG has bit 3 set; the environment is read once per process
  static const int dbg = getenv("WQ_DECODE_DEBUG") ? atoi(getenv("WQ_DECODE_DEBUG")) : 0;
  a.ws_ts = (dbg & 8) ? reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(workspace) + wl.part + wl.cnt)
                      : nullptr;
  return WQ_OK;
}

static wq_status decode_impl(const void *q, const uint8_t *packed, const int64_t *offs,
                             const int32_t *seg_off_l, const wq_geom *g, const void *k_rest,
                             const void *v_rest, const int64_t rest_strides[2], const int32_t *rest_len,
                             int32_t R_max, float sm_scale, void *out, float *partial, void *workspace,
                             size_t workspace_bytes, uint32_t flags, const int64_t *woff, void *stream,
                             const PeerCfg *pc = nullptr) {
  wq::DecodeArgs a;
  wq_status s = decode_args(q, packed, offs, seg_off_l, g, k_rest, v_rest, rest_strides, rest_len, R_max, sm_scale,
                            out, partial, workspace, workspace_bytes, flags, woff, pc, a);
  if (s != WQ_OK) return s;
  return cuda_status(wq::launch_decode(a, wq::device_sm_count(), S_(stream)), "decode");
}

wq_status wq_decode_attention_ex(const void *q, const uint8_t *packed, const int64_t *offs,
                                 const int32_t *seg_off_l, const wq_geom *g, const void *k_rest,
                                 const void *v_rest, const int64_t rest_strides[2], const int32_t *rest_len,
                                 int32_t R_max, float sm_scale, void *out, float *partial, void *workspace,
                                 size_t workspace_bytes, uint32_t flags, void *stream) {
  return decode_impl(q, packed, offs, seg_off_l, g, k_rest, v_rest, rest_strides, rest_len, R_max, sm_scale, out,
                     partial, workspace, workspace_bytes, flags, nullptr, stream);
}

wq_status wq_peer_buffer_bytes(const wq_geom *g, int32_t G, size_t *bytes_host) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!bytes_host) return fail(WQ_EINVAL, "NULL pointer");
  if (G < 1 || G > 64) return fail(WQ_EINVAL, "G=%d", G);
  *bytes_host = wq::peer_buffer_bytes(g->B, g->H, g->Hq, g->d, G);
  return WQ_OK;
}

wq_status wq_peer_error_offset(const wq_geom *g, int32_t G, size_t *offset_host) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!offset_host) return fail(WQ_EINVAL, "NULL pointer");
  if (G < 1 || G > 64) return fail(WQ_EINVAL, "G=%d", G);
  *offset_host = 2ull * G * g->B * g->Hq * (g->d + 2) * sizeof(float) + (size_t)g->B * g->H * sizeof(uint32_t);
  return WQ_OK;
}

wq_status wq_decode_attention_peer(const void *q, const uint8_t *packed, const int64_t *offs,
                                   const int32_t *seg_off_l, const wq_geom *g, const void *k_rest,
                                   const void *v_rest, const int64_t rest_strides[2], const int32_t *rest_len,
                                   int32_t R_max, float sm_scale, void *out, void *workspace,
                                   size_t workspace_bytes, void *const *peer_bufs, void *local_buf, int32_t G,
                                   int32_t rank, uint32_t epoch, void *stream) {
  if (!out || !peer_bufs || !local_buf) return fail(WQ_EINVAL, "NULL pointer (out / peer buffers)");
  if (G < 1 || G > 64 || rank < 0 || rank >= G) return fail(WQ_EINVAL, "rank %d of %d", rank, G);
  if (epoch == 0) return fail(WQ_EINVAL, "epoch must start at 1");
  PeerCfg pc{reinterpret_cast<uint8_t *const *>(peer_bufs), local_buf, G, rank, epoch};
  return decode_impl(q, packed, offs, seg_off_l, g, k_rest, v_rest, rest_strides, rest_len, R_max, sm_scale, out,
                     nullptr, workspace, workspace_bytes, 0u, nullptr, stream, &pc);
}

wq_status wq_decode_attention_peer_emulated(int32_t G, const void *const *q_host, const uint8_t *const *packed_host,
                                            const int64_t *const *offs_host, const int32_t *const *seg_off_host,
                                            const wq_geom *g, const void *const *k_rest_host,
                                            const void *const *v_rest_host, const int64_t rest_strides[2],
                                            const int32_t *const *rest_len_host, int32_t R_max, float sm_scale,
                                            void *const *out_host, void *const *workspace_host,
                                            size_t workspace_bytes, void *const *peer_bufs,
                                            void *const *local_bufs_host, uint32_t epoch, void *stream) {
  if (G != 2) return fail(WQ_EUNSUPPORTED, "emulation runs G = 2 virtual ranks (G=%d)", G);
  if (!q_host || !packed_host || !offs_host || !seg_off_host || !out_host || !workspace_host || !peer_bufs ||
      !local_bufs_host || (R_max > 0 && (!k_rest_host || !v_rest_host || !rest_len_host)))
    return fail(WQ_EINVAL, "NULL pointer array");
  if (epoch == 0) return fail(WQ_EINVAL, "epoch must start at 1");
  if (!((g && g->d == 128 && g->S == 32) || (g && g->d == 64 && g->S == 16)))
    return fail(WQ_EUNSUPPORTED, "emulation built for (d, S) = (128, 32) and (64, 16)");
  wq::DecodeArgs ra[2];
  for (int r = 0; r < G; r++) {
    if (!out_host[r]) return fail(WQ_EINVAL, "NULL out of rank %d", r);
    PeerCfg pc{reinterpret_cast<uint8_t *const *>(peer_bufs), local_bufs_host[r], G, r, epoch};
    wq_status s = decode_args(q_host[r], packed_host[r], offs_host[r], seg_off_host[r], g,
                              R_max > 0 ? k_rest_host[r] : nullptr, R_max > 0 ? v_rest_host[r] : nullptr,
                              rest_strides, R_max > 0 ? rest_len_host[r] : nullptr, R_max, sm_scale, out_host[r],
                              nullptr, workspace_host[r], workspace_bytes, 0u, nullptr, &pc, ra[r]);
    if (s != WQ_OK) return s;
  }
  return cuda_status(wq::launch_decode_emu(ra, G, wq::device_sm_count(), S_(stream)), "decode (peer emulation)");
}

wq_status wq_unreordered_layout(const wq_geom *g, const uint8_t *bits_l, int64_t *woff, void *stream) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!bits_l || !woff) return fail(WQ_EINVAL, "NULL pointer");
  return cuda_status(wq::launch_unreordered_layout(bits_l, g->B, g->M / g->S, g->d, g->S, woff, S_(stream)),
                     "unreordered layout");
}

wq_status wq_unreorder_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off_l,
                             const int32_t *perm_l, const wq_geom *g, const int64_t *woff, uint8_t *uimg,
                             void *stream) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!packed || !offs || !seg_off_l || !perm_l || !woff || !uimg) return fail(WQ_EINVAL, "NULL pointer");
  if (!aligned16(packed) || !aligned16(uimg)) return fail(WQ_EINVAL, "images must be 16-byte aligned");
  return cuda_status(wq::launch_unreorder_image(packed, offs, seg_off_l, perm_l, g->B, g->H, g->M / g->S, g->d, g->S,
                                                woff, uimg, S_(stream)),
                     "unreorder image");
}

wq_status wq_decode_attention_unreordered(const void *q, const uint8_t *uimg, const int64_t *offs,
                                          const int32_t *seg_off_l, const int64_t *woff, const wq_geom *g,
                                          const void *k_rest, const void *v_rest, const int64_t rest_strides[2],
                                          const int32_t *rest_len, int32_t R_max, float sm_scale, void *out,
                                          float *partial, void *workspace, size_t workspace_bytes, void *stream) {
  if (!woff) return fail(WQ_EINVAL, "NULL woff");
  return decode_impl(q, uimg, offs, seg_off_l, g, k_rest, v_rest, rest_strides, rest_len, R_max, sm_scale, out,
                     partial, workspace, workspace_bytes, 0u, woff, stream);
}

wq_status wq_merge_partials(const float *parts, int32_t G, const wq_geom *g, void *out, void *stream) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!parts || !out) return fail(WQ_EINVAL, "NULL pointer");
  if (G < 1) return fail(WQ_EINVAL, "G=%d", G);
  return cuda_status(wq::launch_merge(parts, G, g->B * g->Hq, g->d, (__half *)out, S_(stream)), "merge");
}

wq_status wq_shard_slots(const int32_t *perm_l, const int32_t *seg_off_l, int32_t B, int32_t W, int32_t G,
                         int32_t r, int32_t *perm_r, int32_t *seg_off_r, void *stream) {
  if (!perm_l || !seg_off_l || !perm_r || !seg_off_r) return fail(WQ_EINVAL, "NULL pointer");
  if (B < 1 || W < 1) return fail(WQ_ESHAPE, "B=%d W=%d", B, W);
  if (G < 1 || r < 0 || r >= G) return fail(WQ_EINVAL, "rank %d of %d", r, G);
  return cuda_status(wq::launch_shard_slots(perm_l, seg_off_l, B, W, G, r, perm_r, seg_off_r, S_(stream)),
                     "shard");
}

wq_status wq_dequant_layout(const wq_geom *g, const int32_t *seg_off_l, int32_t *seg16, int64_t *offs16, void *stream) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!seg_off_l || !seg16 || !offs16) return fail(WQ_EINVAL, "NULL pointer");
  if (g->B > 4096) return fail(WQ_ESHAPE, "B=%d > 4096", g->B);
  return cuda_status(wq::launch_dequant_layout(seg_off_l, g->B, g->H, g->d, g->S, seg16, offs16, S_(stream)),
                     "dequant layout");
}

wq_status wq_dequantize_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off_l, const wq_geom *g,
                              const int64_t *offs16, uint8_t *img16, void *stream) {
  wq_status s = check_geom(g, true);
  if (s != WQ_OK) return s;
  if (!packed || !offs || !seg_off_l || !offs16 || !img16) return fail(WQ_EINVAL, "NULL pointer");
  if (!aligned16(packed) || !aligned16(img16)) return fail(WQ_EINVAL, "images must be 16-byte aligned");
  const int W = g->M / g->S;
  return cuda_status(wq::launch_dequant_image(packed, offs, seg_off_l, g->B, g->H, W, g->d, g->S, offs16, img16,
                                              S_(stream)),
                     "dequantize image");
}

}  // extern "C"
