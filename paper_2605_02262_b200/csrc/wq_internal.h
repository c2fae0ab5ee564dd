// wq_internal.h -- launchers shared between the kernels (*.cu) and the C ABI (abi.cu).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace wq {

constexpr int MAX_LAYERS = 64;

struct AssignParams {
  int L, B, W, n_widths, widths[4];
  int pin, vote;
  double budget;
  double thr[MAX_LAYERS * 3];
};

cudaError_t launch_text_pool(const __half *txt, int64_t trs, int64_t tbs, int B, int N, int D,
                             double *tbar, int metric, cudaStream_t st);
cudaError_t launch_window_scores(const __half *vis, int64_t vrs, int64_t vbs, int B, int M, int N,
                                 int D, int S, const double *tbar, double *scores, int metric, cudaStream_t st,
                                 int dh = 0, int64_t hs = 0);
cudaError_t launch_text_pool_q(const __half *qt, int64_t qsb, int64_t qsh, int64_t qsj, int B, int N, int H,
                               int grp, int d, double *tbar, cudaStream_t st);

cudaError_t launch_rank(const double *scores, int B, int W, int32_t *rank, cudaStream_t st);
cudaError_t launch_assign(const double *scores, const AssignParams &p, uint8_t *bits, int32_t *perm,
                          int32_t *seg_off, cudaStream_t st);

// the fused search (search.cu): scores + rank + assign of every layer in one launch
size_t search_smem(int W, int D);
cudaError_t launch_search(const __half *vis, int64_t vrs, int64_t vbs, const __half *txt, int64_t trs, int64_t tbs,
                          int B, int M, int N, int D, int S, int metric, const AssignParams &p, double *tbar,
                          double *scores, int32_t *order, uint8_t *bits, int32_t *rank, int32_t *perm, int32_t *seg,
                          cudaStream_t st);

cudaError_t launch_layer_layout(const int32_t *seg_off, int B, int H, int d, int S, int gran, int64_t *offs,
                                cudaStream_t st);
cudaError_t launch_shard_slots(const int32_t *perm, const int32_t *seg, int B, int W, int G, int r,
                               int32_t *perm_r, int32_t *seg_r, cudaStream_t st);
cudaError_t launch_quant(const __half *k, const __half *v, const int64_t strides[3], int vis_off,
                         int B, int H, int d, int S, int M, const int32_t *perm, int perm_stride,
                         const int32_t *seg_off, const int64_t *offs, uint8_t *packed, int gran,
                         cudaStream_t st);

struct DecodeArgs {
  const __half *q;
  const uint8_t *packed;
  const int64_t *offs;
  const int32_t *seg_off;
  const __half *k_rest, *v_rest;
  int64_t rs_b, rs_h;
  const int32_t *rest_len;
  int R_max;
  int B, H, Hq, grp, d, S;
  float scale_log2;          // sm_scale * log2(e)
  uint32_t flags;            // WQ_DECODE_* flags (include/wq.h)
  __half *out;
  float *partial;
  float *ws_part;            // [(G + B*H)][grp][d + 2]
  int32_t *ws_cnt;           // [B*H]
  uint64_t *ws_ts;           // [num_sms][TS_PER_CTA] timestamps (profiling builds, WQ_DECODE_DEBUG & 8), else NULL
  const int64_t *woff;       // non-NULL: unreordered image, window offsets [B][W+1]
  // fused cross-GPU LSE merge; peer_bufs NULL: off
  uint8_t *const *peer_bufs; // device array [G] of the ranks' symmetric buffers (IPC-mapped)
  int peer_G, peer_rank;
  uint32_t peer_epoch;       // 1, 2, ... per call: the counters reach G * epoch
  __half *peer_out;          // out [B][Hq][d] of the merged result
};
size_t peer_buffer_bytes(int B, int H, int Hq, int d, int G);
struct DecodeWsLayout {
  size_t part, cnt, ts;      // bytes of the partial slots, the counters, the timestamps
};
DecodeWsLayout decode_ws_layout(int B, int H, int d, int num_sms);
size_t decode_workspace_bytes(int B, int H, int Hq, int d, int num_sms);
cudaError_t launch_decode(const DecodeArgs &a, int num_sms, cudaStream_t st);
cudaError_t launch_decode_tc(const DecodeArgs &a, int num_sms, cudaStream_t st);   // d = 128
// nr virtual ranks of the fused peer merge in one launch (tests; nr = 2, (d, S) = (128, 32) / (64, 16))
cudaError_t launch_decode_emu(const DecodeArgs *ra, int nr, int num_sms, cudaStream_t st);
cudaError_t launch_merge(const float *parts, int G, int BHq, int d, __half *out, cudaStream_t st);

cudaError_t launch_dequant_layout(const int32_t *seg_off, int B, int H, int d, int S, int32_t *seg16, int64_t *offs16,
                                  cudaStream_t st);
cudaError_t launch_dequant_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off, int B, int H,
                                 int W, int d, int S, const int64_t *offs16, uint8_t *img16, cudaStream_t st);

cudaError_t launch_unreordered_layout(const uint8_t *bits_l, int B, int W, int d, int S, int64_t *woff, cudaStream_t st);
cudaError_t launch_unreorder_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off,
                                   const int32_t *perm_l, int B, int H, int W, int d, int S, const int64_t *woff,
                                   uint8_t *uimg, cudaStream_t st);

int device_sm_count();

}  // namespace wq
