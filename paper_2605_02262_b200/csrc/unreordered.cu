// unreordered.cu -- the "Module III off" baseline of the paper's reordering ablation
// (T8; without reordering, windows of different precision sit
// interleaved in the cache).  SURVEY.md §8(f) row 1.
//
// The unreordered image holds exactly the window records of the packed image (each
// record is quantized independently, so the bytes are the same), but in ORIGINAL window
// order: record of window w of request b at offs[b*H + h] + woff[b][w], woff the prefix
// of the record sizes in window order (shared by the heads of a request).  The decode of
// this image (wq_decode_attention_unreordered) visits windows in original order and
// dispatches each window on its own width (decode.cu, UR instantiation).
#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {

// woff[b][w] = sum_{w' < w} record_bytes(bits[b][w']), w = 0..W (block scan per request)
__global__ void k_unreordered_layout(const uint8_t *__restrict__ bits_l, int W, int d, int S, int64_t *__restrict__ woff) {
  const int b = blockIdx.x;
  __shared__ int64_t carry;
  __shared__ int64_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int base = 0; base < W; base += blockDim.x) {
    const int w = base + threadIdx.x;
    const int64_t v = w < W ? record_bytes(bits_l[(int64_t)b * W + w], d, S) : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int64_t pre = carry;
    for (int i = 0; i < warp; i++) pre += wsum[i];
    if (w < W) woff[(int64_t)b * (W + 1) + w] = pre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int i = 0; i < nw; i++) t += wsum[i];
      carry += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) woff[(int64_t)b * (W + 1) + W] = carry;
}

// copy the record of slot i (window perm[b][i]) to its original-order position
__global__ void k_unreorder_image(const uint8_t *__restrict__ packed, const int64_t *__restrict__ offs,
                                  const int32_t *__restrict__ seg_off, const int32_t *__restrict__ perm_l, int W, int H,
                                  int d, int S, const int64_t *__restrict__ woff, uint8_t *__restrict__ uimg) {
  const int u = blockIdx.y, b = u / H;
  const int32_t *so = seg_off + 5 * b;
  const int slot = blockIdx.x;
  if (slot >= so[4]) return;
  int k = 0;
  while (k < 3 && slot >= so[k + 1]) k++;
  int64_t roff = 0;
  for (int kk = 0; kk < k; kk++) roff += (int64_t)(so[kk + 1] - so[kk]) * record_bytes(class_bits(kk), d, S);
  const int64_t rb = record_bytes(class_bits(k), d, S);
  const uint4 *src = reinterpret_cast<const uint4 *>(packed + offs[u] + roff + (int64_t)(slot - so[k]) * rb);
  const int w = perm_l[(int64_t)b * W + slot];
  uint4 *dst = reinterpret_cast<uint4 *>(uimg + offs[u] + woff[(int64_t)b * (W + 1) + w]);
  for (int i = threadIdx.x; i < rb / 16; i += blockDim.x) dst[i] = src[i];
}

cudaError_t launch_unreordered_layout(const uint8_t *bits_l, int B, int W, int d, int S, int64_t *woff, cudaStream_t st) {
  k_unreordered_layout<<<B, 256, 0, st>>>(bits_l, W, d, S, woff);
  return cudaGetLastError();
}

cudaError_t launch_unreorder_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off,
                                   const int32_t *perm_l, int B, int H, int W, int d, int S, const int64_t *woff,
                                   uint8_t *uimg, cudaStream_t st) {
  if (W < 1) return cudaSuccess;
  k_unreorder_image<<<dim3(W, B * H), 128, 0, st>>>(packed, offs, seg_off, perm_l, W, H, d, S, woff, uimg);
  return cudaGetLastError();
}

}  // namespace wq
