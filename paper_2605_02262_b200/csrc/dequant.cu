// dequant.cu -- the UNFUSED baseline of the paper's fusion ablation (T9, P:1026-1027;
// P:510 fuses the dequantization into attention, the ablation dequantizes the whole
// cache to FP16 in HBM first).  SURVEY.md §8(f) row 3.
//
// wq_dequantize_image: every window record of a packed layer image (contract D-1) is
// rewritten as an FP16 record of the same slot (same fragment order, segments kept in
// slot order), x^16 = RN_fp16(mn + s * code) -- the exact dequantized value (Eq.15 with
// z = -mn/s, reading Q17) rounded once to fp16.  FP16 records are copied.  The FP16
// image is then decoded by the ordinary decode kernel with every slot in class 16.
// Work item = 4 element pairs (lane chunk pairs 4m..4m+3 of one 16-token tile); the
// fragment position of a pair is the same in the b-bit and the FP16 record, only the
// packing differs.  HBM-bound: read the record, write 4*S*d bytes.
#include "wq_device.cuh"
#include "wq_internal.h"

namespace wq {

template <int D, int S>
__global__ void __launch_bounds__(256, 8) k_dequant_image(const uint8_t *__restrict__ packed, const int64_t *__restrict__ offs,
                                                       const int32_t *__restrict__ seg_off, int H,
                                                       const int64_t *__restrict__ offs16, uint8_t *__restrict__ img16) {
  const int u = blockIdx.y, b = u / H;
  const int32_t *so = seg_off + 5 * b;
  const int slot = blockIdx.x;
  if (slot >= so[4]) return;
  int k = 0;
  while (k < 3 && slot >= so[k + 1]) k++;
  int64_t roff = 0;
  for (int kk = 0; kk < k; kk++) roff += (int64_t)(so[kk + 1] - so[kk]) * record_bytes(class_bits(kk), D, S);
  const int bits = class_bits(k);
  const uint8_t *rec = packed + offs[u] + roff + (int64_t)(slot - so[k]) * record_bytes(bits, D, S);
  uint8_t *dst = img16 + offs16[u] + (int64_t)slot * (4LL * S * D);
  if (bits == 16) {                              // already FP16: copy the record
    const uint4 *s4 = reinterpret_cast<const uint4 *>(rec);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    for (int i = threadIdx.x; i < S * D / 4; i += blockDim.x) d4[i] = s4[i];
    return;
  }
  const int PPW = 16 / bits;
  const int WPL = D * bits / 64;                 // words per lane chunk of a code tile
  const int64_t kbytes = (int64_t)S * D * bits / 8;
  const __half *kp = reinterpret_cast<const __half *>(rec + 2 * kbytes);
  const __half *vp = kp + 2 * D;
  // work item = (K|V, tile, k16 block m, lane L): the 4 pairs P = 4m..4m+3 of lane L's
  // chunk -> one 16-byte FP16 store; consecutive threads write consecutive 16 B.  All of
  // a thread's loads are issued before any arithmetic (latency, not bandwidth, bounds
  // a thread's items otherwise).
  constexpr int NIT = (S / 16) * (D / 16) * 32;
  constexpr int IPT = (2 * NIT + 255) / 256;         // items per thread (blockDim 256)
  const uint32_t msk = (1u << bits) - 1u;
  auto wofs = [&](int w, int L) -> int64_t {
    return WPL >= 4 ? (int64_t)(w >> 2) * 512 + L * 16 + (w & 3) * 4 : (int64_t)L * 8 + 4 * w;
  };
  uint4 pq[IPT];
  uint32_t wa[IPT], wb[IPT];
#pragma unroll
  for (int i = 0; i < IPT; i++) {
    const int it = threadIdx.x + 256 * i;
    if (it >= 2 * NIT) break;
    const int isv = it >= NIT, x = isv ? it - NIT : it;
    const int L = x & 31, m = (x >> 5) % (D / 16), tile = (x >> 5) / (D / 16), q = L & 3;
    const uint8_t *tb = rec + (isv ? kbytes : 0) + (int64_t)tile * 2 * D * bits;
    // one 16-byte parameter group serves the lane's 4 pairs: K group (q, m) =
    // {mn01, s01, mn89, s89}; V group (tile, q) = {s01, s89, mn01, mn89} (D-1)
    pq[i] = __ldg(reinterpret_cast<const uint4 *>(isv ? vp + (4 * tile + q) * 8 : kp + (4 * m + q) * 8));
    const int w0 = (4 * m) / PPW;
    wa[i] = __ldg(reinterpret_cast<const uint32_t *>(tb + wofs(w0, L)));
    wb[i] = bits == 8 ? __ldg(reinterpret_cast<const uint32_t *>(tb + wofs(w0 + 1, L))) : wa[i];
  }
#pragma unroll
  for (int i = 0; i < IPT; i++) {
    const int it = threadIdx.x + 256 * i;
    if (it >= 2 * NIT) break;
    const int isv = it >= NIT, x = isv ? it - NIT : it;
    const int L = x & 31, m = (x >> 5) % (D / 16), tile = (x >> 5) / (D / 16);
    const uint32_t mnw[2] = {isv ? pq[i].z : pq[i].x, isv ? pq[i].w : pq[i].z};
    const uint32_t sw[2] = {isv ? pq[i].x : pq[i].y, isv ? pq[i].y : pq[i].w};
    uint32_t out[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int j = (4 * m + r) % PPW;
      const uint32_t word = (bits == 8 && r >= 2) ? wb[i] : wa[i];
      // both codes as exact fp16 integers: (1024 + code) - 1024
      const uint32_t cc = ((word >> (bits * j)) & (msk | (msk << 16))) | 0x64006400u;
      const __half2 code = __hsub2(u2h(cc), u2h(0x64006400u));
      // x^16 = RN_fp16(mn + s * code): one fused fp16 multiply-add = one rounding of the
      // exact value (s * code and the sum are formed exactly inside the FMA)
      out[r] = h2u(__hfma2(u2h(sw[r >> 1]), code, u2h(mnw[r >> 1])));
    }
    // FP16 tile: 32-word lane chunks, words 4m..4m+3 of lane L at m*512 + L*16
    uint8_t *ob = dst + (isv ? (int64_t)S * D * 2 : 0) + (int64_t)tile * 32 * D;
    *reinterpret_cast<uint4 *>(ob + m * 512 + L * 16) = make_uint4(out[0], out[1], out[2], out[3]);
  }
}

// seg16[b] = {0, 0, 0, 0, nslots_b}: every slot of the FP16 image is in class 16
__global__ void k_seg16(const int32_t *seg_off, int B, int32_t *seg16) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  for (int k = 0; k < 4; k++) seg16[5 * b + k] = 0;
  seg16[5 * b + 4] = seg_off[5 * b + 4];
}

cudaError_t launch_dequant_layout(const int32_t *seg_off, int B, int H, int d, int S, int32_t *seg16, int64_t *offs16,
                                  cudaStream_t st) {
  k_seg16<<<(B + 127) / 128, 128, 0, st>>>(seg_off, B, seg16);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_layer_layout(seg16, B, H, d, S, 0, offs16, st);
}

cudaError_t launch_dequant_image(const uint8_t *packed, const int64_t *offs, const int32_t *seg_off, int B, int H,
                                 int W, int d, int S, const int64_t *offs16, uint8_t *img16, cudaStream_t st) {
  if (W < 1) return cudaSuccess;
  const dim3 grid(W, B * H);
#define WQ_DQ(DD, SS) \
  if (d == DD && S == SS) { k_dequant_image<DD, SS><<<grid, 256, 0, st>>>(packed, offs, seg_off, H, offs16, img16); return cudaGetLastError(); }
  WQ_DQ(64, 16) WQ_DQ(64, 32) WQ_DQ(64, 64) WQ_DQ(64, 128)
  WQ_DQ(128, 16) WQ_DQ(128, 32) WQ_DQ(128, 64) WQ_DQ(128, 128)
#undef WQ_DQ
  return cudaErrorInvalidValue;
}

}  // namespace wq
