// wq_device.cuh -- device helpers for libwq (sm_100a): PTX wrappers for mbarrier,
// 1-D bulk copies (TMA, cp.async.bulk), mma.sync, ldmatrix, and the packed-layout
// constants of contract D-1 (include/wq.h).  Product code only; the CPU oracle
// (oracle/) re-derives the layout independently.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define WQ_DEV __device__ __forceinline__

namespace wq {

// bits of width class k (segment order of a packed image, Alg.2)
WQ_DEV int class_bits(int k) { return k == 0 ? 2 : k == 1 ? 4 : k == 2 ? 8 : 16; }

// Bytes of one window record (D-1): codes K|V, then (s, mn) params K|V.
__host__ __device__ __forceinline__ int64_t record_bytes(int bits, int d, int S) {
  return bits == 16 ? 4LL * S * d : (int64_t)S * d * bits / 4 + 4LL * d + 4LL * S;
}

// ---------------------------------------------------------------------------
// shared-memory addresses, mbarriers, bulk copies
// ---------------------------------------------------------------------------
WQ_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

WQ_DEV void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
WQ_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
WQ_DEV void mbar_arrive_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
WQ_DEV void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
WQ_DEV void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWQ_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WQ_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (TMA engine, 1-D), completes tx bytes on mbarrier b.
// dst/src 16-byte aligned, bytes a multiple of 16.
WQ_DEV void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
WQ_DEV void bulk_g2s_evict_first(void *dst, const void *src, uint32_t bytes, uint64_t *b,
                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(policy)
      : "memory");
}
WQ_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Programmatic dependent launch (PDL): wait for the prerequisite grid (no-op when the
// grid was launched without a programmatic dependency); allow dependents to launch.
WQ_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
WQ_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

WQ_DEV int atom_add_acq_rel_gpu(int *p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

WQ_DEV void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// shared memory vector loads
// ---------------------------------------------------------------------------
WQ_DEV uint4 lds128(const void *p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
WQ_DEV uint2 lds64(const void *p) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)));
  return v;
}
WQ_DEV uint32_t lds32(const void *p) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
  return v;
}
WQ_DEV void sts32(void *p, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

WQ_DEV void ldsm_x4(uint32_t (&r)[4], const void *row_addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(row_addr)));
}
WQ_DEV void ldsm_x4_t(uint32_t (&r)[4], const void *row_addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(row_addr)));
}
WQ_DEV void ldsm_x2_t(uint32_t (&r)[2], const void *row_addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(smem_u32(row_addr)));
}

// ---------------------------------------------------------------------------
// tensor core: D = A(16x16, row) * B(16x8, col) + C, fp16 in, fp32 accumulate
// ---------------------------------------------------------------------------
WQ_DEV void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                     const float (&c)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};\n"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]),
        "f"(c[2]), "f"(c[3]));
}

// ---------------------------------------------------------------------------
// packed fp16x2 helpers
// ---------------------------------------------------------------------------
WQ_DEV uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }
WQ_DEV __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2 *>(&u); }
WQ_DEV uint32_t hmul2u(uint32_t a, uint32_t b) { return h2u(__hmul2(u2h(a), u2h(b))); }
// exact residual a*b - c with a single rounding (fp16 FMA)
WQ_DEV uint32_t hfma2u(uint32_t a, uint32_t b, uint32_t c) {
  return h2u(__hfma2(u2h(a), u2h(b), u2h(c)));
}
WQ_DEV uint32_t hneg2u(uint32_t a) { return a ^ 0x80008000u; }
WQ_DEV uint32_t pack_f2h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
WQ_DEV uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t magic) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(r) : "r"(a), "r"(mask), "r"(magic));  // (a & b) | c
  return r;
}

// Exact fp16 values of the two codes of pair slot P in word w (D-1 packing):
// element e sits at bit 16*e + BITS*j.  A code at bit p of each half is ORed into
// the mantissa of 2^(10-p)*(1 + .) (exponent field 25 - p), giving 2^(10-p) + code
// exactly; subtracting 2^(10-p) leaves the code (CENTER: subtracting
// 2^(10-p) + 2^(BITS-1) leaves code - 2^(BITS-1), also exact).  Positions
// p + BITS <= 10 only; higher slots use the word shifted right by 8.
template <int BITS, int J, bool CENTER = false>
WQ_DEV uint32_t dq_pair(uint32_t w, uint32_t w8) {
  constexpr int SLOT_BITS = BITS * J;
  constexpr bool HI = (SLOT_BITS + BITS > 10);
  constexpr int P = HI ? SLOT_BITS - 8 : SLOT_BITS;
  constexpr uint32_t MASK1 = ((1u << BITS) - 1u) << P;
  constexpr uint32_t MASK = MASK1 | (MASK1 << 16);
  constexpr uint32_t MAG1 = (uint32_t)(25 - P) << 10;
  constexpr uint32_t MAG = MAG1 | (MAG1 << 16);
  constexpr uint32_t SUB1 = MAG1 | (CENTER ? (1u << (BITS - 1)) << P : 0u);
  constexpr uint32_t SUB = SUB1 | (SUB1 << 16);
  uint32_t x = lop3_and_or(HI ? w8 : w, MASK, MAG);
  return h2u(__hsub2(u2h(x), u2h(SUB)));
}
// 8-bit codes: bytes 0/2 (J = 0) or 1/3 (J = 1) under the exponent byte 0x64 -> 1024 + code
template <int J, bool CENTER = false>
WQ_DEV uint32_t dq_pair8(uint32_t w) {
  uint32_t x;
  if constexpr (J == 0) asm("prmt.b32 %0, %1, %2, 0x7250;" : "=r"(x) : "r"(w), "r"(0x64646464u));
  else asm("prmt.b32 %0, %1, %2, 0x7351;" : "=r"(x) : "r"(w), "r"(0x64646464u));
  return h2u(__hsub2(u2h(x), u2h(CENTER ? 0x64806480u : 0x64006400u)));
}

WQ_DEV float warp_max(float v, int xor_from = 1) {
  for (int o = 16; o >= xor_from; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace wq
