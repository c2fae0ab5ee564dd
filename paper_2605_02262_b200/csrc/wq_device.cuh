// wq_device.cuh -- device helpers for libwq (sm_100a): PTX wrappers for mbarrier,
// 1-D bulk copies (TMA, cp.async.bulk), mma.sync, ldmatrix, and the packed-layout
// constants of contract D-1 (include/wq.h).  Product code only; the CPU oracle
// (oracle/) re-derives the layout independently.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define WQ_DEV __device__ __forceinline__

// Checked builds (-DWQ_CHECKS=1, tests/test_gpu_checked.py): device-side bounds checks on
// every bulk copy, record write and permutation index of the path; a failed check prints
// its condition and traps (the call then fails with a CUDA error).  Product builds compile
// the checks out.
#ifndef WQ_CHECKS
#define WQ_CHECKS 0
#endif
#if WQ_CHECKS
#include <cstdio>
#define WQ_CHECK(cond)                                                                   \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("WQ_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,       \
             (int)blockIdx.x, (int)threadIdx.x, #cond);                                  \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define WQ_CHECK(cond) do { } while (0)
#endif

namespace wq {

// bits of width class k (segment order of a packed image, Alg.2)
WQ_DEV int class_bits(int k) { return k == 0 ? 2 : k == 1 ? 4 : k == 2 ? 8 : 16; }

// Bytes of one window record (D-1): codes K|V, then (s, mn) params K|V -- per channel /
// per token (gran 0), or one 16-byte block {mn_K, s_K, mn_V, s_V, 0...} per window-head
// (gran 1: the paper-literal groups of P:508, reading Q37).
__host__ __device__ __forceinline__ int64_t record_bytes(int bits, int d, int S, int gran = 0) {
  return bits == 16 ? 4LL * S * d : (int64_t)S * d * bits / 4 + (gran ? 16LL : 4LL * d + 4LL * S);
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
// blocking wait with a suspend-time hint: the thread sleeps in hardware until the phase
// completes (no spin loop competing for issue slots)
WQ_DEV void mbar_wait_hint(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWQ_WAITH_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WQ_WAITH_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(0x989680)
      : "memory");
}
// non-blocking: has the phase with this parity completed?
WQ_DEV bool mbar_test(uint64_t *b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// polling wait with a nanosleep back-off, for waiters off the critical path (the
// producer refilling a ring slot, consumers idling while the bottleneck stage runs)
WQ_DEV void mbar_wait_sleep(uint64_t *b, uint32_t parity, uint32_t ns) {
  while (!mbar_test(b, parity)) __nanosleep(ns);
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

WQ_DEV uint64_t gtime() {      // profiling clock (debug & 8 only): global ns timer
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// tcgen05 (5th-gen tensor cores) and tensor memory, sm_100a.  Register layouts
// and descriptor encodings verified against a CPU product by tools/tc_probe.cu.
// ---------------------------------------------------------------------------
WQ_DEV void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {     // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
WQ_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {      // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
WQ_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
WQ_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
WQ_DEV void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
WQ_DEV void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
WQ_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16 TMEM lanes x 256 bits, x1: thread t holds r0,r1 = (lane t/4, cols 2(t%4), +1),
// r2,r3 = (lane t/4 + 8, same cols): an mma.sync A fragment {a0,a1,a2,a3} stored as
// {a0,a2,a1,a3} puts column pair p of each k16 block at elements 2(p>>1)+8(p&1)+{0,1}.
WQ_DEV void tmem_st_16x256b_x1(uint32_t ta, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(r0), "r"(r1),
               "r"(r2), "r"(r3)
               : "memory");
}
// x8: 8 consecutive 8-column blocks, registers 4i..4i+3 -> block i
WQ_DEV void tmem_st_16x256b_x8(uint32_t ta, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// 32 lanes x 32 bits: thread t <-> lane (warp%4)*32 + t, registers = 8 consecutive columns
WQ_DEV void tmem_ld_32x32b_x8(uint32_t ta, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta)
               : "memory");
}
WQ_DEV void tmem_ld_32x32b_x16(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta)
      : "memory");
}
WQ_DEV void tmem_st_32x32b_x8(uint32_t ta, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem descriptor], kind::f16, fp32 accumulate (one thread)
WQ_DEV void tc_mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on an mbarrier once every previously issued tcgen05.mma of this thread completed
WQ_DEV void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// warp-wide variants: every lane executes, one elected lane issues
WQ_DEV void tc_mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
WQ_DEV void tc_commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// instruction descriptor: fp16 A/B, fp32 D, A K-major, B K-major (0) or MN-major (1)
__host__ __device__ constexpr uint32_t tc_idesc_f16(int M, int N, int b_mn_major) {
  return (1u << 4) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// shared-memory matrix descriptor, no swizzle: core matrices of 8 rows x 16 B;
// lbo = byte stride between core matrices along K, sbo = along M/N
WQ_DEV uint64_t tc_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
WQ_DEV void mbar_arrive_cnt(uint64_t *b, uint32_t cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
WQ_DEV void sts128(void *p, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
WQ_DEV void sts64(void *p, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(smem_u32(p)), "r"(x), "r"(y) : "memory");
}

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
#ifndef WQ_EXP_NOSUB
#define WQ_EXP_NOSUB 0     // timing experiments only (tools/ubench_window.cu): skip the HSUB2 of the
#endif                     // dequantization on the K side (1), the V side (2) or both (3): wrong values
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
  if constexpr ((WQ_EXP_NOSUB & (CENTER ? 2 : 1)) != 0) return x;
  return h2u(__hsub2(u2h(x), u2h(SUB)));
}
// 8-bit codes: bytes 0/2 (J = 0) or 1/3 (J = 1) under the exponent byte 0x64 -> 1024 + code
template <int J, bool CENTER = false>
WQ_DEV uint32_t dq_pair8(uint32_t w) {
  uint32_t x;
  if constexpr (J == 0) asm("prmt.b32 %0, %1, %2, 0x7250;" : "=r"(x) : "r"(w), "r"(0x64646464u));
  else asm("prmt.b32 %0, %1, %2, 0x7351;" : "=r"(x) : "r"(w), "r"(0x64646464u));
  if constexpr ((WQ_EXP_NOSUB & (CENTER ? 2 : 1)) != 0) return x;
  return h2u(__hsub2(u2h(x), u2h(CENTER ? 0x64806480u : 0x64006400u)));
}

WQ_DEV float ex2f(float x) {                 // 2^x, MUFU.EX2 (rel. error ~2^-22, denormals flushed)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

WQ_DEV float warp_max(float v, int xor_from = 1) {
  for (int o = 16; o >= xor_from; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace wq
