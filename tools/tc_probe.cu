// tc_probe.cu -- standalone check of the tcgen05 building blocks the decode kernel
// uses (sm_100a): TMEM alloc, tcgen05.st 32x32b / 16x256b register layouts, A operand
// in TMEM, B operand in shared memory (K-major and MN-major, no swizzle, core-matrix
// strides LBO/SBO), tcgen05.mma kind::f16 M=128 with N = 8/16/32/64, commit to an
// mbarrier, tcgen05.ld 32x32b.  Every case is compared against a CPU fp64 product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/tc_probe tools/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>

#define DEV __device__ __forceinline__
DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

DEV void tmem_alloc(uint32_t *dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
DEV void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DEV void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
DEV void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
DEV void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

DEV void st_32x32b_x8(uint32_t ta, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
DEV void st_16x256b_x1(uint32_t ta, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(r0), "r"(r1),
               "r"(r2), "r"(r3)
               : "memory");
}
DEV void ld_32x32b_x8(uint32_t ta, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
}
DEV void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
DEV void mbar_wait(uint64_t *b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(b)),
               "r"(par)
               : "memory");
}
DEV void mma_commit(uint64_t *b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
DEV void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__host__ __device__ uint32_t make_idesc(int M, int N, int b_mn_major) {
  return (1u << 4)                      // D fp32
         | (0u << 7) | (0u << 10)       // A, B fp16
         | ((uint32_t)b_mn_major << 16) // B major
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
DEV uint64_t make_sdesc(const void *p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= 1ull << 46;                      // version (sm_100)
  return d;                             // base offset 0, lbo mode 0, SWIZZLE_NONE
}

// One test: A [128][K] fp16 (row-major, global), B [N][K] fp16 (global, n-major rows).
// mode bit0: A stored with 16x256b in mma-fragment order (else 32x32b natural)
// mode bit1: B MN-major in smem (else K-major)
// D[128][N] fp32 out.
__global__ void k_probe(const __half *A, const __half *B, float *D, int K, int N, int mode, uint32_t lbo,
                        uint32_t sbo) {
  __shared__ __align__(1024) uint8_t bs[40 * 1024];
  __shared__ uint32_t taddr_s;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc(&taddr_s, 256);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = taddr_s;
  const uint32_t tA = tbase, tD = tbase + 128;  // A: cols [0, K/2), D: cols [128, 128+N)
  // --- B into shared memory (core matrices of 8 x 16 B) ---
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    size_t off;
    if (mode & 2) off = (size_t)(n % 8) * 2 + (size_t)(k % 8) * 16 + (size_t)(k / 8) * lbo + (size_t)(n / 8) * sbo;
    else off = (size_t)(k % 8) * 2 + (size_t)(n % 8) * 16 + (size_t)(k / 8) * lbo + (size_t)(n / 8) * sbo;
    *reinterpret_cast<__half *>(bs + off) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  // --- A into TMEM ---
  const int row0 = 32 * (warp & 3);
  if (!(mode & 1)) {
    const int r = row0 + lane;
    for (int c8 = 0; c8 < K / 16; c8++) {       // 8 columns (16 halves) per store
      uint32_t v[8];
      for (int j = 0; j < 8; j++) {
        __half2 h = __halves2half2(A[r * K + 16 * c8 + 2 * j], A[r * K + 16 * c8 + 2 * j + 1]);
        v[j] = *reinterpret_cast<uint32_t *>(&h);
      }
      st_32x32b_x8(tA + ((uint32_t)row0 << 16) + 8 * c8, v);
    }
  } else {
    // mma.sync A fragment of rows [r16, r16+16), k-block m: a0 (g, 2q), a1 (g+8, 2q),
    // a2 (g, 2q+8), a3 (g+8, 2q+8); stored as {a0, a2, a1, a3}
    const int g = lane >> 2, q = lane & 3;
    for (int half = 0; half < 2; half++) {
      const int r16 = row0 + 16 * half;
      for (int m = 0; m < K / 16; m++) {
        auto pr = [&](int row, int col) {
          __half2 h = __halves2half2(A[row * K + col], A[row * K + col + 1]);
          return *reinterpret_cast<uint32_t *>(&h);
        };
        const uint32_t a0 = pr(r16 + g, 16 * m + 2 * q), a1 = pr(r16 + g + 8, 16 * m + 2 * q);
        const uint32_t a2 = pr(r16 + g, 16 * m + 2 * q + 8), a3 = pr(r16 + g + 8, 16 * m + 2 * q + 8);
        st_16x256b_x1(tA + ((uint32_t)r16 << 16) + 8 * m, a0, a2, a1, a3);
      }
    }
  }
  st_wait();
  fence_before();
  __syncthreads();
  if (tid == 0) {
    fence_after();
    const uint32_t idesc = make_idesc(128, N, (mode & 2) ? 1 : 0);
    for (int ks = 0; ks < K / 16; ks++) {
      // K-major: K step of 16 = 2 core matrices along K = 2*lbo; MN-major: 2 K-groups of 8 rows = 2*lbo
      const uint64_t bd = make_sdesc(bs + (size_t)ks * 2 * lbo, lbo, sbo);
      mma_ts(tD, tA + 8 * ks, bd, idesc, ks > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  const int r = row0 + lane;
  for (int c8 = 0; c8 < N / 8; c8++) {
    uint32_t v[8];
    ld_32x32b_x8(tD + ((uint32_t)row0 << 16) + 8 * c8, v);
    ld_wait();
    for (int j = 0; j < 8; j++) D[r * N + 8 * c8 + j] = __uint_as_float(v[j]);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

// The fragment-order A store permutes K within each 16-block: TMEM column pair p of
// block m holds K elements 16m + 2*(p>>1) + 8*(p&1) + {0,1}.  kperm(k') = that element.
static int kperm(int kp) {
  const int m = kp / 16, r = kp % 16, p = r / 2, e = r % 2;
  return 16 * m + 2 * (p >> 1) + 8 * (p & 1) + e;
}

int main() {
  struct Case { int K, N, mode; };
  Case cases[] = {{16, 32, 0}, {128, 32, 0}, {128, 32, 1}, {128, 64, 1}, {128, 16, 2}, {128, 8, 2},
                  {128, 16, 3}, {128, 8, 0}, {64, 16, 1}, {128, 128, 1}};
  int fails = 0;
  for (const Case &cs : cases) {
    const int M = 128, K = cs.K, N = cs.N;
    std::vector<__half> hA(M * K), hB(N * K);
    std::vector<float> fA(M * K), fB(N * K);
    srand(K * 131 + N * 7 + cs.mode);
    for (int i = 0; i < M * K; i++) { fA[i] = (float)((rand() % 17) - 8); hA[i] = __float2half(fA[i]); }
    for (int i = 0; i < N * K; i++) { fB[i] = (float)((rand() % 2001) - 1000) / 256.f; hB[i] = __float2half(fB[i]); fB[i] = __half2float(hB[i]); }
    __half *dA, *dB; float *dD;
    cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, M * N * 4);
    // K-major: LBO = 128 (next 8 K), SBO = (K/8)*128 (next 8 N rows)
    // MN-major: LBO = (N/8)*128 ... we put N-groups adjacent: SBO = 128, LBO = (N/8)*128
    uint32_t lbo, sbo;
    if (cs.mode & 2) { sbo = 128; lbo = (uint32_t)((N + 7) / 8) * 128; }
    else { lbo = 128; sbo = (uint32_t)(K / 8) * 128; }
    k_probe<<<1, 128>>>(dA, dB, dD, K, N, cs.mode, lbo, sbo);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(M * N);
    cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxerr_perm = 0;
    for (int m = 0; m < M; m++)
      for (int n = 0; n < N; n++) {
        double ref = 0, refp = 0;
        for (int k = 0; k < K; k++) {
          ref += (double)fA[m * K + k] * fB[n * K + k];
          // permuted: A element kperm(k') meets B element k'
          refp += (double)fA[m * K + kperm(k)] * fB[n * K + k];
        }
        maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
        maxerr_perm = fmax(maxerr_perm, fabs(refp - hD[m * N + n]));
      }
    const double err = (cs.mode & 1) ? maxerr_perm : maxerr;
    const bool ok = e == cudaSuccess && err < 1e-3;
    fails += !ok;
    printf("K=%3d N=%3d mode=%d (A %s, B %s) lbo=%u sbo=%u: %s  err=%.3g (natural %.3g, permuted %.3g) D[0]=%g %s\n", K, N,
           cs.mode, (cs.mode & 1) ? "16x256b" : "32x32b", (cs.mode & 2) ? "MN" : "K", lbo, sbo,
           ok ? "OK" : "FAIL", err, maxerr, maxerr_perm, hD[0], cudaGetErrorString(e));
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    if (e != cudaSuccess) break;
  }
  printf("%s\n", fails ? "PROBE FAILED" : "PROBE OK");
  return fails ? 1 : 0;
}
