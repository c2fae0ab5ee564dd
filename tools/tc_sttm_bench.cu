// tc_sttm_bench.cu -- microbenchmark of tcgen05.st (16x256b.x8, 4 KB per warp instruction)
// issue and completion cost, as used by the dequantizer warps of k_decode_tc: per warp,
// N stores then tcgen05.wait::st, with 1, 2, 4 or 8 warps storing concurrently (each to
// its own TMEM lane quarter / columns).  Prints cycles per store per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/tc_sttm_bench tools/tc_sttm_bench.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NW>
__global__ void k_bench(long long *out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = taddr_s;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; i++) r[i] = lane * 32 + i;
  // warp w: lane quarter w % 4, column block (w / 4) * 64, half (16 lanes) by iteration parity
  const uint32_t base = t + ((uint32_t)(32 * (warp & 3)) << 16) + (warp >> 2) * 64;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t ta = base + ((uint32_t)(16 * (it & 1)) << 16) + ((it >> 1) & 1) * 128;
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
    r[it & 31] += 1;
  }
  long long t1 = clock64();
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  long long t2 = clock64();
  if (lane == 0) { out[2 * warp] = t1 - t0; out[2 * warp + 1] = t2 - t0; }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int NW>
void run(int iters) {
  long long *d, h[64];
  cudaMalloc(&d, sizeof(h));
  k_bench<NW><<<1, NW * 32>>>(d, iters);
  k_bench<NW><<<1, NW * 32>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(long long) * 2 * NW, cudaMemcpyDeviceToHost);
  double issue = 0, done = 0;
  for (int w = 0; w < NW; w++) { issue += h[2 * w]; done += h[2 * w + 1]; }
  printf("%d warps x %d STTM.16x256b.x8 (4 KB each): issue %.1f cyc/store/warp, complete %.1f cyc/store/warp, "
         "SM store rate %.1f B/cyc  %s\n", NW, iters, issue / NW / iters, done / NW / iters,
         NW * iters * 4096.0 / (done / NW), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<1>(256);
  run<2>(256);
  run<4>(256);
  run<8>(256);
  return 0;
}
