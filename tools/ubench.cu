// Microbenchmarks for design decisions (B200, sm_100a): legacy mma.sync rate,
// dequant ALU rate, 1-D bulk-copy (TMA) streaming vs LDG streaming, fp64 FMA rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void k_mma(float* out, int iters, long long* clk) {
  uint32_t a0=0x3c003c00u+threadIdx.x,a1=a0^1,a2=a0^2,a3=a0^3,b0=0x3c003c00u,b1=b0^5;
  float acc[8][4]; for(int i=0;i<8;i++) for(int j=0;j<4;j++) acc[i][j]=0.f;
  long long t0=clock64();
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<8;i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
        : "+f"(acc[i][0]),"+f"(acc[i][1]),"+f"(acc[i][2]),"+f"(acc[i][3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));
  }
  long long t1=clock64();
  float s=0; for(int i=0;i<8;i++) for(int j=0;j<4;j++) s+=acc[i][j];
  if(s==12345.f) out[0]=s;
  if(threadIdx.x==0 && blockIdx.x==0) clk[0]=t1-t0;
}

__global__ void k_deq(uint32_t* out, int iters, long long* clk) {
  uint32_t w = threadIdx.x*0x9e3779b9u; uint32_t acc[8]={0,0,0,0,0,0,0,0};
  long long t0=clock64();
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int j=0;j<8;j++){
      uint32_t x; asm volatile("lop3.b32 %0, %1, %2, %3, 0xea;\n" : "=r"(x) : "r"(w), "r"(0x00030003u<<(2*(j&3))), "r"(0x64006400u));
      __half2 h = *reinterpret_cast<__half2*>(&x);
      __half2 m = __halves2half2(__ushort_as_half(0x6400),__ushort_as_half(0x6400));
      h = __hsub2(h, m);
      acc[j] ^= *reinterpret_cast<uint32_t*>(&h);
    }
    w = w*1664525u+1013904223u;
  }
  long long t1=clock64();
  uint32_t s=0; for(int j=0;j<8;j++) s^=acc[j];
  if(s==0x12345678u) out[0]=s;
  if(threadIdx.x==0 && blockIdx.x==0) clk[0]=t1-t0;
}

__global__ void k_fp64(double* out, int iters) {
  double a[8]; for(int i=0;i<8;i++) a[i]=threadIdx.x*1e-3+i;
  double b=1.0000001, c=1e-7;
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<8;i++) a[i]=fma(a[i],b,c);
  }
  double s=0; for(int i=0;i<8;i++) s+=a[i];
  if(s==1.2345) out[0]=s;
}

__global__ void k_ldg(const int4* __restrict__ in, size_t n16, int4* out) {
  int4 acc = make_int4(0,0,0,0);
  size_t stride = (size_t)gridDim.x*blockDim.x;
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i < n16; i += stride*4) {
    int4 v[4];
#pragma unroll
    for(int u=0;u<4;u++){ size_t j=i+u*stride; if(j<n16) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3},[%4];" : "=r"(v[u].x),"=r"(v[u].y),"=r"(v[u].z),"=r"(v[u].w) : "l"(in+j)); else v[u]=make_int4(0,0,0,0);}
#pragma unroll
    for(int u=0;u<4;u++){acc.x^=v[u].x;acc.y^=v[u].y;acc.z^=v[u].z;acc.w^=v[u].w;}
  }
  if(acc.x==0x7fffffff) out[0]=acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt){ asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes){ asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b){ asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity){
  asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" :: "r"(smem_u32(b)), "r"(parity) : "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b){
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory"); }

template<int STAGES, int CHUNK>
__global__ void __launch_bounds__(288,1) k_bulk(const uint8_t* in, size_t bytes, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + STAGES*CHUNK);
  uint64_t* empty = full + STAGES;
  int warp = threadIdx.x/32, lane=threadIdx.x%32;
  if(threadIdx.x==0){ for(int s=0;s<STAGES;s++){ mbar_init(&full[s],1); mbar_init(&empty[s],8);} asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  size_t nchunks = bytes / CHUNK;
  size_t per = (nchunks + gridDim.x - 1)/gridDim.x;
  size_t c0 = blockIdx.x*per, c1 = min(nchunks, c0+per);
  if (warp == 8) {
    if (lane==0) {
      int s=0; uint32_t ph=0;
      for(size_t c=c0;c<c1;c++){
        mbar_wait(&empty[s], ph^1);
        mbar_expect_tx(&full[s], CHUNK);
        bulk_g2s(sm + s*CHUNK, in + c*CHUNK, CHUNK, &full[s]);
        if(++s==STAGES){s=0;ph^=1;}
      }
    }
  } else {
    int s=0; uint32_t ph=0; uint32_t acc=0;
    for(size_t c=c0;c<c1;c++){
      mbar_wait(&full[s], ph);
      const uint4* p = (const uint4*)(sm + s*CHUNK) + warp*32*(CHUNK/16/256) ;
      for(int i=0;i<CHUNK/16/256;i++){ uint4 v = p[i*32+lane]; acc ^= v.x^v.w; }
      __syncwarp();
      if(lane==0) mbar_arrive(&empty[s]);
      if(++s==STAGES){s=0;ph^=1;}
    }
    if(acc==0x12345u) out[0]=acc;
  }
}

int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  int sms=pr.multiProcessorCount; printf("GPU %s SMs %d L2 %d MB smemOptin %zu\n", pr.name, sms, pr.l2CacheSize>>20, pr.sharedMemPerBlockOptin);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  float* fo; long long* clk; CK(cudaMalloc(&fo, 1<<20)); CK(cudaMalloc(&clk, 64));
  // mma.sync rate
  for (int wpb : {4, 8, 16}) {
    int iters=4000; k_mma<<<sms*2, 32*wpb>>>(fo, 10, clk); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_mma<<<sms*2, 32*wpb>>>(fo, iters, clk); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); long long c; cudaMemcpy(&c,clk,8,cudaMemcpyDeviceToHost);
    double fma = (double)sms*2*wpb*iters*8*2048.0;
    printf("mma.sync m16n8k16 f32acc: warps/SM %d: %.1f TFLOP/s  (%.1f FMA/clk/SM at clk from clock64: %.0f MHz)\n", 2*wpb, 2*fma/ms/1e9, fma/sms/(double)c, (double)c/(ms*1e3));
  }
  // dequant ALU
  { int iters=20000; k_deq<<<sms*4,256>>>((uint32_t*)fo,10,clk); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_deq<<<sms*4,256>>>((uint32_t*)fo,iters,clk); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); long long c; cudaMemcpy(&c,clk,8,cudaMemcpyDeviceToHost);
    double pairs=(double)sms*4*256*iters*8; printf("dequant lop3+hsub2: %.2f Tpairs/s  (%.2f warp-pairs/clk/SM)\n", pairs/ms/1e9, pairs/32/sms/(double)c); }
  // fp64
  { int iters=20000; k_fp64<<<sms*4,256>>>((double*)fo,10); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_fp64<<<sms*4,256>>>((double*)fo,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("fp64 FMA: %.2f TFLOP/s\n", (double)sms*4*256*iters*8*2/ms/1e9); }
  // streaming reads
  size_t bytes = (size_t)2<<30; uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  for (int rep=0; rep<2; rep++) {
    k_ldg<<<sms*8,256>>>((const int4*)buf, bytes/16, (int4*)fo); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_ldg<<<sms*8,256>>>((const int4*)buf, bytes/16, (int4*)fo); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("LDG.128 stream read: %.0f GB/s\n", bytes/ms/1e6);
  }
  {
    const int ST=4, CH=32768; size_t sm = ST*CH + 64;
    CK(cudaFuncSetAttribute(k_bulk<ST,CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (int rep=0;rep<2;rep++){
      k_bulk<ST,CH><<<sms,288,sm>>>(buf, bytes, (uint32_t*)fo); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); k_bulk<ST,CH><<<sms,288,sm>>>(buf, bytes, (uint32_t*)fo); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms,e0,e1); printf("bulk-copy ring 4x32KB, 1 CTA/SM: %.0f GB/s\n", bytes/ms/1e6);
    }
    const int ST2=6, CH2=16384; size_t sm2 = ST2*CH2+128;
    CK(cudaFuncSetAttribute(k_bulk<ST2,CH2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    for (int rep=0;rep<2;rep++){
      k_bulk<ST2,CH2><<<sms,288,sm2>>>(buf, bytes, (uint32_t*)fo); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); k_bulk<ST2,CH2><<<sms,288,sm2>>>(buf, bytes, (uint32_t*)fo); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms,e0,e1); printf("bulk-copy ring 6x16KB, 1 CTA/SM: %.0f GB/s\n", bytes/ms/1e6);
    }
    // 108 MB (the C5 decode size) — small-transfer efficiency
    size_t small = (size_t)108<<20;
    for (int rep=0;rep<3;rep++){
      cudaEventRecord(e0); k_bulk<ST,CH><<<sms,288,sm>>>(buf + (rep%2)*(size_t)(1<<30), small, (uint32_t*)fo); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms,e0,e1); printf("bulk-copy 108MB: %.1f us = %.0f GB/s\n", ms*1e3, small/ms/1e6);
    }
  }
  CK(cudaGetLastError());
  printf("done\n");
  return 0;
}
