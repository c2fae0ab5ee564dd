// Microbenchmark of the decode consumer's per-window compute (do_window / do_rest of
// paper_2605_02262_b200/csrc/decode.cu) on shared-memory-resident records: cycles per
// window for a given number of warps per SM, with no producer, ring or epilogue.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I include tools/ubench_window.cu -o tools/ubench_window
#include "../paper_2605_02262_b200/csrc/decode.cu"
#include <cstdio>

using namespace wq;
// (the launchers of decode.cu are not used here)
int wq::device_sm_count() { return 148; }
cudaError_t wq::launch_decode_tc(const DecodeArgs &, int, cudaStream_t) { return cudaErrorNotSupported; }

template <int BITS, int TP>
__global__ void __launch_bounds__(384, 1) kbench(int iters, unsigned long long *cyc, float *sink) {
  constexpr int D = 128, S = 32, KT = D / 16;
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int REC = BITS == 16 ? 4 * S * D : S * D * BITS / 4 + 4 * D + 4 * S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // records: small codes, unit scales, zero offsets (finite scores)
  for (int i = tid; i < 4 * REC / 4; i += blockDim.x) {
    uint32_t v = (uint32_t)(i * 2654435761u);
    reinterpret_cast<uint32_t *>(sm)[i] = BITS == 16 ? (v & 0x33ff33ffu) : v;
  }
  __syncthreads();
  if (BITS < 16) {
    for (int r = 0; r < 4; r++) {
      uint8_t *kp = sm + r * REC + 2 * (S * D * BITS / 8);
      for (int i = tid; i < (4 * D + 4 * S) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(kp)[i] = (i & 2) ? 0u : 0x1c001c00u;   // s = 2^-8, mn = 0
    }
  }
  __syncthreads();
  uint8_t *scratch = sm + 4 * REC + warp * 512;
  uint8_t *qs = sm + 4 * REC + 16 * 512;          // q fragment table [KT][32][2]
  if (warp == 0)
    for (int kt = 0; kt < KT; kt++)
      *reinterpret_cast<uint2 *>(qs + (kt * 32 + lane) * 8) = make_uint2(0x3c003c00u ^ (lane * kt), 0x38003800u);
  float o[KT][4] = {};
  WarpState st;
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = st.vb[0] = st.vb[1] = 0.f;
  const uint8_t *rec = sm + (warp & 3) * REC;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    if constexpr (TP && BITS < 16) do_window_tp<D, BITS>(rec, qs, 0.1275f, st, o, scratch, lane);
    else do_window<D, S, BITS>(rec, qs, 0.1275f, st, o, scratch, lane);
  }
  __syncwarp();
  const unsigned long long t1 = clock64();
  float acc = st.l[0] + st.vb[1];
  for (int kt = 0; kt < KT; kt++) acc += o[kt][0] + o[kt][3];
  if (acc == 12345.f) sink[0] = acc;
  if (lane == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
}

template <int BITS, int TP>
void run(int sms, unsigned long long *dc, float *ds) {
  constexpr int D = 128, S = 32;
  constexpr int REC = BITS == 16 ? 4 * S * D : S * D * BITS / 4 + 4 * D + 4 * S;
  const size_t smem = 4 * REC + 16 * 512 + 2048;
  cudaFuncSetAttribute(kbench<BITS, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 200;
  for (int nw : {1, 11}) {
    kbench<BITS, TP><<<sms, nw * 32, smem>>>(iters, dc, ds);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kbench<BITS, TP><<<sms, nw * 32, smem>>>(iters, dc, ds);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    static unsigned long long h[148 * 16];
    cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
    double mc = 0;
    for (int w = 0; w < nw; w++) mc += h[w];
    mc /= nw;
    const double win_per_us = (double)sms * nw * iters / (ms * 1e3);
    printf("tp %d bits %2d warps/SM %2d: %7.0f cycles/window/warp  %6.3f us/window/warp  %8.1f windows/us (all SMs)  "
           "-> C5 layer (25088 windows) %6.2f us\n",
           TP, BITS, nw, mc / iters, ms * 1e3 / iters, win_per_us, 25088.0 / win_per_us);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *dc;
  float *ds;
  cudaMalloc(&dc, 148 * 16 * sizeof(unsigned long long));
  cudaMalloc(&ds, 16);
  run<2, 0>(sms, dc, ds);
  run<2, 1>(sms, dc, ds);
  run<4, 0>(sms, dc, ds);
  run<4, 1>(sms, dc, ds);
  run<8, 0>(sms, dc, ds);
  run<8, 1>(sms, dc, ds);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
