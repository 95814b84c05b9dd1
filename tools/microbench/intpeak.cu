// INT32 / DPX issue-rate microbenchmark for sm_100a (B200).
// Measures lane-ops per SM clock for the integer instructions the 3-way DP
// recurrence uses (VIADDMNMX, VIMNMX3, IADD3, IMNMX, IMAD, PRMT, LOP3, and the
// packed .S16x2 forms), one full wave of CTAs, 8 independent chains per thread.
// Output: one JSON object per op on stdout.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o intpeak intpeak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 8

template <int OP>
__device__ __forceinline__ void step(uint32_t (&x)[CHAINS], uint32_t y0, uint32_t y1) {
  uint32_t n[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) {
    const uint32_t a = x[k], b = x[(k + 1) % CHAINS], c = x[(k + 2) % CHAINS];
    if constexpr (OP == 0) n[k] = a + y0 + b;                                   // IADD3
    if constexpr (OP == 1) n[k] = (uint32_t)max((int)a, (int)b);                // IMNMX
    if constexpr (OP == 2) n[k] = (uint32_t)__viaddmax_s32((int)a, (int)y0, (int)b);  // VIADDMNMX
    if constexpr (OP == 3) n[k] = (uint32_t)__vimax3_s32((int)a, (int)b, (int)c);    // VIMNMX3
    if constexpr (OP == 4) n[k] = __viaddmax_s16x2(a, y0, b);                   // VIADDMNMX.S16x2
    if constexpr (OP == 5) n[k] = __vimax3_s16x2(a, b, c);                      // VIMNMX3.S16x2
    if constexpr (OP == 6) n[k] = a * y0 + b;                                   // IMAD
    if constexpr (OP == 7) n[k] = (a & y0) ^ b;                                 // LOP3
    if constexpr (OP == 8) n[k] = __byte_perm(a, b, y1);                        // PRMT
    if constexpr (OP == 9) n[k] = (k & 1) ? a * y0 + b : (uint32_t)__viaddmax_s32((int)a, (int)y0, (int)b);  // mix DPX+IMAD
  }
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) x[k] = n[k];
}

template <int OP>
__global__ void __launch_bounds__(1024, 1) bench(const uint32_t* in, uint32_t* out, long long* cyc) {
  uint32_t x[CHAINS];
  const uint32_t y0 = in[0], y1 = in[1];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) x[k] = in[2 + k] + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) step<OP>(x, y0, y1);
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) acc ^= x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int ops_per_step, uint32_t* din, uint32_t* dout, long long* dcyc, int nsm) {
  const int threads = 1024;
  bench<OP><<<nsm, threads>>>(din, dout, dcyc);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<nsm, threads>>>(din, dout, dcyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* hc = new long long[nsm];
  cudaMemcpy(hc, dcyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < nsm; ++i) mean += double(hc[i]);
  mean /= nsm;
  delete[] hc;
  const double lane_ops = double(threads) * ITERS * 4 * CHAINS * ops_per_step / CHAINS;
  const double per_clk = lane_ops / mean;            // instructions*lanes per SM clock
  const double clk_ghz = mean / (ms * 1e6);          // implied SM clock
  const double chip = double(nsm) * lane_ops / (ms * 1e-3);
  printf("{\"op\": \"%s\", \"lane_instr_per_clk_per_sm\": %.2f, \"implied_sm_ghz\": %.3f, "
         "\"chip_lane_instr_per_s\": %.4e, \"ms\": %.3f}\n",
         name, per_clk, clk_ghz, chip, ms);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t hin[16];
  for (int i = 0; i < 16; ++i) hin[i] = 0x00030005u * (i + 1);
  hin[1] = 0x5140u;  // PRMT selector
  uint32_t *din, *dout;
  long long* dcyc;
  cudaMalloc(&din, sizeof(hin));
  cudaMalloc(&dout, sizeof(uint32_t) * nsm * 1024);
  cudaMalloc(&dcyc, sizeof(long long) * nsm);
  cudaMemcpy(din, hin, sizeof(hin), cudaMemcpyHostToDevice);
  printf("{\"sms\": %d}\n", nsm);
  run<0>("IADD3", CHAINS, din, dout, dcyc, nsm);
  run<1>("IMNMX", CHAINS, din, dout, dcyc, nsm);
  run<2>("VIADDMNMX", CHAINS, din, dout, dcyc, nsm);
  run<3>("VIMNMX3", CHAINS, din, dout, dcyc, nsm);
  run<4>("VIADDMNMX.S16x2", CHAINS, din, dout, dcyc, nsm);
  run<5>("VIMNMX3.S16x2", CHAINS, din, dout, dcyc, nsm);
  run<6>("IMAD", CHAINS, din, dout, dcyc, nsm);
  run<7>("LOP3", CHAINS, din, dout, dcyc, nsm);
  run<8>("PRMT", CHAINS, din, dout, dcyc, nsm);
  run<9>("VIADDMNMX+IMAD", CHAINS, din, dout, dcyc, nsm);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
