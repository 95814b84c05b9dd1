// Issue-rate microbenchmark for instruction MIXES on sm_100a (B200): how many
// lane-instructions per SM clock a stream of k1 DPX VIADDMNMX.S16x2 and k2
// other instructions (IMAD, IADD3, FFMA, PRMT, LOP3, SEL, VIMNMX3, ...)
// sustains, i.e. whether those instructions share throughput with the DPX
// recurrence.  32 warps per SM, 12 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mixpeak mixpeak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define CH 12

template <int OTHER>
__device__ __forceinline__ uint32_t other(uint32_t a, uint32_t b, uint32_t y0, uint32_t y1) {
  if constexpr (OTHER == 0) {  // IMAD
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(y0), "r"(b));
    return d;
  }
  if constexpr (OTHER == 1) {  // IADD3
    uint32_t d;
    asm volatile("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(y0));
    return d;
  }
  if constexpr (OTHER == 2) return __float_as_uint(fmaf(__uint_as_float(a), __uint_as_float(y0), __uint_as_float(b)));  // FFMA
  if constexpr (OTHER == 3) return __byte_perm(a, b, y1);  // PRMT
  if constexpr (OTHER == 4) return (a & y0) ^ b;           // LOP3
  if constexpr (OTHER == 5) return __vimax3_s16x2(a, b, y0);  // VIMNMX3.S16x2
  if constexpr (OTHER == 6) return __viaddmax_s16x2(a, y0, b);  // another DPX
  if constexpr (OTHER == 7) {  // IMAD.SHL-like (mul by power of two)
    uint32_t d;
    asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(y1));
    return d;
  }
  return a;
}

// per step: K1 DPX ops and K2 "other" ops over CH chains
template <int K1, int K2, int OTHER>
__global__ void __launch_bounds__(1024, 1) bench(const uint32_t* in, uint32_t* out, long long* cyc) {
  uint32_t x[CH];
  const uint32_t y0 = in[0], y1 = in[1];
#pragma unroll
  for (int k = 0; k < CH; ++k) x[k] = in[2 + k] + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      uint32_t a = x[k];
      const uint32_t b = x[(k + 1) % CH];
#pragma unroll
      for (int u = 0; u < K1; ++u) a = __viaddmax_s16x2(a, y0, b + 0 * u);
#pragma unroll
      for (int u = 0; u < K2; ++u) a = other<OTHER>(a, b, y0, y1);
      x[k] = a;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) acc ^= x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K1, int K2, int OTHER>
void run(const char* name, int nsm, uint32_t* din, uint32_t* dout, long long* dcyc) {
  bench<K1, K2, OTHER><<<nsm, 1024>>>(din, dout, dcyc);
  bench<K1, K2, OTHER><<<nsm, 1024>>>(din, dout, dcyc);
  cudaDeviceSynchronize();
  long long* hc = new long long[nsm];
  cudaMemcpy(hc, dcyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < nsm; ++i) mean += double(hc[i]);
  mean /= nsm;
  delete[] hc;
  const int k2i = (OTHER == 1) ? 2 * K2 : K2;  // IADD3 form emits two adds (may fuse to one IADD3)
  const double lanes = 1024.0 * ITERS * CH;
  printf("{\"mix\": \"%s\", \"dpx\": %d, \"other\": %d, \"dpx_lane_per_clk\": %.2f, \"other_lane_per_clk\": %.2f, \"cycles_per_warp_step\": %.3f}\n",
         name, K1, K2, lanes * K1 / mean, lanes * k2i / mean, mean / (ITERS * CH) / 1.0 * 4 / 32);
  (void)k2i;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t hin[16];
  for (int i = 0; i < 16; ++i) hin[i] = 0x00030005u * (i + 1);
  hin[1] = 0x5140u;
  uint32_t *din, *dout;
  long long* dcyc;
  cudaMalloc(&din, sizeof(hin));
  cudaMalloc(&dout, sizeof(uint32_t) * nsm * 1024);
  cudaMalloc(&dcyc, sizeof(long long) * nsm);
  cudaMemcpy(din, hin, sizeof(hin), cudaMemcpyHostToDevice);
  run<4, 0, 0>("dpx only", nsm, din, dout, dcyc);
  run<0, 4, 0>("imad only", nsm, din, dout, dcyc);
  run<0, 4, 2>("ffma only", nsm, din, dout, dcyc);
  run<0, 2, 1>("iadd3 only", nsm, din, dout, dcyc);
  run<4, 4, 0>("dpx+imad 1:1", nsm, din, dout, dcyc);
  run<5, 2, 0>("dpx+imad 5:2", nsm, din, dout, dcyc);
  run<4, 4, 2>("dpx+ffma 1:1", nsm, din, dout, dcyc);
  run<4, 2, 1>("dpx+iadd3 (2 adds)", nsm, din, dout, dcyc);
  run<4, 4, 3>("dpx+prmt 1:1", nsm, din, dout, dcyc);
  run<4, 4, 4>("dpx+lop3 1:1", nsm, din, dout, dcyc);
  run<4, 4, 5>("dpx+vimnmx3 1:1", nsm, din, dout, dcyc);
  run<4, 4, 7>("dpx+imul 1:1", nsm, din, dout, dcyc);
  return 0;
}
