// FP32 CUDA-core peak microbenchmark for the roofline denominator of the pair kernels.
// Measures sustained FFMA throughput (3-register form, the form the pair kernels use)
// and packed FFMA2 (fma.rn.f32x2, sm_100+) across the whole chip, with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define NACC 16

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = threadIdx.x * 1e-3f + k;
  float m = a + threadIdx.x * 1e-9f, c = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = fmaf(acc[k], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s += acc[k];
  if (s == 1234.5f) out[blockIdx.x] = s;
}

__device__ __forceinline__ unsigned long long f2_fma(unsigned long long x, unsigned long long y,
                                                     unsigned long long z) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z));
  return d;
}

__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}

__global__ void ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long acc[NACC / 2];
#pragma unroll
  for (int k = 0; k < NACC / 2; ++k) acc[k] = pack2(threadIdx.x * 1e-3f + k, k + 0.5f);
  unsigned long long m = pack2(a + threadIdx.x * 1e-9f, a), c = pack2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC / 2; ++k) acc[k] = f2_fma(acc[k], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NACC / 2; ++k)
    s += __uint_as_float((unsigned)acc[k]) + __uint_as_float((unsigned)(acc[k] >> 32));
  if (s == 1234.5f) out[blockIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  float* out;
  cudaMalloc(&out, 1 << 20);
  const int threads = 512, blocks = sms * 4, iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    double best = 0;
    for (int rep = 0; rep < 8; ++rep) {
      cudaEventRecord(e0);
      if (variant == 0)
        ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
      else
        ffma2_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * NACC * (double)iters * threads * blocks;
      double tf = flop / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf("{\"kernel\": \"%s\", \"fp32_tflops\": %.2f, \"sms\": %d}\n",
           variant == 0 ? "ffma" : "ffma2_f32x2", best, sms);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
