// probe.cu — FP32 CUDA-core throughput probe: the measured roofline denominator of the
// FP32-bound pair kernels (MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).
// Packed FFMA2 (fma.rn.f32x2) on independent accumulators; 2 FLOP per lane-FMA.
#include "common.cuh"

namespace spic {

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void __launch_bounds__(512) k_fp32_probe(int iters, float* out) {
  unsigned long long acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    acc[k] = ((unsigned long long)__float_as_uint(k + 0.5f) << 32) | __float_as_uint(threadIdx.x * 1e-3f);
  const unsigned long long m = ((unsigned long long)__float_as_uint(0.999f) << 32) | __float_as_uint(0.999f);
  const unsigned long long c = ((unsigned long long)__float_as_uint(1e-3f) << 32) | __float_as_uint(1e-3f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = ffma2(acc[k], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += __uint_as_float((unsigned)acc[k]);
  if (s == 1234.5f) out[blockIdx.x] = s;
}

}  // namespace spic

// Launches blocks x 512 threads x iters x 16 lane-FMAs; returns the FLOP count in *flop.
extern "C" int spic_fp32_probe(int32_t iters, int32_t blocks, float* out, double* flop,
                               void* stream) {
  if (iters < 1 || blocks < 1) return SPIC_ERR_ARG;
  spic::k_fp32_probe<<<blocks, 512, 0, (cudaStream_t)stream>>>(iters, out);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  if (flop) *flop = 2.0 * 16.0 * (double)iters * 512.0 * (double)blocks;
  return SPIC_OK;
}
