// Microbenchmark: cycles per tcgen05.mma (kind::f16, bf16 in, f32 accumulate, M = 128,
// cta_group::1, both operands in shared memory) as a function of N, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_rate tools/umma_rate.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2603_25832_b200/csrc/pairs.cuh"
#include "../paper_2603_25832_b200/csrc/umma.cuh"

using namespace spic;

template <int N, bool AMN = false, bool BMN = false>
__global__ void __launch_bounds__(128, 1) k_rate(int reps, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
  uint8_t* base = smem_raw + ((1024u - (a0 & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 4 * 32768 / 4; i += 128) ((uint32_t*)base)[i] = 0x3f803f80u;
  if (threadIdx.x < 32) umma::tmem_alloc(&tslot, 512);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tslot, sa = (uint32_t)__cvta_generic_to_shared(base), sb = sa + 32768;
  constexpr uint32_t id = umma::idesc_bf16(AMN ? 1 : 0, BMN ? 1 : 0, N);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        umma::mma(tm, AMN ? umma::desc_mn(sa, ks) : umma::desc_k(sa, ks),
                  BMN ? umma::desc_mn(sb, ks, 2 * 32768) : umma::desc_k(sb, ks, 2 * 32768), id,
                  (r | ks) ? 1u : 0u);
    umma::commit(&bar);
    umma::wait_mma(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  umma::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_free(tm, 512);
}

template <int N, bool AMN = false, bool BMN = false>
void run(int reps) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 4 * 32768 + 1024;
  cudaFuncSetAttribute(k_rate<N, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_rate<N, AMN, BMN><<<148, 128, smem>>>(reps, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<N, AMN, BMN><<<148, 128, smem>>>(reps, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double mmas = 8.0 * reps;
  const double flop = 2.0 * 128 * N * 16 * mmas * 148;
  printf("{\"N\": %d, \"A\": \"%s\", \"B\": \"%s\", \"cycles_per_mma\": %.2f, \"tflops_bf16\": %.1f, \"err\": \"%s\"}\n", N,
         AMN ? "MN" : "K", BMN ? "MN" : "K", h[0] / mmas, flop / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<32>(4000);
  run<48>(4000);
  run<64>(4000);
  run<128>(4000);
  run<256>(2000);
  run<48, true, false>(4000);
  run<128, true, false>(4000);
  run<48, false, true>(4000);
  run<128, true, true>(4000);
  return 0;
}
