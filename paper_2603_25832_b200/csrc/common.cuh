// common.cuh — shared device helpers for the scorepic B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scorepic_b200.h"

#define SPIC_CHECK_LAUNCH()                                  \
  do {                                                       \
    cudaError_t e__ = cudaGetLastError();                    \
    if (e__ != cudaSuccess) return SPIC_ERR_CUDA - (int)e__; \
  } while (0)

namespace spic {

// host-side count of kernel launches issued by this library (bench evidence)
void count_launch();

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

// MUFU.RCP without the IEEE slow path (__frcp_rn compiles to a refinement + a CALL);
// ~1 ulp, used where the argument is >= 1 (softsign) or the result feeds float32 sums.
__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block-wide sum of NV doubles per thread; result valid in thread 0.
// `scratch` must hold (blockDim.x/32) * NV doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[wid * NV + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += scratch[w * NV + k];
      v[k] = s;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void raise_flag(int32_t* flags, int idx) {
  if (flags) atomicOr(flags + idx, 1);
}

// Grid.cell_of (ref: pic.py:27-30) in float64: min(floor(x/eta) mod M, M-1), with the
// sub-cell index floor(frac(x/eta) * S) used to order particles inside a cell.
struct CellKey {
  int cell;
  int sub;
  bool wrapped;  // floor(x/eta) was >= M (x rounds onto L): cell 0, stored as x - L
};

__device__ __forceinline__ CellKey cell_key(float xf, double eta, int M, int S) {
  double q = (double)xf / eta;
  double fl = floor(q);
  long long idx = (long long)fl;
  // positions lie in [0, L): idx in [0, M] almost always; the 64-bit modulo (a software
  // division) only for the rest. Same result as the floor-mod either way.
  long long r = idx;
  if (idx < 0 || idx >= (long long)M) {
    r = idx % (long long)M;
    if (r < 0) r += M;
  }
  CellKey k;
  k.cell = (int)r;  // already <= M-1; the reference's min(., M-1) is a no-op after mod
  k.wrapped = idx >= M;
  int sub = 0;
  if (S > 1) {
    sub = (int)((q - fl) * (double)S);
    sub = sub < 0 ? 0 : (sub >= S ? S - 1 : sub);
  }
  k.sub = sub;
  return k;
}

}  // namespace spic
