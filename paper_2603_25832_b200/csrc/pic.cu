// pic.cu — particle push, charge/current deposit + field update, Poisson init, moments.
//
// Replaces interpolate_fields (ref: pic.py:61-74), lorentz_push (pic.py:77-88),
// advance_positions (pic.py:91-93) with wrap_position (state.py:14-27), deposit
// (pic.py:43-58), maxwell_step (pic.py:96-110), vpl_field_step (pic.py:113-115),
// poisson_solve (pic.py:118-134) and the reductions of compute_diagnostics
// (diagnostics.py:20-35) / ParticleEnsemble.validate (state.py:46-53).
//
// push: one fused streaming pass over pid-order SoA planes (read x, v; write x, v:
//       16 B + 16 B per particle at dv = 3), fields read through L1 (M <= 32768 doubles).
// deposit: from the cell-sorted records; CTA (cell c, chunk k) sums its particles' hat
//       weights into the 3 nodes {c-1, c, c+1} in float64 registers (a particle in cell c
//       only touches those), fixed-order block reduction -> partials; a single CTA then sums
//       each node's partials in a fixed order and applies the field step: deterministic,
//       no atomics (the reference uses np.bincount).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace spic {

constexpr int kDepThreads = 256;

// one particle of the fused interpolate + Lorentz + advance + wrap
__device__ __forceinline__ void push_one(float& xi, float& v0, float& v1,
                                         const double* __restrict__ E1,
                                         const double* __restrict__ E2,
                                         const double* __restrict__ B3, int M, float ie, float dt,
                                         double Ld, bool& badx, bool& badv) {
  // hat weights (ref: pic.py:33-40): g = x/eta - 1/2, i0 = floor(g) mod M, i1 = i0 + 1
  const float g = fmaf(xi, ie, -0.5f);
  const float fl = floorf(g);
  const float f1 = g - fl, f0 = 1.f - f1;
  int i0 = (int)fl;
  i0 = i0 < 0 ? i0 + M : (i0 >= M ? i0 - M : i0);
  const int i1 = i0 + 1 == M ? 0 : i0 + 1;
  const float e1 = f0 * (float)__ldg(E1 + i0) + f1 * (float)__ldg(E1 + i1);
  const float e2 = f0 * (float)__ldg(E2 + i0) + f1 * (float)__ldg(E2 + i1);
  const float b3 = f0 * (float)__ldg(B3 + i0) + f1 * (float)__ldg(B3 + i1);
  // Lorentz (ref: pic.py:77-88): dv = (E1 + v2 B3, E2 - v1 B3, 0)
  const float v0n = fmaf(dt, fmaf(v1, b3, e1), v0);
  const float v1n = fmaf(dt, fmaf(-v0, b3, e2), v1);
  v0 = v0n;
  v1 = v1n;
  badv |= !(isfinite(v0n) && isfinite(v1n));
  // advance + wrap (ref: pic.py:91-93, state.py:14-27), the wrap in float64
  const float xn = fmaf(dt, v0n, xi);
  if (!isfinite(xn)) {  // the position keeps its old value; the flag raises the error
    badx = true;
    return;
  }
  double xd = (double)xn;
  if (xd < 0.0) xd += Ld; else if (xd >= Ld) xd -= Ld;
  if (xd < 0.0 || xd >= Ld) xd -= Ld * floor(xd / Ld);
  float xo = (float)xd;
  if ((double)xo >= Ld || xo < 0.f) xo = 0.f;  // values rounding onto L fold to 0
  xi = xo;
}

// Streaming pass over the pid-order planes x, v0, v1 (v2 is untouched by the Lorentz step
// with B = (0, 0, B3)): 24 B moved per particle. VEC: four particles per thread through
// 16-B loads/stores (more bytes in flight per thread), planes 16-B aligned.
template <bool VEC>
__global__ void __launch_bounds__(256) k_push(float* __restrict__ x, float* __restrict__ v,
                                              int64_t ldv, int64_t n, const double* __restrict__ E1,
                                              const double* __restrict__ E2,
                                              const double* __restrict__ B3, int M, float ie,
                                              float dt, double Ld, int32_t* flags) {
  bool badx = false, badv = false;
  if (VEC) {
    float4* __restrict__ x4 = reinterpret_cast<float4*>(x);
    float4* __restrict__ a4 = reinterpret_cast<float4*>(v);
    float4* __restrict__ b4 = reinterpret_cast<float4*>(v + ldv);
    const int64_t n4 = n >> 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
      float4 X = x4[i], A = a4[i], B = b4[i];
      push_one(X.x, A.x, B.x, E1, E2, B3, M, ie, dt, Ld, badx, badv);
      push_one(X.y, A.y, B.y, E1, E2, B3, M, ie, dt, Ld, badx, badv);
      push_one(X.z, A.z, B.z, E1, E2, B3, M, ie, dt, Ld, badx, badv);
      push_one(X.w, A.w, B.w, E1, E2, B3, M, ie, dt, Ld, badx, badv);
      x4[i] = X;
      a4[i] = A;
      b4[i] = B;
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      float xi = x[i], v0 = v[i], v1 = v[ldv + i];
      push_one(xi, v0, v1, E1, E2, B3, M, ie, dt, Ld, badx, badv);
      x[i] = xi;
      v[i] = v0;
      v[ldv + i] = v1;
    }
  }
  if (badx) raise_flag(flags, SPIC_FLAG_NONFINITE_X);
  if (badv) raise_flag(flags, SPIC_FLAG_NONFINITE_V);
}

// partials[(c*CH + k)*12 + slot*4 + q], q = (rho, J0, J1, J2), slot s -> node c + s - 1
template <int DV>
__global__ void __launch_bounds__(kDepThreads) k_deposit_partials(
    const float4* __restrict__ xv, const float4* __restrict__ sw,
    const int32_t* __restrict__ cell_start, int M, int CH, double eta, float uniform_w,
    double* __restrict__ partials) {
  __shared__ double red[(kDepThreads / 32) * 12];
  const int c = blockIdx.x / CH, k = blockIdx.x % CH;
  const int cs = cell_start[c], cnt = cell_start[c + 1] - cs;
  const int p0 = cs + (int)(((long long)cnt * k) / CH);
  const int p1 = cs + (int)(((long long)cnt * (k + 1)) / CH);
  double a[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) a[q] = 0.0;
  constexpr int U = 4;  // records loaded ahead of their (float64) arithmetic
  for (int pb = p0 + threadIdx.x; pb < p1; pb += U * blockDim.x) {
    float4 AU[U];
    float WU[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = pb + u * blockDim.x;
      AU[u] = p < p1 ? xv[p] : make_float4(0.f, 0.f, 0.f, 0.f);
      WU[u] = (p < p1 && !(uniform_w > 0.f)) ? sw[p].w : 0.f;
    }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (pb + u * (int)blockDim.x >= p1) break;
    const float4 A = AU[u];
    const double wv = uniform_w > 0.f ? (double)uniform_w : (double)WU[u];
    const double g = (double)A.x / eta - 0.5;
    const double fl = floor(g);
    const double f = g - fl;
    int s0 = (int)((long long)fl - c + 1);
    s0 = s0 < 0 ? 0 : (s0 > 1 ? 1 : s0);
    if (M == 1) s0 = 0;
    const double w0 = wv * (1.0 - f), w1 = wv * f;
    const double q[4] = {1.0, (double)A.y, (double)A.z, (double)A.w};
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double ws = (s == s0 ? w0 : 0.0) + (s == s0 + 1 ? w1 : 0.0);
#pragma unroll
      for (int j = 0; j < 1 + DV; ++j) a[s * 4 + j] = fma(ws, q[j], a[s * 4 + j]);
    }
  }
  }
  block_sum<12>(a, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < 12; ++q) partials[(size_t)blockIdx.x * 12 + q] = a[q];
}

// Single CTA: node sums (fixed order) -> rho, J; field step; field energies.
__device__ void field_update(double* E1, double* E2, double* B3, const double* J, int M,
                             double eta, double dt, int mode, double* diag_out, int32_t* flags,
                             double* red) {
  if (mode == 1 || mode == 2)
    for (int j = threadIdx.x; j < M; j += blockDim.x) E1[j] -= dt * J[j];
  if (mode == 2) {
    const double two_eta = 2.0 * eta;
    __syncthreads();
    // E2 -= dt ((B3_{j+1} - B3_{j-1}) / 2eta + J2), then B3 with the fresh E2
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      const double dB = (B3[(j + 1) % M] - B3[(j - 1 + M) % M]) / two_eta;
      E2[j] -= dt * (dB + J[M + j]);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      const double dE = (E2[(j + 1) % M] - E2[(j - 1 + M) % M]) / two_eta;
      B3[j] -= dt * dE;
    }
  }
  __syncthreads();
  double e[2] = {0.0, 0.0};
  bool bad = false;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    e[0] += E1[j] * E1[j] + E2[j] * E2[j];
    e[1] += B3[j] * B3[j];
    bad |= !(isfinite(E1[j]) && isfinite(E2[j]) && isfinite(B3[j]));
  }
  if (bad) raise_flag(flags, SPIC_FLAG_NONFINITE_FIELD);
  block_sum<2>(e, red);
  if (threadIdx.x == 0 && diag_out) {
    diag_out[0] = 0.5 * eta * e[0];
    diag_out[1] = 0.5 * eta * e[1];
    diag_out[2] = sqrt(eta * e[0]);
  }
}

__global__ void __launch_bounds__(1024) k_deposit_finalize(
    const double* __restrict__ partials, int M, int CH, int dv, double eta,
    double* __restrict__ rho, double* __restrict__ J, int mode, double dt, double* E1, double* E2,
    double* B3, double* diag_out, int32_t* flags) {
  __shared__ double red[32 * 2];
  const double inv_eta = 1.0 / eta;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int s = 0; s < 3; ++s) {
      const int c = ((j - s + 1) % M + M) % M;
      for (int k = 0; k < CH; ++k) {
        const double* q = partials + ((size_t)c * CH + k) * 12 + s * 4;
        for (int t = 0; t < 4; ++t) acc[t] += q[t];
      }
    }
    // the reference divides the summed weights by eta (ref: pic.py:52-57)
    rho[j] = acc[0] / eta;
    for (int t = 0; t < dv; ++t) J[t * M + j] = acc[1 + t] / eta;
  }
  (void)inv_eta;
  __syncthreads();
  field_update(E1, E2, B3, J, M, eta, dt, mode, diag_out, flags, red);
}

__global__ void __launch_bounds__(1024) k_field_step(double* E1, double* E2, double* B3,
                                                     const double* J, int M, double eta,
                                                     double dt, int mode, double* diag_out,
                                                     int32_t* flags) {
  __shared__ double red[32 * 2];
  field_update(E1, E2, B3, J, M, eta, dt, mode, diag_out, flags, red);
}

// Spectral Poisson (ref: pic.py:118-134) as a single-CTA float64 DFT (M <= 16384).
__global__ void __launch_bounds__(1024) k_poisson(const double* __restrict__ rho, double rho_ion,
                                                  int M, double eta, double* __restrict__ E1,
                                                  int32_t* flags) {
  extern __shared__ double sm[];
  double* src = sm;           // [M]
  double* Fr = sm + M;        // [M/2+1]
  double* Fi = Fr + M / 2 + 1;
  __shared__ double red[32];
  double tot[1] = {0.0};
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    src[j] = rho[j] - rho_ion;
    tot[0] += src[j];
  }
  block_sum<1>(tot, red);
  __shared__ int nonneutral;
  if (threadIdx.x == 0) nonneutral = fabs(tot[0] * eta) > 1e-8;
  __syncthreads();
  if (nonneutral) {
    if (threadIdx.x == 0) raise_flag(flags, SPIC_FLAG_NON_NEUTRAL);
    return;
  }
  const int K = M / 2;
  for (int k = threadIdx.x; k <= K; k += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int j = 0; j < M; ++j) {
      double s, c;
      sincospi(2.0 * (double)(((long long)j * k) % M) / (double)M, &s, &c);
      re += src[j] * c;
      im -= src[j] * s;
    }
    Fr[k] = re;
    Fi[k] = im;
  }
  __syncthreads();
  const int kmax = (M % 2 == 0) ? K - 1 : K;  // Nyquist bin dropped for even M
  const double two_pi_over_L = 2.0 * M_PI / ((double)M * eta);
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    double acc = 0.0;
    for (int k = 1; k <= kmax; ++k) {
      double s, c;
      sincospi(2.0 * (double)(((long long)j * k) % M) / (double)M, &s, &c);
      const double kp = two_pi_over_L * k;
      // E_hat = -i F / k ; Re(E_hat e^{i theta}) = (Fi cos + Fr sin) / k
      acc += (Fi[k] * c + Fr[k] * s) / kp;
    }
    E1[j] = 2.0 * acc / (double)M;
  }
}

template <int DV>
__global__ void __launch_bounds__(256) k_moments(const float* __restrict__ v, int64_t ldv,
                                                 const float* __restrict__ w, int64_t n,
                                                 float uniform_w, double* __restrict__ partials,
                                                 int32_t* flags) {
  __shared__ double red[8 * 5];
  double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // E_K, P0, P1, P2, sum w
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = uniform_w > 0.f ? (double)uniform_w : (double)w[i];
    double e = 0.0;
#pragma unroll
    for (int d = 0; d < DV; ++d) {
      const float vv = v[d * ldv + i];
      bad |= !isfinite(vv);
      e += (double)vv * (double)vv;
      a[1 + d] += wi * (double)vv;
    }
    a[0] += 0.5 * wi * e;
    a[4] += wi;
  }
  if (bad) raise_flag(flags, SPIC_FLAG_NONFINITE_V);
  block_sum<5>(a, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 5; ++k) partials[(size_t)blockIdx.x * 5 + k] = a[k];
}

__global__ void k_reduce_rows_pic(const double* __restrict__ part, int rows, int cols,
                                  double* __restrict__ out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int col = wid; col < cols; col += nw) {
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += part[(size_t)r * cols + col];
    s = warp_sum(s);
    if (lane == 0) out[col] = s;
  }
}

static int dep_chunks(int M) {
  int ch = (4 * kNumSMs + M - 1) / M;  // 4x the SM count: more CTAs only grow the finalize
  return std::max(1, std::min(ch, 1024));
}

constexpr int kMomBlocks = 2 * kNumSMs;

}  // namespace spic

using namespace spic;

extern "C" int spic_push(float* x, float* v, int64_t ldv, int64_t n, int32_t dv, const double* E1,
                         const double* E2, const double* B3, int32_t M, double eta, float dt,
                         int32_t* flags, void* stream) {
  if (n < 0 || M < 1 || !(eta > 0) || (dv != 2 && dv != 3)) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const double Ld = (double)M * eta;
  const bool vec = n % 4 == 0 && ldv % 4 == 0 && ((uintptr_t)x & 15) == 0 &&
                   ((uintptr_t)v & 15) == 0;
  const int64_t work = vec ? n / 4 : n;
  const int blocks = (int)std::min<int64_t>((work + 255) / 256, kNumSMs * 8);
  (void)dv;  // the Lorentz step leaves v2 unchanged: the same kernel serves dv = 2 and 3
  if (vec)
    k_push<true><<<blocks, 256, 0, st>>>(x, v, ldv, n, E1, E2, B3, M, (float)(1.0 / eta), dt, Ld,
                                         flags);
  else
    k_push<false><<<blocks, 256, 0, st>>>(x, v, ldv, n, E1, E2, B3, M, (float)(1.0 / eta), dt, Ld,
                                          flags);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" size_t spic_deposit_scratch_bytes(int32_t M, int32_t dv) {
  (void)dv;
  return sizeof(double) * (size_t)M * dep_chunks(M) * 12 + 64;
}

extern "C" int spic_deposit_field(const float* xv, const float* sw, int64_t n, int32_t dv,
                                  const int32_t* cell_start, int32_t M, double eta,
                                  float uniform_w, double* rho, double* J, int32_t field_mode,
                                  double dt, double* E1, double* E2, double* B3, double* diag_out,
                                  int32_t* flags, void* scratch, size_t scratch_bytes,
                                  void* stream) {
  if (n < 0 || M < 1 || !(eta > 0) || (dv != 2 && dv != 3) || field_mode < 0 || field_mode > 2)
    return SPIC_ERR_ARG;
  if (scratch_bytes < spic_deposit_scratch_bytes(M, dv)) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  const int CH = dep_chunks(M);
  double* part = (double*)scratch;
  if (dv == 3)
    k_deposit_partials<3><<<M * CH, kDepThreads, 0, st>>>((const float4*)xv, (const float4*)sw,
                                                          cell_start, M, CH, eta, uniform_w, part);
  else
    k_deposit_partials<2><<<M * CH, kDepThreads, 0, st>>>((const float4*)xv, (const float4*)sw,
                                                          cell_start, M, CH, eta, uniform_w, part);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  k_deposit_finalize<<<1, 1024, 0, st>>>(part, M, CH, dv, eta, rho, J, field_mode, dt, E1, E2, B3,
                                         diag_out, flags); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_field_step(double* E1, double* E2, double* B3, const double* J, int32_t M,
                               double eta, double dt, int32_t field_mode, double* diag_out,
                               int32_t* flags, void* stream) {
  if (M < 1 || field_mode < 0 || field_mode > 2) return SPIC_ERR_ARG;
  k_field_step<<<1, 1024, 0, (cudaStream_t)stream>>>(E1, E2, B3, J, M, eta, dt, field_mode,
                                                     diag_out, flags); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_poisson(const double* rho, double rho_ion, int32_t M, double eta, double* E1,
                            int32_t* flags, void* stream) {
  if (M < 1 || !(eta > 0)) return SPIC_ERR_ARG;
  if (M > 16384) return SPIC_ERR_UNSUPPORTED;
  size_t smem = sizeof(double) * ((size_t)M + 2 * (M / 2 + 1));
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_poisson, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_poisson<<<1, 1024, smem, (cudaStream_t)stream>>>(rho, rho_ion, M, eta, E1, flags); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" size_t spic_moments_scratch_bytes(int64_t n) {
  (void)n;
  return sizeof(double) * kMomBlocks * 5 + 64;
}

extern "C" int spic_moments(const float* v, int64_t ldv, const float* w, int64_t n, int32_t dv,
                            float uniform_w, double* out, int32_t* flags, void* scratch,
                            size_t scratch_bytes, void* stream) {
  if (n < 0 || (dv != 2 && dv != 3)) return SPIC_ERR_ARG;
  if (scratch_bytes < spic_moments_scratch_bytes(n)) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)scratch;
  if (dv == 3)
    k_moments<3><<<kMomBlocks, 256, 0, st>>>(v, ldv, w, n, uniform_w, part, flags);
  else
    k_moments<2><<<kMomBlocks, 256, 0, st>>>(v, ldv, w, n, uniform_w, part, flags);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  k_reduce_rows_pic<<<1, 256, 0, st>>>(part, kMomBlocks, 5, out); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

// ---- unfused operator forms (API parity with interpolate_fields / lorentz_push) ----------
namespace spic {
template <int DV>
__global__ void k_interpolate(const float* __restrict__ x, int64_t n, const double* __restrict__ E1,
                              const double* __restrict__ E2, const double* __restrict__ B3, int M,
                              float ie, float* __restrict__ Ep, int64_t lde,
                              float* __restrict__ Bp, int64_t ldb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float g = fmaf(x[i], ie, -0.5f);
    const float fl = floorf(g);
    const float f1 = g - fl, f0 = 1.f - f1;
    int i0 = (int)fl;
    i0 = i0 < 0 ? i0 + M : (i0 >= M ? i0 - M : i0);
    const int i1 = i0 + 1 == M ? 0 : i0 + 1;
    Ep[i] = f0 * (float)E1[i0] + f1 * (float)E1[i1];
    Ep[lde + i] = f0 * (float)E2[i0] + f1 * (float)E2[i1];
    if (DV == 3) Ep[2 * lde + i] = 0.f;
    Bp[i] = 0.f;
    Bp[ldb + i] = 0.f;
    Bp[2 * ldb + i] = f0 * (float)B3[i0] + f1 * (float)B3[i1];
  }
}

__global__ void k_lorentz(float* __restrict__ v, int64_t ldv, int64_t n, int dv,
                          const float* __restrict__ Ep, int64_t lde, const float* __restrict__ Bp,
                          int64_t ldb, float dt, int32_t* flags) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float b3 = Bp[2 * ldb + i];
    const float v0 = v[i], v1 = v[ldv + i];
    const float a0 = Ep[i] + v1 * b3, a1 = Ep[lde + i] - v0 * b3;
    v[i] = fmaf(dt, a0, v0);
    v[ldv + i] = fmaf(dt, a1, v1);
    if (dv == 3) v[2 * ldv + i] = fmaf(dt, Ep[2 * lde + i], v[2 * ldv + i]);
    bad |= !(isfinite(v[i]) && isfinite(v[ldv + i]));
  }
  if (bad) raise_flag(flags, SPIC_FLAG_NONFINITE_V);
}
}  // namespace spic

extern "C" int spic_interpolate(const float* x, int64_t n, int32_t dv, const double* E1,
                                const double* E2, const double* B3, int32_t M, double eta,
                                float* Ep, int64_t lde, float* Bp, int64_t ldb, void* stream) {
  if (n < 0 || M < 1 || (dv != 2 && dv != 3)) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  if (dv == 3)
    k_interpolate<3><<<blocks, 256, 0, (cudaStream_t)stream>>>(x, n, E1, E2, B3, M, (float)(1.0 / eta),
                                                               Ep, lde, Bp, ldb);
  else
    k_interpolate<2><<<blocks, 256, 0, (cudaStream_t)stream>>>(x, n, E1, E2, B3, M, (float)(1.0 / eta),
                                                               Ep, lde, Bp, ldb);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_lorentz(float* v, int64_t ldv, int64_t n, int32_t dv, const float* Ep,
                            int64_t lde, const float* Bp, int64_t ldb, float dt, int32_t* flags,
                            void* stream) {
  if (n < 0 || (dv != 2 && dv != 3)) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  k_lorentz<<<blocks, 256, 0, (cudaStream_t)stream>>>(v, ldv, n, dv, Ep, lde, Bp, ldb, dt, flags);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}
