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
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "pairs.cuh"

namespace spic {

constexpr int kDepThreads = 256;

// node fields (E1, E2, B3) as floats: read from the float64 grid arrays through L1, or from a
// float4-per-node copy in shared memory (one 16-B load per node instead of three 8-B gathers)
struct FieldsGlobal {
  const double* __restrict__ E1;
  const double* __restrict__ E2;
  const double* __restrict__ B3;
  __device__ __forceinline__ float4 operator()(int i) const {
    return make_float4((float)__ldg(E1 + i), (float)__ldg(E2 + i), (float)__ldg(B3 + i), 0.f);
  }
};
struct FieldsShared {
  const float4* F;
  __device__ __forceinline__ float4 operator()(int i) const { return F[i]; }
};

// one particle of the fused interpolate + Lorentz + advance + wrap
template <class Fld>
__device__ __forceinline__ void push_one(float& xi, float& v0, float& v1, const Fld& fld, int M,
                                         double ie, float dt, double Ld, bool& badx, bool& badv) {
  // hat weights (ref: pic.py:33-40): g = x/eta - 1/2, i0 = floor(g) mod M, i1 = i0 + 1; g in
  // float64 (one DFMA) so the weights keep full precision at large M (float32 g would carry
  // an absolute error of ~M * 6e-8 into f1)
  const double g = fma((double)xi, ie, -0.5);
  const double fl = floor(g);
  const float f1 = (float)(g - fl), f0 = 1.f - f1;
  int i0 = (int)fl;
  i0 = i0 < 0 ? i0 + M : (i0 >= M ? i0 - M : i0);
  const int i1 = i0 + 1 == M ? 0 : i0 + 1;
  const float4 Fa = fld(i0), Fb = fld(i1);
  const float e1 = f0 * Fa.x + f1 * Fb.x;
  const float e2 = f0 * Fa.y + f1 * Fb.y;
  const float b3 = f0 * Fa.z + f1 * Fb.z;
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
// 16-B loads/stores (more bytes in flight per thread), planes 16-B aligned. SMEM: the node
// fields staged once per CTA as float4 in shared memory (M <= kPushSmemM; particles are in pid
// order, so the per-particle node reads are scattered: three 8-B L1 gathers per node cost far
// more LSU wavefronts than one conflict-light 16-B shared load).
constexpr int kPushSmemM = 4096;
template <bool VEC, bool SMEM>
__global__ void __launch_bounds__(256) k_push(float* __restrict__ x, float* __restrict__ v,
                                              int64_t ldv, int64_t n, const double* __restrict__ E1,
                                              const double* __restrict__ E2,
                                              const double* __restrict__ B3, int M, double ie,
                                              float dt, double Ld, int32_t* flags) {
  extern __shared__ float4 s_fld[];
  bool badx = false, badv = false;
  auto body = [&](const auto& fld) {
    if (VEC) {
      float4* __restrict__ x4 = reinterpret_cast<float4*>(x);
      float4* __restrict__ a4 = reinterpret_cast<float4*>(v);
      float4* __restrict__ b4 = reinterpret_cast<float4*>(v + ldv);
      const int64_t n4 = n >> 2;
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
           i += (int64_t)gridDim.x * blockDim.x) {
        float4 X = x4[i], A = a4[i], B = b4[i];
        push_one(X.x, A.x, B.x, fld, M, ie, dt, Ld, badx, badv);
        push_one(X.y, A.y, B.y, fld, M, ie, dt, Ld, badx, badv);
        push_one(X.z, A.z, B.z, fld, M, ie, dt, Ld, badx, badv);
        push_one(X.w, A.w, B.w, fld, M, ie, dt, Ld, badx, badv);
        x4[i] = X;
        a4[i] = A;
        b4[i] = B;
      }
    } else {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
           i += (int64_t)gridDim.x * blockDim.x) {
        float xi = x[i], v0 = v[i], v1 = v[ldv + i];
        push_one(xi, v0, v1, fld, M, ie, dt, Ld, badx, badv);
        x[i] = xi;
        v[i] = v0;
        v[ldv + i] = v1;
      }
    }
  };
  if (SMEM) {
    for (int j = threadIdx.x; j < M; j += blockDim.x)
      s_fld[j] = make_float4((float)E1[j], (float)E2[j], (float)B3[j], 0.f);
    __syncthreads();
    body(FieldsShared{s_fld});
  } else {
    body(FieldsGlobal{E1, E2, B3});
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

// One record's hat weights into the 12 slot sums of its cell c (slot s -> node c + s - 1).
template <int DV>
__device__ __forceinline__ void dep_accum(double (&a)[12], const float4 A, float w, double inv_eta,
                                          double cm, int M) {
  const double wv = (double)w;  // 0 for padding: adds nothing
  const double g = fma((double)A.x, inv_eta, -0.5);
  const double fl = floor(g);
  const double w1 = wv * (g - fl), w0 = wv - w1;
  // particle in cell c: fl is c - 1 (nodes c-1, c) or c (nodes c, c+1)
  const bool hi = (M == 1) ? false : fl > cm;
  const double wm = hi ? 0.0 : w0, wc = hi ? w0 : w1, wp = hi ? w1 : 0.0;
  const double q[4] = {1.0, (double)A.y, (double)A.z, (double)A.w};
#pragma unroll
  for (int j = 0; j < 1 + DV; ++j) {
    a[j] = fma(wm, q[j], a[j]);
    a[4 + j] = fma(wc, q[j], a[4 + j]);
    a[8 + j] = fma(wp, q[j], a[8 + j]);
  }
}

// Deposit partials, v2: the same per-(cell, chunk) slot sums with a lighter float64 body —
// g = x * (1/eta) - 1/2 by one DFMA (the reference divides; the hat weights are continuous in
// g, so a 1-ulp difference moves nothing across a node), w0 = w - w1, the three node weights
// selected once per particle — and <= 64 registers so four CTAs fit per SM. Records are
// loaded U ahead; the chunk count gives >= 4 waves so the tail wave is short.
template <int DV, int U, int MINB>
__global__ void __launch_bounds__(kDepThreads, MINB) k_deposit_partials_v2(
    const float4* __restrict__ xv, const float4* __restrict__ sw,
    const int32_t* __restrict__ cell_start, int M, int CH, double inv_eta, float uniform_w,
    double* __restrict__ partials) {
  __shared__ double red[(kDepThreads / 32) * 12];
  const int c = blockIdx.x / CH, k = blockIdx.x % CH;
  const int cs = cell_start[c], cnt = cell_start[c + 1] - cs;
  const int p0 = cs + (int)(((long long)cnt * k) / CH);
  const int p1 = cs + (int)(((long long)cnt * (k + 1)) / CH);
  const bool uni = uniform_w > 0.f;
  const double cm = (double)c - 0.5;  // fl > c - 1/2 picks the node pair (c, c+1)
  double a[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) a[q] = 0.0;
  for (int pb = p0 + threadIdx.x; pb < p1; pb += U * kDepThreads) {
    float4 AU[U];
    float WU[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = pb + u * kDepThreads;
      AU[u] = p < p1 ? xv[p] : make_float4(0.f, 0.f, 0.f, 0.f);
      WU[u] = p < p1 ? (uni ? 1.f : sw[p].w) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) dep_accum<DV>(a, AU[u], WU[u], inv_eta, cm, M);
  }
  if (uni)
#pragma unroll
    for (int q = 0; q < 12; ++q) a[q] *= (double)uniform_w;
  block_sum<12>(a, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < 12; ++q) partials[(size_t)blockIdx.x * 12 + q] = a[q];
}

// Deposit partials, v4: the CTA's contiguous record range [p0, p1) of its (cell, chunk) unit
// streamed into shared memory by bulk copies (cp.async.bulk + mbarrier, nstages stages of rs
// records; the sw records alongside for per-particle weights), so each SM keeps ~190 KB of
// reads in flight independent of the float64 arithmetic; threads then take records from
// shared memory. Same slot sums and fixed reduction order as v2. (A persistent form that walks
// several units per CTA with one pipeline measured 2-3x slower: ~5 us per unit start.)
constexpr int kMaxStages = 8;
struct BulkCfg {  // records per stage, stages, CTAs per SM (SPIC_DEP_CFG="rs,stages,ctas")
  int rs, stages, ctas;
};
static BulkCfg bulk_cfg(const char* env, BulkCfg def) {
  const char* e = getenv(env);
  BulkCfg c = def;
  if (e && sscanf(e, "%d,%d,%d", &c.rs, &c.stages, &c.ctas) == 3 && c.rs % 4 == 0 && c.rs > 0 &&
      c.stages >= 1 && c.stages <= kMaxStages && c.ctas >= 1 && c.ctas <= 16)
    return c;
  return def;
}

static size_t dep_bulk_smem(int rs, int stages, bool nonuni) {
  return 128 + (size_t)stages * rs * sizeof(float4) * (nonuni ? 2 : 1) +
         kMaxStages * sizeof(uint64_t);
}

template <int DV, bool NONUNI>
__global__ void __launch_bounds__(kDepThreads) k_deposit_bulk(
    const float4* __restrict__ xv, const float4* __restrict__ sw,
    const int32_t* __restrict__ cell_start, int M, int CH, double inv_eta, float uniform_w,
    double* __restrict__ partials, int rs, int nstages) {
  extern __shared__ unsigned char s_dyn[];
  unsigned char* s_base = s_dyn + ((128u - (uint32_t)((uintptr_t)s_dyn & 127u)) & 127u);
  float4* s_x = reinterpret_cast<float4*>(s_base);                 // [stage][rs]
  float4* s_w = s_x + (size_t)nstages * rs;                        // [stage][rs] (NONUNI)
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_x + (size_t)nstages * rs * (NONUNI ? 2 : 1));
  __shared__ double red[(kDepThreads / 32) * 12];
  const int c = blockIdx.x / CH, k = blockIdx.x % CH;
  const int cs = cell_start[c], cnt = cell_start[c + 1] - cs;
  const int p0 = cs + (int)(((long long)cnt * k) / CH);
  const int p1 = cs + (int)(((long long)cnt * (k + 1)) / CH);
  const int nrec = p1 - p0, nst = (nrec + rs - 1) / rs;
  const double cm = (double)c - 0.5;
  auto issue = [&](int q) {
    const int st = q % nstages, b = q * rs, m = min(rs, nrec - b);
    const uint32_t bytes = (uint32_t)m * sizeof(float4);
    mbar_expect_tx(&s_bar[st], NONUNI ? 2 * bytes : bytes);
    bulk_g2s(s_x + (size_t)st * rs, xv + p0 + b, bytes, &s_bar[st]);
    if (NONUNI) bulk_g2s(s_w + (size_t)st * rs, sw + p0 + b, bytes, &s_bar[st]);
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < nstages; ++st) mbar_init(&s_bar[st], 1);
    fence_barrier_init();
    for (int q = 0; q < min(nst, nstages); ++q) issue(q);
  }
  __syncthreads();
  double a[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) a[q] = 0.0;
  for (int q = 0; q < nst; ++q) {
    const int st = q % nstages, m = min(rs, nrec - q * rs);
    mbar_wait(&s_bar[st], (uint32_t)((q / nstages) & 1));
    const float4* X = s_x + (size_t)st * rs;
    const float4* Wr = s_w + (size_t)st * rs;
#pragma unroll 4
    for (int i = threadIdx.x; i < m; i += kDepThreads)
      dep_accum<DV>(a, X[i], NONUNI ? Wr[i].w : 1.f, inv_eta, cm, M);
    __syncthreads();  // stage st consumed
    if (threadIdx.x == 0 && q + nstages < nst) {
      fence_proxy_async();
      issue(q + nstages);
    }
  }
  if (!NONUNI)
#pragma unroll
    for (int q = 0; q < 12; ++q) a[q] *= (double)uniform_w;
  block_sum<12>(a, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < 12; ++q) partials[(size_t)blockIdx.x * 12 + q] = a[q];
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Deposit partials, v5: v4 with a dedicated producer warp and per-stage "empty" mbarriers in
// place of the CTA-wide barrier after every stage: the 8 consumer warps release a stage as
// each finishes it (lane 0 arrives after __syncwarp), and the producer refills it as soon as
// the last one has, so no warp waits for the slowest before taking the next stage.
template <int DV, bool NONUNI>
__global__ void __launch_bounds__(kDepThreads + 32) k_deposit_bulk_ws(
    const float4* __restrict__ xv, const float4* __restrict__ sw,
    const int32_t* __restrict__ cell_start, int M, int CH, double inv_eta, float uniform_w,
    double* __restrict__ partials, int rs, int nstages) {
  extern __shared__ unsigned char s_dyn[];
  unsigned char* s_base = s_dyn + ((128u - (uint32_t)((uintptr_t)s_dyn & 127u)) & 127u);
  float4* s_x = reinterpret_cast<float4*>(s_base);
  float4* s_w = s_x + (size_t)nstages * rs;
  uint64_t* s_full = reinterpret_cast<uint64_t*>(s_x + (size_t)nstages * rs * (NONUNI ? 2 : 1));
  uint64_t* s_empty = s_full + kMaxStages;
  __shared__ double red[(kDepThreads / 32) * 12];
  constexpr int kCW = kDepThreads / 32;  // consumer warps
  const int c = blockIdx.x / CH, k = blockIdx.x % CH;
  const int cs = cell_start[c], cnt = cell_start[c + 1] - cs;
  const int p0 = cs + (int)(((long long)cnt * k) / CH);
  const int p1 = cs + (int)(((long long)cnt * (k + 1)) / CH);
  const int nrec = p1 - p0, nst = (nrec + rs - 1) / rs;
  if (threadIdx.x == 0) {
    for (int st = 0; st < nstages; ++st) {
      mbar_init(&s_full[st], 1);
      mbar_init(&s_empty[st], kCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x >= kDepThreads) {  // producer warp
    if (threadIdx.x == kDepThreads) {
      for (int q = 0; q < nst; ++q) {
        const int st = q % nstages;
        if (q >= nstages) mbar_wait(&s_empty[st], (uint32_t)(((q / nstages) - 1) & 1));
        const int b = q * rs, m = min(rs, nrec - b);
        const uint32_t bytes = (uint32_t)m * sizeof(float4);
        mbar_expect_tx(&s_full[st], NONUNI ? 2 * bytes : bytes);
        bulk_g2s(s_x + (size_t)st * rs, xv + p0 + b, bytes, &s_full[st]);
        if (NONUNI) bulk_g2s(s_w + (size_t)st * rs, sw + p0 + b, bytes, &s_full[st]);
      }
    }
  } else {
    const double cm = (double)c - 0.5;
    double a[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) a[q] = 0.0;
    for (int q = 0; q < nst; ++q) {
      const int st = q % nstages, m = min(rs, nrec - q * rs);
      mbar_wait(&s_full[st], (uint32_t)((q / nstages) & 1));
      const float4* X = s_x + (size_t)st * rs;
      const float4* Wr = s_w + (size_t)st * rs;
#pragma unroll 4
      for (int i = threadIdx.x; i < m; i += kDepThreads)
        dep_accum<DV>(a, X[i], NONUNI ? Wr[i].w : 1.f, inv_eta, cm, M);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s_empty[st]);
    }
    if (!NONUNI)
#pragma unroll
      for (int q = 0; q < 12; ++q) a[q] *= (double)uniform_w;
    // fixed-order reduction over the consumer warps (named barrier: the producer is not in it)
#pragma unroll
    for (int q = 0; q < 12; ++q) a[q] = warp_sum(a[q]);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 12; ++q) red[wid * 12 + q] = a[q];
    asm volatile("bar.sync 1, %0;" ::"n"(kDepThreads));
    if (threadIdx.x < 12) {
      double t = 0.0;
      for (int w = 0; w < kCW; ++w) t += red[w * 12 + threadIdx.x];
      partials[(size_t)blockIdx.x * 12 + threadIdx.x] = t;
    }
  }
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


static int dep_variant() {  // SPIC_DEP_VARIANT=1/2/3: register-streaming kernels, 4: bulk (A/B)
  const char* e = getenv("SPIC_DEP_VARIANT");
  return e && e[0] ? e[0] - '0' : 5;
}

// v4 (bulk copies): stage records, stages, target CTAs per SM
static BulkCfg dep_bulk_cfg(bool nonuni) {
  return bulk_cfg("SPIC_DEP_CFG", nonuni ? BulkCfg{512, 3, 4} : BulkCfg{1024, 3, 4});
}

static int dep_chunks(int M, int variant, int64_t n) {
  (void)n;
  // v1: 4x the SM count; v2/v3: >= 4 waves of their 3-4 resident CTAs per SM; v4/v5: at most
  // ctas x SMs CTAs — few long record streams: every CTA pays a pipeline fill (measured at
  // n = 2^24, M = 1024: 1024 CTAs 0.069 ms, 4096 CTAs 0.108 ms, whatever the wave fill)
  const int want = variant == 1 ? 4 * kNumSMs
                   : variant >= 4 ? dep_bulk_cfg(false).ctas * kNumSMs : 16 * kNumSMs;
  const int ch = variant >= 4 ? want / M : (want + M - 1) / M;
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
  (void)dv;  // the Lorentz step leaves v2 unchanged: the same kernel serves dv = 2 and 3
  const double ie = 1.0 / eta;
  const char* pe = getenv("SPIC_PUSH_VARIANT");  // "1": fields through L1 (A/B)
  if (M <= kPushSmemM && !(pe && pe[0] == '1')) {
    // one resident wave: every CTA stages the fields once
    auto kern = vec ? k_push<true, true> : k_push<false, true>;
    const size_t sm = sizeof(float4) * (size_t)M;
    if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, sm);
    const int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)kNumSMs * std::max(occ, 1));
    kern<<<blocks, 256, sm, st>>>(x, v, ldv, n, E1, E2, B3, M, ie, dt, Ld, flags);
  } else {
    const int blocks = (int)std::min<int64_t>((work + 255) / 256, kNumSMs * 8);
    if (vec)
      k_push<true, false><<<blocks, 256, 0, st>>>(x, v, ldv, n, E1, E2, B3, M, ie, dt, Ld, flags);
    else
      k_push<false, false><<<blocks, 256, 0, st>>>(x, v, ldv, n, E1, E2, B3, M, ie, dt, Ld, flags);
  }
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" size_t spic_deposit_scratch_bytes(int32_t M, int32_t dv) {
  (void)dv;
  // sized for any variant / configuration (at most 1024 chunks per cell)
  return sizeof(double) * (size_t)M * std::min(1024, std::max(16 * kNumSMs / M + 1, 64)) * 12 + 64;
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
  const int var = dep_variant();
  const int CH = dep_chunks(M, var, n);
  double* part = (double*)scratch;
  // v2: two records ahead, four CTAs/SM; v3: four ahead, three CTAs/SM; v4: bulk copies
  if (var == 5) {
    const bool nonuni = !(uniform_w > 0.f);
    const BulkCfg c = dep_bulk_cfg(nonuni);
    const size_t sm = dep_bulk_smem(c.rs, c.stages, nonuni) + kMaxStages * sizeof(uint64_t);
    auto kern = dv == 3 ? (nonuni ? k_deposit_bulk_ws<3, true> : k_deposit_bulk_ws<3, false>)
                        : (nonuni ? k_deposit_bulk_ws<2, true> : k_deposit_bulk_ws<2, false>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<M * CH, kDepThreads + 32, sm, st>>>((const float4*)xv, (const float4*)sw, cell_start, M,
                                               CH, 1.0 / eta, uniform_w, part, c.rs, c.stages);
  } else if (var == 4) {
    const bool nonuni = !(uniform_w > 0.f);
    const BulkCfg c = dep_bulk_cfg(nonuni);
    const size_t sm = dep_bulk_smem(c.rs, c.stages, nonuni);
    auto kern = dv == 3 ? (nonuni ? k_deposit_bulk<3, true> : k_deposit_bulk<3, false>)
                        : (nonuni ? k_deposit_bulk<2, true> : k_deposit_bulk<2, false>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<M * CH, kDepThreads, sm, st>>>((const float4*)xv, (const float4*)sw, cell_start, M, CH,
                                          1.0 / eta, uniform_w, part, c.rs, c.stages);
  } else if (var == 2 && dv == 3)
    k_deposit_partials_v2<3, 2, 4><<<M * CH, kDepThreads, 0, st>>>(
        (const float4*)xv, (const float4*)sw, cell_start, M, CH, 1.0 / eta, uniform_w, part);
  else if (var == 2)
    k_deposit_partials_v2<2, 2, 4><<<M * CH, kDepThreads, 0, st>>>(
        (const float4*)xv, (const float4*)sw, cell_start, M, CH, 1.0 / eta, uniform_w, part);
  else if (var == 3 && dv == 3)
    k_deposit_partials_v2<3, 4, 3><<<M * CH, kDepThreads, 0, st>>>(
        (const float4*)xv, (const float4*)sw, cell_start, M, CH, 1.0 / eta, uniform_w, part);
  else if (var == 3)
    k_deposit_partials_v2<2, 4, 3><<<M * CH, kDepThreads, 0, st>>>(
        (const float4*)xv, (const float4*)sw, cell_start, M, CH, 1.0 / eta, uniform_w, part);
  else if (dv == 3)
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
                              double ie, float* __restrict__ Ep, int64_t lde,
                              float* __restrict__ Bp, int64_t ldb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double g = fma((double)x[i], ie, -0.5);  // as in push_one
    const double fl = floor(g);
    const float f1 = (float)(g - fl), f0 = 1.f - f1;
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
    k_interpolate<3><<<blocks, 256, 0, (cudaStream_t)stream>>>(x, n, E1, E2, B3, M, 1.0 / eta,
                                                               Ep, lde, Bp, ldb);
  else
    k_interpolate<2><<<blocks, 256, 0, (cudaStream_t)stream>>>(x, n, E1, E2, B3, M, 1.0 / eta,
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
