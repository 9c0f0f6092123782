// silu.cu — the BASELINE "2 x 128 SiLU" score network (M1) with
// its hidden-layer GEMMs on the 5th-generation tensor cores (tcgen05, accumulators in TMEM).
//
// Network (u = [x/L, v], float32 working copy of float64 master parameters, flat order
//   W1[H][4], b1[H], W2[H][H], b2[H], W3[3][H], b3[3]):
//   a1 = W1 u + b1, h1 = silu(a1); a2 = W2 h1 + b2, h2 = silu(a2); s = W3 h2 + b3.
// The ISM loss sum_p w_p (|s_p|^2 + 2 div_p) (ref: score.py:303-338 applied to this network)
// needs the exact Jacobian trace; it is carried by one divergence column per particle,
// div = d2 . (B d1) with B = W2 (.) C, C[h][h'] = sum_k W3[k][h] W1[h'][1+k] (see k_silu).
// Per chunk of 48 particles the CTA runs the layer GEMMs as split-BF16 (hi*hi + hi*lo + lo*hi,
// ~2^-16 relative) on tcgen05 with float32 TMEM accumulation; everything elementwise (SiLU
// and its first two derivatives, the W1/W3 layers, the s / div reductions over h, the loss
// terms) runs on the FP32 pipes with one thread per hidden unit (the TMEM lane) and four
// warpgroups splitting the chunk's particles. One persistent CTA per SM (224 KB of operand
// tiles, 512 TMEM columns); per-CTA float64 partial rows are reduced in a fixed order and
// finalized by the shared AdamW kernel (adamw.cuh).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "adamw.cuh"
#include "common.cuh"
#include "f32x2.cuh"
#include "pairs.cuh"
#include "umma.cuh"

namespace spic {

__global__ void k_ism_reduce_cols(const double* __restrict__ part, int rows, int64_t width,
                                  double* __restrict__ out);  // sbtm.cu

namespace {

constexpr int kH = 128;       // hidden width of the tensor-core path
constexpr int kCP = 48;       // particles per chunk (GEMM N of the layer GEMMs)
constexpr int kNWG = 4;       // compute warpgroups; thread = (hidden unit h, particle slice)
constexpr int kNCW = 128 * kNWG;  // compute threads
constexpr int kNT = kNCW + 32;    // + one MMA-issuer warp
constexpr int kPPT = kCP / kNWG;  // particles per thread per chunk
constexpr uint32_t kTmemCols = 512;
// The weight-gradient accumulators dW2 (D3) and M (D4) stay in TMEM for at most this many
// chunks; then they are added into a per-CTA float32 buffer in global memory (L2) and the
// next G3 starts a fresh accumulation. The tensor pipe's float32 accumulation is not
// round-to-nearest: over ~600 chunks (n = 2^22 on 148 CTAs) its error reached 2e-4 relative
// on the tangent terms, over 64 chunks it stays at ~1e-5, independent of n.
constexpr int kFlushChunks = 64;
constexpr uint32_t kColD1 = 0, kColD2 = 128, kColD3 = 256;  // self-test accumulators

#ifdef SPIC_SILU_TRACE  // tools/silu_trace.cu: per-phase clock64 stamps of CTA 0, thread 0
__device__ long long g_silu_trace[64 * 16];
#define SILU_TRACE(k)                                                                  \
  do {                                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0 && it < 64) g_silu_trace[it * 16 + (k)] = clock64(); \
  } while (0)
#define SILU_TRACE_K(k)                                                                \
  do {                                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_silu_trace[63 * 16 + (k)] = clock64();   \
  } while (0)
#define SILU_TRACE_I(k)                                                                \
  do {                                                                                 \
    if (blockIdx.x == 0 && lane == 0 && iit < 64) g_silu_trace[iit * 16 + (k)] = clock64(); \
  } while (0)
#else
#define SILU_TRACE_K(k) \
  do {                  \
  } while (0)
#define SILU_TRACE_I(k) \
  do {                  \
  } while (0)
#define SILU_TRACE(k) \
  do {                \
  } while (0)
#endif

__host__ __device__ constexpr int64_t silu_params(int H) { return (int64_t)H * H + 9 * H + 3; }

struct SiluShared {
  float4 u[2][kCP];  // chunk records, double-buffered (the layer-1 reverse sweep runs late)
  float w[kCP];
  float4 gs[kCP];              // ISM: (2w s, 2w); MSE: (2w' (s - t), 0)
  uint64_t bar[4];  // [0] G1 done, [1] G3 done (X, Y free again), [2] G2 done,
                    // [3] G1's primal half done (ISM: F2a starts on it while B d1 runs)
  uint32_t tmem;
};
// W2 and B = W2 (.) C as 128-row SWIZZLE_128B operand tiles (hi, lo); X and Y as activation
// tiles (hi, lo) of 96 particle columns in the interleaved core-matrix layout (umma.cuh):
// columns 0..47 = the chunk's primal columns, 48..95 = its divergence columns
constexpr uint32_t kXTile = 2 * (kCP / 8) * umma::kActGroup;  // 96 particle columns: 24 KB
// per-warp-quarter partials (s0, s1, s2, div) per particle and the MSE targets live in the Y
// tile while it is free (after the previous chunk's G2 / G3, before this chunk's F2b)
constexpr uint32_t kRedBytes = 4 * 4 * kPPT * sizeof(float);  // per warpgroup
static_assert(kRedBytes <= umma::kActGroup && kCP * sizeof(float4) <= umma::kActGroup,
              "scratch fits one 8-particle group of the Y tile");
constexpr size_t kSiluTiles = 4 * umma::kTileBytes + 4 * kXTile;
// The dynamic shared window starts 1024-B aligned on sm_100 (checked in-kernel: a
// misaligned start traps), so no alignment slack is requested.
constexpr size_t kSiluSmem = kSiluTiles + sizeof(SiluShared);
static_assert(6 * umma::kTileBytes <= kSiluTiles, "self-test tiles fit");

// 1024-B aligned start inside the dynamic shared buffer (SWIZZLE_128B atoms). The offset is
// applied to the __shared__ array itself so the compiler keeps shared-space (LDS/STS)
// addressing for everything derived from it.
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  if (a & 1023u) __trap();  // SWIZZLE_128B operand tiles need 1024-B aligned atoms
  return p;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// logistic sigmoid: rcp.approx(1 + 2^(-a log2 e)) (MUFU.EX2 + MUFU.RCP)
__device__ __forceinline__ float sigmoid(float a) {
  return fast_rcp(1.f + ex2_approx(a * -1.4426950408889634f));
}
// the same for two values packed in f32x2 (FMUL2 / FADD2 around the per-lane MUFUs)
__device__ __forceinline__ f2 sigmoid2(f2 a) {
  float t0, t1;
  un2(mul2(a, mk2(-1.4426950408889634f, -1.4426950408889634f)), t0, t1);
  float s0, s1;
  un2(add2(mk2(ex2_approx(t0), ex2_approx(t1)), mk2(1.f, 1.f)), s0, s1);
  return mk2(fast_rcp(s0), fast_rcp(s1));
}

// The chunk's records sit in S.u in particle pairs, so the packed (f32x2) phases read two
// particles' components as aligned register pairs: for particles 2j, 2j+1
//   u[2j] = (x_a, x_b, v0_a, v0_b),  u[2j + 1] = (v1_a, v1_b, v2_a, v2_b).
__device__ __forceinline__ void put_u(float4* ub, int p, float4 u) {
  float* f = reinterpret_cast<float*>(ub + (p & ~1));
  const int s = p & 1;
  f[s] = u.x;
  f[2 + s] = u.y;
  f[4 + s] = u.z;
  f[6 + s] = u.w;
}
__device__ __forceinline__ float4 get_u(const float4* ub, int p) {
  const float* f = reinterpret_cast<const float*>(ub + (p & ~1));
  const int s = p & 1;
  return make_float4(f[s], f[2 + s], f[4 + s], f[6 + s]);
}

// one butterfly level over v[0 .. 2w): lanes with bit w set keep the upper half, the others
// the lower, and add the partner's other half (adds paired into FADD2 for w >= 2)
template <int W, int N>
__device__ __forceinline__ void butterfly(float (&v)[N], int lane) {
  const bool up = (lane & W) != 0;
  if constexpr (W == 1) {
    const float send = up ? v[0] : v[1];
    const float keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  } else {
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      const float s0 = up ? v[i] : v[i + W], s1 = up ? v[i + 1] : v[i + 1 + W];
      const float k0 = up ? v[i + W] : v[i], k1 = up ? v[i + 1 + W] : v[i + 1];
      const float r0 = __shfl_xor_sync(0xffffffffu, s0, W);
      const float r1 = __shfl_xor_sync(0xffffffffu, s1, W);
      un2(add2(mk2(k0, k1), mk2(r0, r1)), v[i], v[i + 1]);
    }
  }
}

// lane l ends with the warp-wide sum of v[l] (31 shuffles for 32 values)
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
  butterfly<16>(v, lane);
  butterfly<8>(v, lane);
  butterfly<4>(v, lane);
  butterfly<2>(v, lane);
  butterfly<1>(v, lane);
  return v[0];
}

// lanes l and l ^ 16 end with the warp-wide sum of v[l & 15]: the four butterfly levels leave
// each lane the half-warp sum of one value, one xor-16 exchange finishes it (16 shuffles for 16
// values; exchanging all 16 values across the half-warps first took 31)
__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
  butterfly<8>(v, lane);
  butterfly<4>(v, lane);
  butterfly<2>(v, lane);
  butterfly<1>(v, lane);
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

__device__ __forceinline__ void wg_sync(int wg) {  // named barrier of one warpgroup
  asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
}
// the 512 compute threads (the issuer warp does not take part)
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 5, 512;" ::: "memory"); }
// hand-offs compute -> issuer: X tile ready (6), Y tile ready (7); compute threads arrive,
// the issuer warp waits (544 = 512 + 32)
__device__ __forceinline__ void handoff_arrive(int id) {
  asm volatile("bar.arrive %0, 544;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void handoff_wait(int id) {
  asm volatile("bar.sync %0, 544;" ::"r"(id) : "memory");
}

// Split-BF16 of two values into packed bf16x2 words (lower half = a, upper half = b): hi and
// the rounded remainder lo (x ~= hi + lo to ~2^-17 relative).
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(b), "f"(a));
  const float ra = a - __uint_as_float(hi << 16), rb = b - __uint_as_float(hi & 0xffff0000u);
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(rb), "f"(ra));
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
// This thread's 12 particles (columns kPPT wg .. kPPT wg + 11 of a 48-column block) of hidden
// unit h into an activation tile, hi at the given addresses, lo at + kXTile: one 16-byte
// store for the 8-particle group it covers completely and one 8-byte store for the half
// group it shares with the neighbouring warpgroup. a8 / a4: the thread's byte addresses of
// those two (fixed per thread); odd warpgroups hold the half group first.
__device__ __forceinline__ void store_act12(uint32_t a8, uint32_t a4, bool half_first,
                                            const float (&v)[kPPT]) {
  uint32_t hi[6], lo[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) split2(v[2 * j], v[2 * j + 1], hi[j], lo[j]);
  if (half_first) {
    sts64(a4, hi[0], hi[1]);
    sts64(a4 + kXTile, lo[0], lo[1]);
    sts128(a8, hi[2], hi[3], hi[4], hi[5]);
    sts128(a8 + kXTile, lo[2], lo[3], lo[4], lo[5]);
  } else {
    sts128(a8, hi[0], hi[1], hi[2], hi[3]);
    sts128(a8 + kXTile, lo[0], lo[1], lo[2], lo[3]);
    sts64(a4, hi[4], hi[5]);
    sts64(a4 + kXTile, lo[4], lo[5]);
  }
}

// One CTA per SM, four warpgroups. Thread (h, warpgroup g) owns hidden unit h (its TMEM lane)
// for particles 8g..8g+7 of each 32-particle chunk; one thread issues the CTA's GEMMs.
//
// The exact divergence is carried by one extra column per particle instead of three forward
// tangents: with C[h][h'] = sum_k W3[k][h] W1[h'][1+k] and B = W2 (.) C (elementwise),
//   div = d2 . (B d1),  d1 = silu'(a1), d2 = silu'(a2)
// so per chunk (columns: 32 primal + 32 divergence)
//   G1  [a2 - b2 | e]     = [W2 h1 | B d1]
//   G2  [dh1 | f]         = [W2^T da2 | B^T y2],   y2 = 2w d2 (the dL/de column)
//   G3  dW2 += da2 h1^T,   M += y2 d1^T             (TMEM-resident over the CTA's chunks)
// and at the end of the kernel dW2 += C (.) M, dW3[k][h] += sum_h' W1[h'][1+k] (W2 (.) M)[h][h'],
// dW1[h'][1+k] += sum_h W3[k][h] (W2 (.) M)[h][h'] (the tangent terms, once per CTA).
// MODE 0: forward only (scores into sw_out lanes 0..2, weight lane kept); 1: ISM partials
// (exact divergence); 2: weighted MSE partials to a target score (pretraining, ref:
// score.py:254-300 applied to this network; no divergence columns).
// Inputs: cell-sorted records (xv != NULL) or pid-order planes x, v[3][ldv], w read through
// idx (nullable) together with the target planes Z[3][ldz].
struct SiluInputs {
  const float4* xv;
  const float4* sw;
  const float* x;
  const float* v;
  int64_t ldv;
  const float* w;
  const float* Z;
  int64_t ldz;
  const int32_t* idx;
  float inv_wsum;
};

template <int MODE>
__global__ void __launch_bounds__(kNT, 1) k_silu(const float* __restrict__ params,
                                                 const SiluInputs in, int64_t n,
                                                 float x_scale, float L,
                                                 float4* __restrict__ sw_out,
                                                 double* __restrict__ part,
                                                 float* __restrict__ part_w2,
                                                 float* __restrict__ part_acc) {
  constexpr bool ISM = MODE != 0;  // training modes (loss + gradient partials)
  constexpr bool DIV = MODE == 1;  // divergence columns
  const float4* __restrict__ xv = in.xv;
  const float4* __restrict__ sw = in.sw;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  static_assert(56 * 1024 + 16 * 32 * 17 * 4 <= 4 * 32768, "epilogue staging fits below X");
  uint8_t* W2h = base;
  uint8_t* W2l = base + 1 * umma::kTileBytes;
  uint8_t* Bh = base + 2 * umma::kTileBytes;
  uint8_t* Bl = base + 3 * umma::kTileBytes;
  uint8_t* Xh = base + 4 * umma::kTileBytes;  // lo at + kXTile, Y hi at + 2 kXTile
  SiluShared& S = *reinterpret_cast<SiluShared*>(base + kSiluTiles);
  constexpr uint32_t kY = 2 * kXTile;
  constexpr uint32_t kDivRows = (kCP / 8) * umma::kActGroup;  // byte offset of the divergence columns

  SILU_TRACE_K(0);
  const int tid = threadIdx.x, h = tid & (kH - 1), wg = tid >> 7, lane = tid & 31;
  const int quarter = (tid >> 5) & 3, wtid = tid & 127;
  const float* W1 = params;
  const float* b1 = W1 + 4 * kH;
  const float* W2 = b1 + kH;
  const float* b2 = W2 + kH * kH;
  const float* W3 = b2 + kH;
  const float* b3 = W3 + 3 * kH;

  // operand tiles, eight columns (one 16-B swizzle chunk) per step
  for (int e8 = tid; e8 < kH * kH / 8; e8 += kNT) {
    const int r = (e8 * 8) / kH, c0 = (e8 * 8) % kH;  // W2[r][c0 .. c0+7]
    const float4 wa = __ldg(reinterpret_cast<const float4*>(W2 + r * kH + c0));
    const float4 wb = __ldg(reinterpret_cast<const float4*>(W2 + r * kH + c0 + 4));
    float w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
    umma::store_split8(W2h, W2l, r, c0, w);
    if (DIV) {
      const float a0 = W3[r], a1 = W3[kH + r], a2 = W3[2 * kH + r];
      float bv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 w1c = __ldg(reinterpret_cast<const float4*>(W1) + c0 + k);  // W1[c][0..3]
        bv[k] = w[k] * fmaf(a2, w1c.w, fmaf(a1, w1c.z, a0 * w1c.y));
      }
      umma::store_split8(Bh, Bl, r, c0, bv);
    }
  }
  float w1[4], w3[3];
#pragma unroll
  for (int i = 0; i < 4; ++i) w1[i] = W1[h * 4 + i];
#pragma unroll
  for (int k = 0; k < 3; ++k) w3[k] = W3[k * kH + h];
  const float bb1 = b1[h], bb2 = b2[h];
  if (tid < 32) umma::tmem_alloc(&S.tmem, kTmemCols);
  if (tid == 32) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_init(&S.bar[2], 1);
    mbar_init(&S.bar[3], 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = S.tmem;
  SILU_TRACE_K(1);
  const uint32_t tl = tm + ((uint32_t)(quarter * 32) << 16);  // this warp's TMEM lanes
  const uint32_t sW2h = smem_u32(W2h), sW2l = smem_u32(W2l), sBh = smem_u32(Bh),
                 sBl = smem_u32(Bl), sXh = smem_u32(Xh), sXl = sXh + kXTile,
                 sYh = sXh + kY, sYl = sYh + kXTile;
  // TMEM columns: D1 = [a2 - b2 | e], D2 = [dh1 | f] (kCP each), D3 = dW2, D4 = M
  constexpr uint32_t cD1 = 0, cD2 = 128, cD3 = 256, cD4 = 384;
  // store addresses of this thread's hidden unit h in the X hi tile (primal columns): the
  // 8-particle group its warpgroup covers completely and the half group it shares
  // (warpgroup particles 12 wg .. 12 wg + 11: groups {0, 1lo}, {1hi, 2}, {3, 4lo}, {4hi, 5})
  const bool half_first = (wg & 1) != 0;
  const uint32_t hofs = (uint32_t)((h >> 3) * 128 + (h & 7) * 16);
  const uint32_t xa8 = sXh + hofs + (uint32_t)((wg & 1 ? 3 * (wg >> 1) + 2 : 3 * (wg >> 1)) * umma::kActGroup);
  const uint32_t xa4 = sXh + hofs + (uint32_t)((3 * (wg >> 1) + 1) * umma::kActGroup) + (half_first ? 8u : 0u);
  // per-warp-quarter partials of this warpgroup's 12 particles: in the Y tile while it is
  // free, inside the 8-particle group the warpgroup alone writes in F2b — so F2b of a faster
  // warpgroup never touches another warpgroup's partials and the hand-over to F2b needs only a
  // warpgroup barrier. The MSE targets sit in group 1 (shared by warpgroups 0 and 1: the MSE
  // mode keeps the CTA-wide barrier).
  float (*red)[4 * kPPT] = reinterpret_cast<float (*)[4 * kPPT]>(
      Xh + kY + (size_t)(wg & 1 ? 3 * (wg >> 1) + 2 : 3 * (wg >> 1)) * umma::kActGroup);
  float4* tgt = reinterpret_cast<float4*>(Xh + kY + umma::kActGroup);

  // per-thread sums over the CTA's chunks in float32 (<= ~150 chunk terms each); the CTA and
  // cross-CTA combines are float64
  float gw1[4] = {0, 0, 0, 0}, gb1 = 0, gb2 = 0, gw3[3] = {0, 0, 0};
  float loss = 0, gb3[3] = {0, 0, 0};
  uint32_t phase = 0, phase2 = 0, phase3 = 0, phase_p = 0;
  bool first = true;
  const int64_t nchunks = (n + kCP - 1) / kCP;
  const int p0 = kPPT * wg;  // this warpgroup's particles inside the chunk (= GEMM columns)

  // F3: reverse through layer 1 -> dW1 (input part), db1, for chunk cc whose G2 result is in
  // D2. The ISM runs it one chunk late, while the tensor cores compute the next chunk's G1
  // (re-reading that chunk's records, an L2 hit); MSE runs it in order from S.u.
  int it = 0;  // chunk iteration of this CTA (trace stamps)
  auto layer1_reverse = [&](int ub) {
    umma::wait_mma(&S.bar[2], phase2);
    phase2 ^= 1;
    umma::fence_after();
    SILU_TRACE(9);
#ifdef SPIC_SILU_NO_F3  // timing diagnostic only (wrong gradients): G1 without concurrent F3
    return;
#endif
    float vd[16], vf[16];
    if (DIV) umma::tmem_ld12x2(tl + cD2 + p0, tl + cD2 + kCP + p0, vd, vf);
    else umma::tmem_ld12(tl + cD2 + p0, vd);
    const f2 one2 = mk2(1.f, 1.f);
    f2 aw[4] = {mk2(0.f, 0.f), mk2(0.f, 0.f), mk2(0.f, 0.f), mk2(0.f, 0.f)}, ab = mk2(0.f, 0.f);
#pragma unroll
    for (int pp = 0; pp < kPPT; pp += 2) {  // two particles per f32x2 lane pair
      const float4 A = S.u[ub][p0 + pp], B = S.u[ub][p0 + pp + 1];
      const f2 ux = mk2(A.x, A.y), uy = mk2(A.z, A.w), uz = mk2(B.x, B.y), uw = mk2(B.z, B.w);
      const f2 a = fma2(mk2(w1[3], w1[3]), uw,
                        fma2(mk2(w1[2], w1[2]), uz,
                             fma2(mk2(w1[1], w1[1]), uy, fma2(mk2(w1[0], w1[0]), ux, mk2(bb1, bb1)))));
      const f2 sg = sigmoid2(a);
      const f2 omg = sub2(one2, sg);
      const f2 d1 = mul2(sg, fma2(a, omg, one2));
      f2 da1 = mul2(d1, mk2(vd[pp], vd[pp + 1]));
      if (DIV)
        da1 = fma2(mul2(mul2(sg, omg), fma2(a, fma2(mk2(-2.f, -2.f), sg, one2), mk2(2.f, 2.f))),
                   mk2(vf[pp], vf[pp + 1]), da1);
      ab = add2(ab, da1);
      aw[0] = fma2(da1, ux, aw[0]);
      aw[1] = fma2(da1, uy, aw[1]);
      aw[2] = fma2(da1, uz, aw[2]);
      aw[3] = fma2(da1, uw, aw[3]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float lo, hi;
      un2(aw[i], lo, hi);
      gw1[i] += lo + hi;
    }
    {
      float lo, hi;
      un2(ab, lo, hi);
      gb1 += lo + hi;
    }
  };

  // this thread's 32-column slice of D3 / D4 (row h, columns 32 wg ..) in the CTA's buffer.
  // Only this thread ever touches its slice, so the buffer is laid out for the access, not as
  // a matrix: float4 number k (columns 32 wg + 4k ..) of row h sits at
  // ((which * 4 + wg) * 8 + k) * 128 + h — a warp's 32 rows are 512 contiguous bytes per load
  // instead of 32 half-used sectors.
  int nflush = 0;
  float4* acc_row = part_acc ? reinterpret_cast<float4*>(part_acc + (size_t)blockIdx.x * 2 * kH * kH) +
                                   (size_t)wg * 8 * kH + h
                             : nullptr;
  constexpr size_t kAccWhich = (size_t)kNWG * 8 * kH;  // float4 stride between D3 and D4 sums
  auto flush_acc = [&](uint32_t col, int which) {
    float t[32];
    umma::tmem_ld32(tl + col + (uint32_t)(32 * wg), t);
    float4* g = acc_row + (size_t)which * kAccWhich;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float4 a = make_float4(t[4 * k], t[4 * k + 1], t[4 * k + 2], t[4 * k + 3]);
      if (nflush) {
        const float4 b = g[k * kH];
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      g[k * kH] = a;
    }
  };
  bool pending = false;  // the previous chunk's layer-1 reverse sweep is still to run (ISM)
  int ub = 0;            // S.u buffer of the current chunk
  if (tid >= kNCW) {
    // issuer warp: every GEMM of the CTA in chunk order, as soon as its operands are ready.
    // (An MMA issue blocks while the tensor pipe's queue is full, so a compute warp that
    // issued would stall for most of the GEMM time.)
    bool fst = true;
    int iit = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++iit) {
      handoff_wait(MODE == 0 && (iit & 1) ? 8 : 6);  // X written (F1 of chunk c)
      umma::fence_after();
      SILU_TRACE_I(10);
      {  // the whole warp issues (elect.sync inside), see umma::mma_elect
        if constexpr (MODE == 0) {
          // the forward double-buffers X (odd chunks in the unused B tiles) and D1 (odd chunks
          // in the D2 columns)
          const bool odd = iit & 1;
          const uint32_t xb = odd ? sBh : sXh;
          umma::gemm_split_v<umma::kWK, umma::kActMN, kCP, 8>(tm + (odd ? cD2 : cD1), sW2h, sW2l, xb,
                                                              xb + kXTile, false);
        } else {
          umma::gemm_split_v<umma::kWK, umma::kActMN, kCP, 8>(tm + cD1, sW2h, sW2l, sXh, sXl,
                                                              false);  // W2 h1
        }
        if (DIV) {
          umma::commit_elect(&S.bar[3]);  // primal half: F2a's s partials start on it
          umma::gemm_split_v<umma::kWK, umma::kActMN, kCP, 8>(
              tm + cD1 + kCP, sBh, sBl, sXh + kDivRows, sXl + kDivRows, false);  // B d1
        }
        umma::commit_elect(&S.bar[0]);
      }
      __syncwarp();
      SILU_TRACE_I(11);
      if (ISM) {
        const bool acc3 = !fst && (iit % kFlushChunks) != 0;  // fresh after a flush
        if (DIV) {
          // The divergence columns of Y (y2 = 2w d2) do not depend on the scores: F2a stores
          // them as soon as G1's primal half is in, and their halves of G3 and G2 run on the
          // tensor pipe while the FP32 side does the s / div reductions and F2b.
          handoff_wait(9);  // Y divergence rows written (F2a of chunk c)
          umma::fence_after();
          umma::gemm_split_v<umma::kActK, umma::kActK, 128, kCP / 16>(
              tm + cD4, sYh + kDivRows, sYl + kDivRows, sXh + kDivRows, sXl + kDivRows,
              acc3);  // y2 d1^T
          umma::gemm_split_v<umma::kWMN, umma::kActMN, kCP, 8>(
              tm + cD2 + kCP, sBh, sBl, sYh + kDivRows, sYl + kDivRows, false);  // B^T y2
          __syncwarp();
        }
        handoff_wait(7);  // Y primal rows written (F2b of chunk c)
        umma::fence_after();
        SILU_TRACE_I(12);
        {
          // G3 first: the next chunk's layer-1 sweep waits for it (X, Y reuse)
          umma::gemm_split_v<umma::kActK, umma::kActK, 128, kCP / 16>(tm + cD3, sYh, sYl, sXh, sXl,
                                                                      acc3);  // da2 h1^T
          umma::commit_elect(&S.bar[1]);
#ifdef SPIC_SILU_TRACE_G3  // timing diagnostic: stamp G3's completion before issuing G2
          {
            uint32_t ph = (uint32_t)(iit & 1);
            umma::wait_mma(&S.bar[1], ph);
            SILU_TRACE_I(14);
          }
#endif
          umma::gemm_split_v<umma::kWMN, umma::kActMN, kCP, 8>(tm + cD2, sW2h, sW2l, sYh, sYl,
                                                               false);  // W2^T da2
          umma::commit_elect(&S.bar[2]);
        }
        __syncwarp();
        SILU_TRACE_I(13);
        fst = false;
      }
    }
  } else if constexpr (MODE == 0) {
    // Forward only: layer-1 sweep of chunk i (into X buffer i & 1) runs while the tensor cores
    // compute G1 of chunk i - 1 (from the other buffer, into the other accumulator), whose
    // scores follow. Nothing else shares the B tiles or the D2 columns in this mode.
    const uint32_t xdelta = sBh - sXh;
    int64_t cprev = -1;
    for (int64_t c = blockIdx.x;; c += gridDim.x, ++it) {
      const bool has = c < nchunks;
      const int buf = it & 1;
      if (has) {
        if (wtid < kPPT) {
          const int pl = p0 + wtid;
          const int64_t p = c * kCP + pl;
          float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p < n) {
            const float4 A = xv[p];
            const float x = A.x < 0.f ? A.x + L : A.x;  // % M quirk records carry x - L
            u = make_float4(x * x_scale, A.y, A.z, A.w);
          }
          put_u(S.u[buf], pl, u);
        }
        if (tid == 0 && c + gridDim.x < nchunks) {  // next chunk's records into L2 (see ISM)
          const int64_t p0n = (c + gridDim.x) * kCP;
          const int64_t cntn = n - p0n < (int64_t)kCP ? n - p0n : (int64_t)kCP;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(xv + p0n),
                       "r"((uint32_t)(sizeof(float4) * (size_t)cntn))
                       : "memory");
        }
        wg_sync(wg);
        {
          float f1h[kPPT];
#pragma unroll
          for (int i = 0; i < kPPT; ++i) {
            const float4 u = get_u(S.u[buf], p0 + i);
            const float a = fmaf(w1[3], u.w, fmaf(w1[2], u.z, fmaf(w1[1], u.y, fmaf(w1[0], u.x, bb1))));
            f1h[i] = a * sigmoid(a);
          }
          const uint32_t xo = buf ? xdelta : 0u;
          store_act12(xa8 + xo, xa4 + xo, half_first, f1h);
        }
        fence_proxy_async();
        umma::fence_before();
        // bar.arrive does not wait, so a warpgroup can run one chunk ahead of another (never
        // two: that needs G1 of the chunk before, i.e. everyone's arrival for it). Alternating
        // barrier IDs by chunk parity keep an early arrival from completing the issuer's
        // barrier of the previous chunk before a lagging warpgroup has written its rows.
        handoff_arrive(buf ? 8 : 6);
      }
      if (cprev >= 0) {
        umma::wait_mma(&S.bar[0], phase);
        phase ^= 1;
        umma::fence_after();
        {
          float va[16];
          umma::tmem_ld12(tl + (buf ? cD1 : cD2) + p0, va);  // chunk cprev used buffer buf ^ 1
          float v32[32], v16[16];
#pragma unroll
          for (int pp = 0; pp < kPPT; ++pp) {
            const float a2 = va[pp] + bb2;
            const float h2 = a2 * sigmoid(a2);
            float* dst = pp < 8 ? &v32[4 * pp] : &v16[4 * (pp - 8)];
            dst[0] = w3[0] * h2;
            dst[1] = w3[1] * h2;
            dst[2] = w3[2] * h2;
            dst[3] = 0.f;
          }
          const float r32 = transpose_reduce32(v32, lane);
          const float r16 = transpose_reduce16(v16, lane);
          red[quarter][lane] = r32;
          if (lane < 16) red[quarter][32 + lane] = r16;
        }
        wg_sync(wg);
        if (wtid < kPPT) {
          const int p = p0 + wtid;
          float sc[3];
#pragma unroll
          for (int k = 0; k < 3; ++k)
            sc[k] = b3[k] + ((red[0][4 * wtid + k] + red[1][4 * wtid + k]) +
                             (red[2][4 * wtid + k] + red[3][4 * wtid + k]));
          const int64_t q = cprev * kCP + p;
          if (q < n) sw_out[q] = make_float4(sc[0], sc[1], sc[2], sw[q].w);
        }
        umma::fence_before();
        wg_sync(wg);  // red is rewritten by the next chunk
      }
      if (!has) break;
      cprev = c;
    }
  } else {
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    SILU_TRACE(0);
    // each warpgroup loads, reduces and scores its own 8 particles: only the GEMM issue points
    // need the whole CTA, everything else synchronises one warpgroup (named barrier)
    auto wait_g3 = [&]() {  // the previous chunk's weight-gradient GEMMs still read X and Y
      if (ISM && !first) {
        umma::wait_mma(&S.bar[1], phase3);
        phase3 ^= 1;
        umma::fence_after();
      }
    };
    // MSE keeps its targets in the Y tile: wait before loading; the ISM loads its records and
    // runs the layer-1 arithmetic while G3 drains, and waits only before the X stores
    if (MODE != 1) wait_g3();
    if (wtid < kPPT) {
      const int pl = p0 + wtid;
      const int64_t p = c * kCP + pl;
      float4 u = make_float4(0.f, 0.f, 0.f, 0.f), t = u;
      float wt = 0.f;
      if (p < n) {
        if (xv) {
          const float4 A = xv[p];
          const float x = A.x < 0.f ? A.x + L : A.x;  // % M quirk records carry x - L
          u = make_float4(x * x_scale, A.y, A.z, A.w);
          wt = sw[p].w;
        } else {
          const int64_t r = in.idx ? (int64_t)in.idx[p] : p;
          u = make_float4(in.x[r] * x_scale, in.v[r], in.v[in.ldv + r], in.v[2 * in.ldv + r]);
          wt = in.w[r];
          if (MODE == 2) t = make_float4(in.Z[r], in.Z[in.ldz + r], in.Z[2 * in.ldz + r], 0.f);
        }
      }
      put_u(S.u[ub], pl, u);
      S.w[pl] = wt;
      if (MODE == 2) tgt[pl] = t;
    }
    if (xv && tid == 0) {
      // the CTA's next chunk of records into L2 (one bulk prefetch per record array, no
      // registers held): its loads at the top of the next chunk then miss only to L2
      const int64_t cn = c + gridDim.x;
      if (cn < nchunks) {
        const int64_t p0n = cn * kCP;
        const int64_t cntn = n - p0n < (int64_t)kCP ? n - p0n : (int64_t)kCP;
        const uint32_t bytes = (uint32_t)(sizeof(float4) * (size_t)cntn);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(xv + p0n), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sw + p0n), "r"(bytes)
                     : "memory");
      }
    }
    wg_sync(wg);
    SILU_TRACE(1);

    // F1: layer 1 -> X rows p (h1) and 32 + p (d1 = silu'(a1)), column h
    if (MODE == 1) {
      float f1h[kPPT], f1d[kPPT];
      const f2 one2 = mk2(1.f, 1.f);
#pragma unroll
      for (int i = 0; i < kPPT; i += 2) {  // two particles per f32x2 lane pair
        const float4 A = S.u[ub][p0 + i], B = S.u[ub][p0 + i + 1];
        const f2 a = fma2(mk2(w1[3], w1[3]), mk2(B.z, B.w),
                          fma2(mk2(w1[2], w1[2]), mk2(B.x, B.y),
                               fma2(mk2(w1[1], w1[1]), mk2(A.z, A.w),
                                    fma2(mk2(w1[0], w1[0]), mk2(A.x, A.y), mk2(bb1, bb1)))));
        const f2 sg = sigmoid2(a);
        un2(mul2(a, sg), f1h[i], f1h[i + 1]);
        un2(mul2(sg, fma2(a, sub2(one2, sg), one2)), f1d[i], f1d[i + 1]);
      }
      wait_g3();
      store_act12(xa8, xa4, half_first, f1h);
      store_act12(xa8 + kDivRows, xa4 + kDivRows, half_first, f1d);
    } else {
      float f1h[kPPT];
#pragma unroll
      for (int i = 0; i < kPPT; ++i) {
        const float4 u = get_u(S.u[ub], p0 + i);
        const float a = fmaf(w1[3], u.w, fmaf(w1[2], u.z, fmaf(w1[1], u.y, fmaf(w1[0], u.x, bb1))));
        f1h[i] = a * sigmoid(a);
      }
      store_act12(xa8, xa4, half_first, f1h);
    }
    fence_proxy_async();
    umma::fence_before();
    handoff_arrive(6);
    SILU_TRACE(2);
    if (it > 0 && it % kFlushChunks == 0) {
      // G3 of the previous chunk is complete (wait_g3 above) and the next G3 is issued only
      // after this chunk's F2b hand-off: move D3 (and D4) into the CTA's float32 buffer
      flush_acc(cD3, 0);
      if (DIV) flush_acc(cD4, 1);
      ++nflush;
    }
    if (MODE == 1 && pending) layer1_reverse(ub ^ 1);  // overlaps this chunk's G1
    SILU_TRACE(3);
    if (DIV) {  // the primal half of G1 (the div half is awaited inside F2a)
      umma::wait_mma(&S.bar[3], phase_p);
      phase_p ^= 1;
    } else {
      umma::wait_mma(&S.bar[0], phase);
      phase ^= 1;
    }
    umma::fence_after();
    SILU_TRACE(4);

    // F2a: s and div partials over this thread's h, reduced across the warp (particles
    // 0..7 of the warpgroup by a 32-value, 8..11 by a 16-value transpose-reduce)
    {
      float va[16], ve[16];
      umma::tmem_ld12(tl + cD1 + p0, va);
      float v32[32], v16[16];
      const f2 one2 = mk2(1.f, 1.f);
      // (instantiated for both warpgroup parities so the Y divergence rows leave as soon as a
      // group's values exist: at most four packed words are pending instead of twelve floats)
      auto f2a_loop = [&](auto hf_tag) {
        constexpr bool HF = decltype(hf_tag)::value;  // half group (4 particles) first
        uint32_t yh[4], yl[4];
#pragma unroll
        for (int pp = 0; pp < kPPT; pp += 2) {  // two particles per f32x2 lane pair
          const f2 a2 = add2(mk2(va[pp], va[pp + 1]), mk2(bb2, bb2));
          const f2 sg = sigmoid2(a2);
          const f2 h2 = mul2(a2, sg);
          float* d0 = pp < 8 ? &v32[4 * pp] : &v16[4 * (pp - 8)];
          float* d1 = d0 + 4;
          un2(mul2(mk2(w3[0], w3[0]), h2), d0[0], d1[0]);
          un2(mul2(mk2(w3[1], w3[1]), h2), d0[1], d1[1]);
          un2(mul2(mk2(w3[2], w3[2]), h2), d0[2], d1[2]);
          // d2 = silu'(a2) for now; times e (the div half of G1) below
          un2(DIV ? mul2(sg, fma2(a2, sub2(one2, sg), one2)) : mk2(0.f, 0.f), d0[3], d1[3]);
          if (DIV) {  // Y divergence rows y2 = 2w d2 (no score dependence): G3 / G2 div halves
            const float2 wab = *reinterpret_cast<const float2*>(&S.w[p0 + pp]);  // one 8-B load
            const int j = pp >> 1;
            const int slot = HF ? (j < 2 ? j : j - 2) : (j < 4 ? j : j - 4);
            split2((wab.x + wab.x) * d0[3], (wab.y + wab.y) * d1[3], yh[slot], yl[slot]);
            const uint32_t a8y = xa8 + kY + kDivRows, a4y = xa4 + kY + kDivRows;
            if (HF ? j == 1 : j == 5) {
              sts64(a4y, yh[0], yh[1]);
              sts64(a4y + kXTile, yl[0], yl[1]);
            }
            if (HF ? j == 5 : j == 3) {
              sts128(a8y, yh[0], yh[1], yh[2], yh[3]);
              sts128(a8y + kXTile, yl[0], yl[1], yl[2], yl[3]);
            }
          }
        }
      };
      if (half_first) f2a_loop(std::true_type{}); else f2a_loop(std::false_type{});
      if (DIV) {
        fence_proxy_async();
        umma::fence_before();
        handoff_arrive(9);
        umma::wait_mma(&S.bar[0], phase);
        phase ^= 1;
        umma::fence_after();
        umma::tmem_ld12(tl + cD1 + kCP + p0, ve);
#pragma unroll
        for (int pp = 0; pp < kPPT; pp += 2) {
          float* d0 = pp < 8 ? &v32[4 * pp] : &v16[4 * (pp - 8)];
          float* d1 = d0 + 4;
          un2(mul2(mk2(d0[3], d1[3]), mk2(ve[pp], ve[pp + 1])), d0[3], d1[3]);
        }
      }
      const float r32 = transpose_reduce32(v32, lane);
      const float r16 = transpose_reduce16(v16, lane);
      red[quarter][lane] = r32;
      if (lane < 16) red[quarter][32 + lane] = r16;
    }
    wg_sync(wg);
    SILU_TRACE(5);
    if (wtid < kPPT) {
      const int p = p0 + wtid;
      float s[3], dv = 0.f;
#pragma unroll
      for (int k = 0; k < 3; ++k)
        s[k] = b3[k] + ((red[0][4 * wtid + k] + red[1][4 * wtid + k]) +
                        (red[2][4 * wtid + k] + red[3][4 * wtid + k]));
      dv = (red[0][4 * wtid + 3] + red[1][4 * wtid + 3]) + (red[2][4 * wtid + 3] + red[3][4 * wtid + 3]);
      const int64_t q = c * kCP + p;
      if (MODE == 0) {
        if (q < n) sw_out[q] = make_float4(s[0], s[1], s[2], sw[q].w);
      } else if (MODE == 2) {
        const float wi = S.w[p] * in.inv_wsum;
        const float4 t = tgt[p];
        const float r0 = s[0] - t.x, r1 = s[1] - t.y, r2 = s[2] - t.z;
        S.gs[p] = make_float4(2.f * wi * r0, 2.f * wi * r1, 2.f * wi * r2, 0.f);
        loss += wi * (r0 * r0 + r1 * r1 + r2 * r2);
        gb3[0] += 2.f * wi * r0;
        gb3[1] += 2.f * wi * r1;
        gb3[2] += 2.f * wi * r2;
      } else {
        const float wt = S.w[p], tw = 2.f * wt;
        S.gs[p] = make_float4(tw * s[0], tw * s[1], tw * s[2], tw);
        loss += wt * (s[0] * s[0] + s[1] * s[1] + s[2] * s[2] + 2.f * dv);
#pragma unroll
        for (int k = 0; k < 3; ++k) gb3[k] += tw * s[k];
      }
    }
    if (!ISM) {  // D1 is rewritten by the next chunk's G1 only after the next CTA barrier
      umma::fence_before();
      wg_sync(wg);
      continue;
    }
    // F2b overwrites the Y tile that holds the partials: this warpgroup's own (ISM), or, with
    // the MSE targets in a shared group, anybody's
    if (MODE == 1) wg_sync(wg); else compute_sync();
    SILU_TRACE(6);

    // F2b: reverse through layer 2 -> Y rows p (da2) and 32 + p (y2 = 2w d2); dW3, db2
    {
      const f2 z2 = mk2(0.f, 0.f), one2 = mk2(1.f, 1.f);
      f2 aw3[3] = {z2, z2, z2}, ab2 = z2;
      float va[16], ve[16], da2v[kPPT];
      if (DIV) umma::tmem_ld12x2(tl + cD1 + p0, tl + cD1 + kCP + p0, va, ve);
      else umma::tmem_ld12(tl + cD1 + p0, va);
#pragma unroll
      for (int pp = 0; pp < kPPT; pp += 2) {  // two particles per f32x2 lane pair
        const float4 Ga = S.gs[p0 + pp], Gb = S.gs[p0 + pp + 1];
        const f2 gx = mk2(Ga.x, Gb.x), gy = mk2(Ga.y, Gb.y), gz = mk2(Ga.z, Gb.z);
        const f2 a2 = add2(mk2(va[pp], va[pp + 1]), mk2(bb2, bb2));
        const f2 sg = sigmoid2(a2);
        const f2 omg = sub2(one2, sg);
        const f2 h2 = mul2(a2, sg);
        const f2 d2 = mul2(sg, fma2(a2, omg, one2));
        const f2 dh2 = fma2(mk2(w3[2], w3[2]), gz,
                            fma2(mk2(w3[1], w3[1]), gy, mul2(mk2(w3[0], w3[0]), gx)));
        f2 da2 = mul2(d2, dh2);
        if (DIV) {
          const f2 gw = mk2(Ga.w, Gb.w);
          const f2 e2 = mul2(mul2(sg, omg), fma2(a2, fma2(mk2(-2.f, -2.f), sg, one2), mk2(2.f, 2.f)));
          da2 = fma2(e2, mul2(gw, mk2(ve[pp], ve[pp + 1])), da2);
        }
        aw3[0] = fma2(gx, h2, aw3[0]);
        aw3[1] = fma2(gy, h2, aw3[1]);
        aw3[2] = fma2(gz, h2, aw3[2]);
        ab2 = add2(ab2, da2);
        un2(da2, da2v[pp], da2v[pp + 1]);
      }
      store_act12(xa8 + kY, xa4 + kY, half_first, da2v);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float lo, hi;
        un2(aw3[k], lo, hi);
        gw3[k] += lo + hi;
      }
      {
        float lo, hi;
        un2(ab2, lo, hi);
        gb2 += lo + hi;
      }
    }
    fence_proxy_async();
    umma::fence_before();
    handoff_arrive(7);
    SILU_TRACE(7);
    first = false;
    if (MODE == 1) {
      pending = true;
    } else {
      layer1_reverse(ub);
    }
    umma::fence_before();
    // The ISM needs no barrier here: everything the next chunk's loaders overwrite (S.u of two
    // chunks ago, S.w, the targets) was last read before this chunk's warpgroup barriers, and
    // the shared partials / gs are rewritten only behind the next chunk's own barriers.
    if (MODE != 1) wg_sync(wg);
    SILU_TRACE(8);
    ub ^= 1;
  }
  if (MODE == 1 && pending) layer1_reverse(ub ^ 1);
  }

  SILU_TRACE_K(2);
  if (ISM && tid < kNCW) {
    if (!first) {
      umma::wait_mma(&S.bar[1], phase3);
      umma::fence_after();
    }
    compute_sync();  // every warpgroup is done with the X / Y tiles before they are reused
    SILU_TRACE_K(4);
    const int64_t width = 1 + silu_params(kH);
    const int64_t oW1 = 1, ob1 = oW1 + 4 * kH, oW2 = ob1 + kH, ob2 = oW2 + kH * kH,
                  oW3 = ob2 + kH, ob3 = oW3 + 3 * kH;
    double* row = part + (size_t)blockIdx.x * width;
    float* prow = part_w2 + (size_t)blockIdx.x * kH * kH;  // dW2 partials (float)
    // dW2 = D3 + C (.) M (row h, columns h'); warpgroup g takes columns 32g..32g+31. The
    // tangent terms of dW3 (row sums of (W2 (.) M) W1[:,1+k]) and dW1 (column sums of
    // W3[k] (W2 (.) M)) go through shared memory: WM = W2 (.) M as float [h][h'].
    constexpr int kWMs = kH + 1;  // padded row stride: row writes by lane h hit distinct banks
    static_assert(sizeof(float) * kH * kWMs <= 4 * kXTile, "WM fits the X / Y tiles");
    float* WM = reinterpret_cast<float*>(Xh);  // the X and Y tiles are free now
    float tw3[3] = {0.f, 0.f, 0.f};
    {
      // the dW2 row block (rows 32q.. of this warp, columns 32g..32g+31) goes out through a
      // per-warp shared-memory transpose in two 16-column halves, so each store instruction
      // writes two 128-B row segments instead of 32 scattered doubles (free space after the
      // per-h combine area: base + 56 KB .. + 124 KB, 4352 B per warp). Each half loads its own
      // 16 columns of D3 / D4, of the flushed sums and of the W2 row (48 live registers; with
      // all 32 columns at once the block spilled most of them at the kernel's 96 registers)
      constexpr int kStg = 17;  // padded row stride (floats)
      float* stg = reinterpret_cast<float*>(base + 56 * 1024) + (size_t)(tid >> 5) * 32 * kStg;
      const int q32 = h & ~31;  // first row of this warp
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int c0 = 32 * wg + 16 * half;  // first column of this half
        float v[16], m[16], w2r[16];
        if (half == 0) SILU_TRACE_K(8);
        umma::tmem_ld16(tl + cD3 + (uint32_t)c0, v);
        if (DIV) umma::tmem_ld16(tl + cD4 + (uint32_t)c0, m);
        if (half == 0) SILU_TRACE_K(9);
        if (nflush) {  // the earlier windows' sums (fixed order: earlier windows first)
          const float4* g3 = acc_row + (size_t)(4 * half) * kH;
          const float4* g4 = g3 + kAccWhich;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 a = g3[k * kH];
            v[4 * k] = a.x + v[4 * k]; v[4 * k + 1] = a.y + v[4 * k + 1];
            v[4 * k + 2] = a.z + v[4 * k + 2]; v[4 * k + 3] = a.w + v[4 * k + 3];
            if (DIV) {
              const float4 b = g4[k * kH];
              m[4 * k] = b.x + m[4 * k]; m[4 * k + 1] = b.y + m[4 * k + 1];
              m[4 * k + 2] = b.z + m[4 * k + 2]; m[4 * k + 3] = b.w + m[4 * k + 3];
            }
          }
        }
        if (DIV && !first) {  // this thread's W2 row segment W2[h][c0 .. c0 + 15]
          const float4* w2v = reinterpret_cast<const float4*>(W2 + h * kH + c0);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 t4 = __ldg(w2v + k);
            w2r[4 * k] = t4.x; w2r[4 * k + 1] = t4.y; w2r[4 * k + 2] = t4.z; w2r[4 * k + 3] = t4.w;
          }
        }
        if (half == 0) SILU_TRACE_K(10);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int hp = c0 + j;
          float g = first ? 0.f : v[j];
          if (DIV && !first) {
            const float4 w1c = __ldg(reinterpret_cast<const float4*>(W1) + hp);  // W1[hp][0..3]
            const float Chh = fmaf(w3[2], w1c.w, fmaf(w3[1], w1c.z, w3[0] * w1c.y));
            const float wm = w2r[j] * m[j];
            g = fmaf(Chh, m[j], g);
            WM[h * kWMs + hp] = wm;
            tw3[0] = fmaf(w1c.y, wm, tw3[0]);
            tw3[1] = fmaf(w1c.z, wm, tw3[1]);
            tw3[2] = fmaf(w1c.w, wm, tw3[2]);
          } else if (DIV) {
            WM[h * kWMs + hp] = 0.f;
          }
          stg[lane * kStg + j] = g;
        }
        __syncwarp();
        if (half == 0) SILU_TRACE_K(11);
#pragma unroll
        for (int rr = 0; rr < 32; rr += 2) {
          const int r = rr + (lane >> 4), cc = lane & 15;
          prow[(size_t)(q32 + r) * kH + c0 + cc] = stg[r * kStg + cc];
        }
        __syncwarp();
        if (half == 0) SILU_TRACE_K(12);
      }
    }
    SILU_TRACE_K(5);
    // per-h sums over the four warpgroups in a fixed order (in the free W2 tiles)
    double* comb = reinterpret_cast<double*>(W2h);  // [4][kH][12] + [4][4]
    double* mine = comb + (size_t)(wg * kH + h) * 12;
    mine[0] = gw1[0]; mine[1] = gw1[1]; mine[2] = gw1[2]; mine[3] = gw1[3];
    mine[4] = gb1; mine[5] = gb2; mine[6] = gw3[0]; mine[7] = gw3[1]; mine[8] = gw3[2];
    mine[9] = tw3[0]; mine[10] = tw3[1]; mine[11] = tw3[2];
    double* lcomb = comb + 4 * kH * 12;  // [4 warpgroups][loss, gb3]
    if (wtid < 32) {
      const double lw = warp_sum((double)loss);
      double g3w[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) g3w[k] = warp_sum((double)gb3[k]);
      if (wtid == 0) {
        lcomb[4 * wg] = lw;
#pragma unroll
        for (int k = 0; k < 3; ++k) lcomb[4 * wg + 1 + k] = g3w[k];
      }
    }
    compute_sync();
    SILU_TRACE_K(6);
    // dW1[h][1+k] tangent part: sum over rows r of W3[k][r] WM[r][h] (column h); warpgroup g
    // sums rows 32g..32g+31, the four partials are added in a fixed order below
    float* cwp = reinterpret_cast<float*>(lcomb + 16);  // [4][kH][3]
    if (DIV) {
      float cw[3] = {0.f, 0.f, 0.f};
      for (int r = 32 * wg; r < 32 * wg + 32; ++r) {
        const float wm = WM[r * kWMs + h];
        cw[0] = fmaf(W3[r], wm, cw[0]);
        cw[1] = fmaf(W3[kH + r], wm, cw[1]);
        cw[2] = fmaf(W3[2 * kH + r], wm, cw[2]);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) cwp[(wg * kH + h) * 3 + k] = cw[k];
    }
    compute_sync();
    SILU_TRACE_K(7);
    if (wg == 0) {
      double t[12];
#pragma unroll
      for (int k = 0; k < 12; ++k)
        t[k] = (comb[(0 * kH + h) * 12 + k] + comb[(1 * kH + h) * 12 + k]) +
               (comb[(2 * kH + h) * 12 + k] + comb[(3 * kH + h) * 12 + k]);
      row[oW1 + 4 * h + 0] = t[0];
      row[ob1 + h] = t[4];
      row[ob2 + h] = t[5];
#pragma unroll
      for (int k = 0; k < 3; ++k) row[oW3 + k * kH + h] = t[6 + k] + t[9 + k];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float cw = DIV ? (cwp[(0 * kH + h) * 3 + k] + cwp[(1 * kH + h) * 3 + k]) +
                                   (cwp[(2 * kH + h) * 3 + k] + cwp[(3 * kH + h) * 3 + k])
                             : 0.f;
        row[oW1 + 4 * h + 1 + k] = t[1 + k] + (double)cw;
      }
    }
    if (tid == 0) {
      row[0] = (lcomb[0] + lcomb[4]) + (lcomb[8] + lcomb[12]);
#pragma unroll
      for (int k = 0; k < 3; ++k)
        row[ob3 + k] = (lcomb[1 + k] + lcomb[5 + k]) + (lcomb[9 + k] + lcomb[13 + k]);
    }
  }
  umma::fence_before();
  __syncthreads();
  SILU_TRACE_K(3);
  if (tid < 32) umma::tmem_free(tm, kTmemCols);
}

// One-CTA check of the three GEMM shapes (operand views) against a host reference.
// W, X, Y: float32 [128][128] row-major; D1 = W X^T, D2 = W^T Y^T, D3 = Y^T X.
__global__ void __launch_bounds__(128, 1) k_umma_selftest(const float* __restrict__ W,
                                                          const float* __restrict__ X,
                                                          const float* __restrict__ Y,
                                                          float* __restrict__ D1,
                                                          float* __restrict__ D2,
                                                          float* __restrict__ D3) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = align1024(smem_raw);
  uint8_t* T[6];
  for (int i = 0; i < 6; ++i) T[i] = base + i * umma::kTileBytes;
  SiluShared& S = *reinterpret_cast<SiluShared*>(base + 6 * umma::kTileBytes);
  const int tid = threadIdx.x;
  for (int e = tid; e < kH * kH; e += 128) {
    umma::store_split(T[0], T[1], e / kH, e % kH, W[e]);
    umma::store_split(T[2], T[3], e / kH, e % kH, X[e]);
    umma::store_split(T[4], T[5], e / kH, e % kH, Y[e]);
  }
  if (tid < 32) umma::tmem_alloc(&S.tmem, kTmemCols);
  if (tid == 32) {
    mbar_init(&S.bar[0], 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = S.tmem;
  uint32_t s[6];
  for (int i = 0; i < 6; ++i) s[i] = smem_u32(T[i]);
  if (tid == 0) {
    umma::gemm_split<false, false>(tm + kColD1, s[0], s[1], s[2], s[3], false);
    umma::gemm_split<true, false>(tm + kColD2, s[0], s[1], s[4], s[5], false);
    umma::gemm_split<true, true>(tm + kColD3, s[4], s[5], s[2], s[3], false);
    umma::commit(&S.bar[0]);
  }
  umma::wait_mma(&S.bar[0], 0);
  umma::fence_after();
  const uint32_t tl = tm + ((uint32_t)((tid >> 5) * 32) << 16);
  for (int g = 0; g < 4; ++g) {
    float v[32];
    umma::tmem_ld32(tl + kColD1 + 32 * g, v);
    for (int i = 0; i < 32; ++i) D1[tid * kH + 32 * g + i] = v[i];
    umma::tmem_ld32(tl + kColD2 + 32 * g, v);
    for (int i = 0; i < 32; ++i) D2[tid * kH + 32 * g + i] = v[i];
    umma::tmem_ld32(tl + kColD3 + 32 * g, v);
    for (int i = 0; i < 32; ++i) D3[tid * kH + 32 * g + i] = v[i];
  }
  umma::fence_before();
  __syncthreads();
  if (tid < 32) umma::tmem_free(tm, kTmemCols);
}

int silu_blocks(int64_t n) {
  const int64_t chunks = (n + kCP - 1) / kCP;
  return (int)std::max<int64_t>(1, std::min<int64_t>(chunks, kNumSMs));
}

}  // namespace

// single-CTA finalize: the reduced row [loss, grads] -> AdamW with recovery
__global__ void __launch_bounds__(1024) k_silu_finalize(
    const double* __restrict__ row, int64_t P, bool mse, double* __restrict__ params,
    double* __restrict__ m,
    double* __restrict__ v2, double* __restrict__ opt, double beta1, double beta2, double eps,
    double wd, int reset_lr, int apply_step, float* __restrict__ params32,
    double* __restrict__ grads_out, double* __restrict__ loss_out, double* cand, int32_t* flags) {
  adamw_with_recovery(row[0], row + 1, P, mse, params, m, v2, opt, beta1, beta2, eps, wd,
                      reset_lr, apply_step, params32, grads_out, loss_out, cand, flags);
}

// multi-CTA finalize (kSiluFinCTAs x 256 threads; sync = [ticket, ok flags])
constexpr int kSiluFinCTAs = 32;
__global__ void __launch_bounds__(256) k_silu_finalize_mc(
    const double* __restrict__ row, int64_t P, bool mse, double* __restrict__ params,
    double* __restrict__ m, double* __restrict__ v2, double* __restrict__ opt, double beta1,
    double beta2, double eps, double wd, int reset_lr, int apply_step, float* __restrict__ params32,
    double* __restrict__ grads_out, double* __restrict__ loss_out, double* cand, int32_t* flags,
    int32_t* sync) {
  adamw_with_recovery_mc(row[0], row + 1, P, mse, params, m, v2, opt, beta1, beta2, eps, wd,
                         reset_lr, apply_step, params32, grads_out, loss_out, cand, flags, sync);
}

}  // namespace spic

using namespace spic;

extern "C" int64_t spic_silu_num_params(int32_t H) { return silu_params(H); }

// byte offset of the float dW2 partial block inside the scratch (256-B aligned)
static size_t silu_f32_offset(int64_t n) {
  const size_t width = 1 + (size_t)silu_params(kH);
  const size_t b = sizeof(double) * ((size_t)(silu_blocks(n) + 1) * width + (size_t)silu_params(kH)) +
                   64 + sizeof(int32_t) * 64;
  return (b + 255) & ~(size_t)255;
}

static size_t silu_acc_offset(int64_t n) {
  return silu_f32_offset(n) + sizeof(float) * (size_t)silu_blocks(n) * kH * kH;
}

extern "C" size_t spic_silu_scratch_bytes(int64_t n) {
  // [blocks][1 + P] partials, the reduced row, candidate parameters, finalize sync words,
  // then the per-CTA dW2 partials as float [blocks][H * H] (the rows' W2 range is unused),
  // then the per-CTA flushed TMEM accumulators float [blocks][2][H * H]
  return silu_acc_offset(n) + sizeof(float) * (size_t)silu_blocks(n) * 2 * kH * kH;
}

extern "C" int64_t spic_silu_row_offset(int64_t n) {
  return (int64_t)(sizeof(double) * (size_t)silu_blocks(n) * (1 + (size_t)silu_params(kH)));
}

static int silu_launch(int mode, const float* params32, int32_t H, const SiluInputs& in,
                       int64_t n, float x_scale, float* sw_out, double* part, cudaStream_t st) {
  if (H != kH) return SPIC_ERR_UNSUPPORTED;
  if (n < 1 || !(x_scale > 0.f)) return SPIC_ERR_ARG;
  if (in.xv ? !in.sw : (!in.x || !in.v || !in.w)) return SPIC_ERR_ARG;
  if (mode == 2 && (in.xv || !in.Z)) return SPIC_ERR_ARG;
  const int blocks = silu_blocks(n);
  const float L = 1.0f / x_scale;
#define SPIC_SILU_LAUNCH(MD)                                                                   \
  do {                                                                                         \
    cudaFuncSetAttribute(k_silu<MD>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                         (int)kSiluSmem);                                                      \
    k_silu<MD><<<blocks, kNT, kSiluSmem, st>>>(                                                \
        params32, in, n, x_scale, L, (float4*)sw_out, part,                                    \
        part ? (float*)((char*)part + silu_f32_offset(n)) : nullptr,                           \
        part ? (float*)((char*)part + silu_acc_offset(n)) : nullptr);                          \
  } while (0)
  if (mode == 0) SPIC_SILU_LAUNCH(0);
  else if (mode == 1) SPIC_SILU_LAUNCH(1);
  else SPIC_SILU_LAUNCH(2);
#undef SPIC_SILU_LAUNCH
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

// Deterministic column sums of the per-CTA partial rows (one warp per column, float64): the
// dW2 columns come from the float block, the rest from the float64 rows.
__global__ void k_silu_reduce_cols(const double* __restrict__ part, const float* __restrict__ pw2,
                                   int rows, int64_t width, int64_t oW2, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t col = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (col >= width) return;
  double s = 0.0;
  if (col >= oW2 && col < oW2 + kH * kH) {
    const int64_t c = col - oW2;
    for (int r = lane; r < rows; r += 32) s += (double)pw2[(size_t)r * kH * kH + c];
  } else {
    for (int r = lane; r < rows; r += 32) s += part[(size_t)r * width + col];
  }
  s = warp_sum(s);
  if (lane == 0) out[col] = s;
}

// Same column sums with the rows spread over 4 thread groups per column: consecutive threads
// take consecutive columns (each warp reads one 128/256-B row segment per load instead of 32
// rows of one column), each group sums rows q, q + 4, ... in order and the four group sums
// are added in a fixed order: deterministic.
__global__ void __launch_bounds__(256) k_silu_reduce_cols4(
    const double* __restrict__ part, const float* __restrict__ pw2, int rows, int64_t width,
    int64_t oW2, double* __restrict__ out) {
  __shared__ double red[4][64];
  const int cl = threadIdx.x & 63, q = threadIdx.x >> 6;
  const int64_t col = blockIdx.x * (int64_t)64 + cl;
  double s = 0.0;
  if (col < width) {
    if (col >= oW2 && col < oW2 + kH * kH) {
      const float* src = pw2 + (col - oW2);
#pragma unroll 4
      for (int r = q; r < rows; r += 4) s += (double)src[(size_t)r * kH * kH];
    } else {
      const double* src = part + col;
#pragma unroll 4
      for (int r = q; r < rows; r += 4) s += src[(size_t)r * width];
    }
  }
  red[q][cl] = s;
  __syncthreads();
  if (q == 0 && col < width) out[col] = (red[0][cl] + red[1][cl]) + (red[2][cl] + red[3][cl]);
}

static int silu_reduce(int64_t n, void* scratch, cudaStream_t st) {
  const int rows = silu_blocks(n);
  const int64_t width = 1 + silu_params(kH);
  double* part = (double*)scratch;
  const int64_t oW2 = 1 + 4 * kH + kH;
  const char* e = getenv("SPIC_SILU_REDUCE");  // "1": one warp per column (A/B)
  if (e && e[0] == '1')
    k_silu_reduce_cols<<<(unsigned)((width + 7) / 8), 256, 0, st>>>(
        part, (const float*)((char*)scratch + silu_f32_offset(n)), rows, width, oW2,
        part + (size_t)rows * width);
  else
    k_silu_reduce_cols4<<<(unsigned)((width + 63) / 64), 256, 0, st>>>(
        part, (const float*)((char*)scratch + silu_f32_offset(n)), rows, width, oW2,
        part + (size_t)rows * width);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_silu_forward(const float* params32, int32_t H, const float* xv,
                                 const float* sw, int64_t n, float x_scale, float* sw_out,
                                 void* stream) {
  if (n < 0) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;  // empty ensemble: nothing to score
  if (!sw_out || !xv) return SPIC_ERR_ARG;
  SiluInputs in{(const float4*)xv, (const float4*)sw, nullptr, nullptr, 0, nullptr, nullptr, 0,
                nullptr, 0.f};
  return silu_launch(0, params32, H, in, n, x_scale, sw_out, nullptr, (cudaStream_t)stream);
}

extern "C" int spic_silu_ism_partials(const float* params32, int32_t H, const float* xv,
                                      const float* sw, int64_t n, float x_scale, void* scratch,
                                      size_t scratch_bytes, void* stream) {
  if (n >= 1 && scratch_bytes < spic_silu_scratch_bytes(n)) return SPIC_ERR_SCRATCH;
  if (!xv) return SPIC_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SiluInputs in{(const float4*)xv, (const float4*)sw, nullptr, nullptr, 0, nullptr, nullptr, 0,
                nullptr, 0.f};
  int rc = silu_launch(1, params32, H, in, n, x_scale, nullptr, (double*)scratch, st);
  return rc != SPIC_OK ? rc : silu_reduce(n, scratch, st);
}

extern "C" int spic_silu_mse_partials(const float* params32, int32_t H, const float* x,
                                      const float* v, int64_t ldv, const float* w, int64_t n,
                                      float x_scale, const float* Z, int64_t ldz,
                                      const int32_t* idx, double inv_wsum, void* scratch,
                                      size_t scratch_bytes, void* stream) {
  if (n >= 1 && scratch_bytes < spic_silu_scratch_bytes(n)) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  SiluInputs in{nullptr, nullptr, x, v, ldv, w, Z, ldz, idx, (float)inv_wsum};
  int rc = silu_launch(2, params32, H, in, n, x_scale, nullptr, (double*)scratch, st);
  return rc != SPIC_OK ? rc : silu_reduce(n, scratch, st);
}

extern "C" int spic_silu_finalize(void* scratch, int64_t n, int32_t H, int32_t mse,
                                  double* params64, double* m, double* v2, double* opt_state,
                                  double beta1, double beta2, double eps, double weight_decay,
                                  int32_t reset_lr, int32_t apply_step, float* params32,
                                  double* grads_out, double* loss_out, int32_t* flags,
                                  void* stream) {
  if (H != kH) return SPIC_ERR_UNSUPPORTED;
  if (n < 1) return SPIC_ERR_ARG;
  const int64_t P = silu_params(kH);
  double* row = (double*)((char*)scratch + spic_silu_row_offset(n));
  int32_t* sync = (int32_t*)(row + 1 + P + P);
  cudaStream_t st = (cudaStream_t)stream;
  const char* fv = getenv("SPIC_SILU_FINALIZE");  // "1": the single-CTA kernel (A/B tests)
  if (fv && fv[0] == '1') {
    k_silu_finalize<<<1, 1024, 0, st>>>(row, P, mse != 0, params64, m, v2, opt_state, beta1, beta2,
                                        eps, weight_decay, reset_lr, apply_step, params32,
                                        grads_out, loss_out, row + 1 + P, flags);
  } else {
    cudaMemsetAsync(sync, 0, sizeof(int32_t), st);  // the barrier ticket
    // cooperative launch: the runtime guarantees the kSiluFinCTAs CTAs are co-resident (or
    // fails the launch) so the spin barrier cannot deadlock behind other work holding SMs;
    // cudaLaunchKernelEx with the cooperative attribute is stream-capturable
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kSiluFinCTAs);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool mse_b = mse != 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_silu_finalize_mc, row, P, mse_b, params64, m, v2,
                                       opt_state, beta1, beta2, eps, weight_decay, (int)reset_lr,
                                       (int)apply_step, params32, grads_out, loss_out,
                                       row + 1 + P, flags, sync);
    if (e != cudaSuccess) return SPIC_ERR_CUDA - (int)e;
  }
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_umma_selftest(const float* W, const float* X, const float* Y, float* D1,
                                  float* D2, float* D3, void* stream) {
  cudaFuncSetAttribute(k_umma_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kSiluSmem);
  k_umma_selftest<<<1, 128, kSiluSmem, (cudaStream_t)stream>>>(W, X, Y, D1, D2, D3);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}
