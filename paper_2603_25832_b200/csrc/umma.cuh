// umma.cuh — tcgen05 (5th-gen tensor core) helpers for the 128x128 split-BF16 GEMMs of the
// SiLU score network (silu.cu).
//
// Operand tiles are 128 x 128 bf16 in shared memory, SWIZZLE_128B: two 64-column halves of
// 16 KB, row r at r*128 B inside a half, 16-B chunk index XOR (r & 7). One physical tile is
// read either K-major (rows = M/N index, cols = K) or MN-major (rows = K, cols = M/N), so a
// single copy of an activation block serves as a K-major B operand in one GEMM and an
// MN-major A/B operand in the transposed GEMMs (the backward pass and the weight gradient).
// Accumulators are float32 in TMEM (lane = M row, column = N).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace spic {
namespace umma {

constexpr uint32_t kTileBytes = 32768;  // 128 x 128 bf16

// byte offset of element (r, c) inside a tile
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
  return (uint32_t)((c >> 6) * 16384 + r * 128 + ((((c >> 3) & 7) ^ (r & 7)) << 4) + (c & 7) * 2);
}

// shared-memory matrix descriptor: start, leading/stride byte offsets, version 1 (sm_100),
// layout type 2 = SWIZZLE_128B
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// A tile of R rows x 128 bf16 columns is two 64-column halves of R * 128 B ("half" below;
// 16 KB for R = 128). K-major view; K-step ks covers columns 16ks..16ks+15 (32 B inside a
// 128-B swizzle row)
__device__ __forceinline__ uint64_t desc_k(uint32_t tile, int ks, uint32_t half = 16384) {
  return sdesc(tile + (uint32_t)(ks >> 2) * half + (uint32_t)((ks & 3) * 32), 16, 1024);
}
// MN-major view; K-step ks covers rows 16ks..16ks+15; MN groups of 64 are the two halves
__device__ __forceinline__ uint64_t desc_mn(uint32_t tile, int ks, uint32_t half = 16384) {
  return sdesc(tile + (uint32_t)(ks * 2048), half, 1024);
}

// byte offset of element (r, c) inside an R-row tile (half = R * 128)
__device__ __forceinline__ uint32_t tile_off_h(int r, int c, uint32_t half) {
  return (uint32_t)(c >> 6) * half +
         (uint32_t)(r * 128 + ((((c >> 3) & 7) ^ (r & 7)) << 4) + (c & 7) * 2);
}

// ---- activation tiles: no-swizzle ("interleaved") core-matrix layout --------------------
// The X / Y tiles hold P particle columns x 128 hidden units as 8 x 8 core matrices of
// 128 contiguous bytes: element (p, h) at
//     (p / 8) * kActGroup + (h / 8) * 128 + (h % 8) * 16 + (p % 8) * 2.
// A thread that owns hidden unit h writes 8 consecutive particles with ONE 16-byte store (and
// a warp's 32 stores cover 512 contiguous bytes, conflict free), instead of 8 two-byte stores
// into a particle-major swizzled tile. The same bytes are an MN-major operand over
// (N = particles, K = h): LBO = 128 between the 8-wide K groups, SBO = kActGroup between the
// 8-particle groups; and a K-major operand over (M or N = h, K = particles): LBO = kActGroup,
// SBO = 128 (canonical INTERLEAVE layouts of the sm_100 shared-memory descriptor).
constexpr uint32_t kActGroup = 2048;  // bytes per group of 8 particles (16 K-groups x 128 B)

__device__ __forceinline__ uint64_t sdesc_i(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // layout type 0: no swizzle
}

// operand views of the split-BF16 GEMMs
enum View {
  kWK = 0,    // 128-row SWIZZLE_128B tile read K-major (rows = M, cols = K)
  kWMN = 1,   // the same tile read MN-major (rows = K, cols = M)
  kActMN = 2, // activation tile as (N = particles, K = h), MN-major; K-step = 16 hidden units
  kActK = 3   // activation tile as (M / N = h, K = particles), K-major; K-step = 16 particles
};
template <int V>
__device__ __forceinline__ uint64_t view_desc(uint32_t tile) {
  if constexpr (V == kWK) return desc_k(tile, 0, 16384);
  else if constexpr (V == kWMN) return desc_mn(tile, 0, 16384);
  else if constexpr (V == kActMN) return sdesc_i(tile, 128, kActGroup);
  else return sdesc_i(tile, kActGroup, 128);
}
template <int V>
__host__ __device__ constexpr uint64_t view_step(int ks) {  // start-address increment, 16-B units
  if constexpr (V == kWK) return (uint64_t)(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4);
  else if constexpr (V == kWMN) return (uint64_t)(ks * 2048 >> 4);
  else if constexpr (V == kActMN) return (uint64_t)(ks * 256 >> 4);
  else return (uint64_t)(ks * 2 * kActGroup >> 4);
}
__host__ __device__ constexpr uint32_t view_mn(int V) { return (V == kWMN || V == kActMN) ? 1u : 0u; }

// instruction descriptor: kind::f16, A/B bf16, D f32, M = 128, N, operand majors
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t a_mn, uint32_t b_mn, uint32_t N = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
         ((128u >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Warp-wide issue: every lane of the issuing warp executes the same (warp-uniform) instruction
// stream and elect.sync picks the one lane that issues. Compared with `if (lane == 0) mma(...)`
// this keeps the control flow convergent, so the operands stay in uniform registers instead of
// a per-instruction ELECT / R2UR / BRA.U.ANY waterfall (the issue rate, not the tensor pipe,
// bounded the small-N GEMMs when the issuing warp shares its scheduler with busy warps).
__device__ __forceinline__ void mma_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// D[128 x N] (+)= A * B over K = 16 * KSTEPS with split-BF16 operands:
// Ahi*Bhi + Ahi*Blo + Alo*Bhi (~2^-16 relative per product; float32 accumulation in TMEM).
// Operand addresses are tile (sub-)block starts. Issued by one thread. The four base
// descriptors are built once; every K-step only adds a constant to their start-address
// field (addresses stay below 2^18, so the 14-bit field never carries).
template <bool A_MN, bool B_MN, int N = 128, int KSTEPS = 8, uint32_t AH = 16384,
          uint32_t BH = 16384, bool WARP = false>
__device__ __forceinline__ void gemm_split(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo,
                                           uint32_t b_hi, uint32_t b_lo, bool accumulate) {
  constexpr uint32_t id = idesc_bf16(A_MN ? 1u : 0u, B_MN ? 1u : 0u, (uint32_t)N);
  const uint64_t ah0 = A_MN ? desc_mn(a_hi, 0, AH) : desc_k(a_hi, 0, AH);
  const uint64_t al0 = A_MN ? desc_mn(a_lo, 0, AH) : desc_k(a_lo, 0, AH);
  const uint64_t bh0 = B_MN ? desc_mn(b_hi, 0, BH) : desc_k(b_hi, 0, BH);
  const uint64_t bl0 = B_MN ? desc_mn(b_lo, 0, BH) : desc_k(b_lo, 0, BH);
#pragma unroll
  for (int ks = 0; ks < KSTEPS; ++ks) {
    const uint64_t ao = A_MN ? (uint64_t)(ks * 2048 >> 4)
                             : (uint64_t)(((ks >> 2) * AH + (ks & 3) * 32) >> 4);
    const uint64_t bo = B_MN ? (uint64_t)(ks * 2048 >> 4)
                             : (uint64_t)(((ks >> 2) * BH + (ks & 3) * 32) >> 4);
    if (WARP) {
      mma_elect(d_tmem, ah0 + ao, bh0 + bo, id, (accumulate || ks > 0) ? 1u : 0u);
      mma_elect(d_tmem, ah0 + ao, bl0 + bo, id, 1u);
      mma_elect(d_tmem, al0 + ao, bh0 + bo, id, 1u);
    } else {
      mma(d_tmem, ah0 + ao, bh0 + bo, id, (accumulate || ks > 0) ? 1u : 0u);
      mma(d_tmem, ah0 + ao, bl0 + bo, id, 1u);
      mma(d_tmem, al0 + ao, bh0 + bo, id, 1u);
    }
  }
}

// The same over operand views (see View): warp-wide issue, descriptors built once per GEMM.
template <int AV, int BV, int N, int KSTEPS>
__device__ __forceinline__ void gemm_split_v(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo,
                                             uint32_t b_hi, uint32_t b_lo, bool accumulate) {
  constexpr uint32_t id = idesc_bf16(view_mn(AV), view_mn(BV), (uint32_t)N);
  const uint64_t ah0 = view_desc<AV>(a_hi), al0 = view_desc<AV>(a_lo);
  const uint64_t bh0 = view_desc<BV>(b_hi), bl0 = view_desc<BV>(b_lo);
#pragma unroll
  for (int ks = 0; ks < KSTEPS; ++ks) {
    const uint64_t ao = view_step<AV>(ks), bo = view_step<BV>(ks);
    mma_elect(d_tmem, ah0 + ao, bh0 + bo, id, (accumulate || ks > 0) ? 1u : 0u);
    mma_elect(d_tmem, ah0 + ao, bl0 + bo, id, 1u);
    mma_elect(d_tmem, al0 + ao, bh0 + bo, id, 1u);
  }
}

// mbarrier parity wait that traps (instead of hanging the GPU) if the MMA never completes
__device__ __forceinline__ void wait_mma(uint64_t* bar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  for (uint32_t spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
    if (ok) return;
    if (spin > (1u << 24)) __trap();
  }
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// TMEM allocation (whole warp) / release
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// 32 consecutive float32 columns of this thread's TMEM lane (warp w reads lanes 32(w%4)..)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&f)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(r[i]);
}

// 8 consecutive float32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&f)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[i]);
}

// 16 consecutive float32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&f)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(r[i]);
}

// 12 consecutive float32 columns (three x4 loads, 4-column aligned) of this thread's lane
__device__ __forceinline__ void tmem_ld12(uint32_t taddr, float (&f)[16]) {
  uint32_t r[12];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%12];\n"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [%13];\n"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [%14];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
      : "r"(taddr), "r"(taddr + 4), "r"(taddr + 8)
      : "memory");
#pragma unroll
  for (int i = 0; i < 12; ++i) f[i] = __uint_as_float(r[i]);
#pragma unroll
  for (int i = 12; i < 16; ++i) f[i] = 0.f;
}

// two 12-column slices of this thread's lane with one wait (the second load's latency hides
// behind the first's)
__device__ __forceinline__ void tmem_ld12x2(uint32_t ta, uint32_t tb, float (&f)[16], float (&g)[16]) {
  uint32_t r[24];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%24];\n"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [%25];\n"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [%26];\n"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12,%13,%14,%15}, [%27];\n"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16,%17,%18,%19}, [%28];\n"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%20,%21,%22,%23}, [%29];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23])
      : "r"(ta), "r"(ta + 4), "r"(ta + 8), "r"(tb), "r"(tb + 4), "r"(tb + 8)
      : "memory");
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    f[i] = __uint_as_float(r[i]);
    g[i] = __uint_as_float(r[12 + i]);
  }
#pragma unroll
  for (int i = 12; i < 16; ++i) f[i] = g[i] = 0.f;
}

// split x into bf16 hi + lo (x ~= hi + lo to ~2^-17 relative) and store both tiles
__device__ __forceinline__ void store_split(uint8_t* hi_tile, uint8_t* lo_tile, int r, int c,
                                            float x) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
  const uint32_t o = tile_off(r, c);
  *reinterpret_cast<__nv_bfloat16*>(hi_tile + o) = h;
  *reinterpret_cast<__nv_bfloat16*>(lo_tile + o) = l;
}

// Eight consecutive columns c0..c0+7 (c0 % 8 == 0) of row r: one 16-B swizzle chunk per tile.
__device__ __forceinline__ void store_split8(uint8_t* hi_tile, uint8_t* lo_tile, int r, int c0,
                                             const float (&x)[8]) {
  uint32_t hw[4], lw[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * k], x[2 * k + 1]);
    const float2 hf = __bfloat1622float2(h2);
    const __nv_bfloat162 l2 = __floats2bfloat162_rn(x[2 * k] - hf.x, x[2 * k + 1] - hf.y);
    hw[k] = *reinterpret_cast<const uint32_t*>(&h2);
    lw[k] = *reinterpret_cast<const uint32_t*>(&l2);
  }
  const uint32_t o = tile_off(r, c0);
  *reinterpret_cast<uint4*>(hi_tile + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  *reinterpret_cast<uint4*>(lo_tile + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

}  // namespace umma
}  // namespace spic
