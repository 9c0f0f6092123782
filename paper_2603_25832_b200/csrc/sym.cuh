// sym.cuh — shared machinery of the antisymmetric / symmetric (unordered-pair) pair kernels
// (landau_sym.cu, blob_sym.cu): the forward-window enumeration of unordered pairs, the tile
// table (k_sym_tiles), the slot layout of the streamed-side sums and the warp reduce-scatter.
#pragma once
#include <algorithm>
#include <cstdlib>

#include "f32x2.cuh"
#include "pairs.cuh"

namespace spic {

constexpr int kSymTJ = 256;     // records per stage
constexpr int kSymStages = 3;

struct SymMeta {
  int len1;  // own-cell forward length ce - t1; -1 marks a halo tile (seg2 only)
  int len2;  // next-cell prefix length
};

// Single CTA: tile_start[0..M] (targets tiles per cell, incl. the halo cell c_lo-1 of a
// partial range), per-tile SymMeta, slot offsets off[0..T], the symmetric-path flag.
__global__ void __launch_bounds__(1024) k_sym_tiles(
    const int32_t* __restrict__ cell_start, const int32_t* __restrict__ sub_start, int M, int S,
    int TI, int c_lo, int c_hi, int64_t cap_slots, int32_t* __restrict__ tile_start,
    SymMeta* __restrict__ meta, int64_t* __restrict__ off, int32_t* __restrict__ symflag);

// j-window tile with its kind: two-sided tiles also carry the slot offset of their first
// record relative to off[tile]
struct SymTileDesc {
  int pos, cnt, wofs;
  float shift;
  bool two;
};

struct SymWindow {
  int start[3], len[3], wofs[3];
  float shift[3];
  bool two[3];
  int nseg;
};

__device__ __forceinline__ int sym_window_tiles(const SymWindow& w, int jlo, int jhi) {
  int o = 0, nt = 0;
  for (int s = 0; s < w.nseg; ++s) {
    const int a = max(jlo, o), b = min(jhi, o + w.len[s]);
    if (b > a) nt += (b - a + kSymTJ - 1) / kSymTJ;
    o += w.len[s];
  }
  return nt;
}

__device__ __forceinline__ SymTileDesc sym_window_tile(const SymWindow& w, int jlo, int jhi,
                                                       int q) {
  int o = 0;
  SymTileDesc d{0, 0, 0, 0.f, false};
  for (int s = 0; s < w.nseg; ++s) {
    const int a = max(jlo, o), b = min(jhi, o + w.len[s]);
    if (b > a) {
      const int nt = (b - a + kSymTJ - 1) / kSymTJ;
      if (q < nt) {
        const int lo = a + q * kSymTJ;
        d.pos = w.start[s] + (lo - o);
        d.cnt = min(kSymTJ, b - lo);
        d.shift = w.shift[s];
        d.two = w.two[s];
        d.wofs = w.wofs[s] + (lo - o);
        return d;
      }
      q -= nt;
    }
    o += w.len[s];
  }
  return d;
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// Window of tile `tile` (cell c, targets [t0, t1)): with the symmetric path on, the diagonal
// block (one-sided), the rest of cell c and the culled prefix of cell c+1 (two-sided); else
// the ordered full stencil (one-sided).
__device__ __forceinline__ SymWindow sym_build_window(
    bool sym, const SymMeta* __restrict__ meta, const int32_t* __restrict__ cell_start,
    const int32_t* __restrict__ sub_start, int M, int S, int c, int tile, int t0, int t1, float L,
    bool minimg) {
  SymWindow win;
  win.nseg = 0;
  if (sym) {
    const SymMeta m = meta[tile];
    if (m.len1 >= 0) {
      win.start[0] = t0; win.len[0] = t1 - t0; win.shift[0] = 0.f; win.two[0] = false;
      win.wofs[0] = 0;
      win.start[1] = t1; win.len[1] = m.len1; win.shift[1] = 0.f; win.two[1] = true;
      win.wofs[1] = 0;
      win.nseg = 2;
    }
    const int cn = c + 1 == M ? 0 : c + 1;
    const int k = win.nseg;
    win.start[k] = cell_start[cn]; win.len[k] = m.len2;
    win.shift[k] = (c + 1 == M && !minimg) ? L : 0.f; win.two[k] = true;
    win.wofs[k] = max(m.len1, 0);
    win.nseg = k + 1;
  } else {
    const Window w = build_window(cell_start, sub_start, M, S, c, t0, t1, L);
    for (int s = 0; s < w.nseg; ++s) {
      win.start[s] = w.start[s]; win.len[s] = w.len[s]; win.shift[s] = w.shift[s];
      win.two[s] = false; win.wofs[s] = 0;
    }
    win.nseg = w.nseg;
  }
  return win;
}

// Warp reduce-scatter of NC per-record sums over 8 records read in the XOR order
// (lane l holds record k ^ m_l, m_l = (l >> 2) & 7): afterwards every lane holds the warp sums
// of record m_l in P[c][0] (xor-16/8/4 exchanges need no selects, xor-2/1 butterflies finish).
template <int NC>
__device__ __forceinline__ void sym_reduce_scatter8(float (&P)[NC][8]) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < NC; ++c) P[c][k] += __shfl_xor_sync(0xffffffffu, P[c][k + 4], 16);
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int c = 0; c < NC; ++c) P[c][k] += __shfl_xor_sync(0xffffffffu, P[c][k + 2], 8);
#pragma unroll
  for (int c = 0; c < NC; ++c) P[c][0] += __shfl_xor_sync(0xffffffffu, P[c][1], 4);
#pragma unroll
  for (int c = 0; c < NC; ++c) P[c][0] += __shfl_xor_sync(0xffffffffu, P[c][0], 2);
#pragma unroll
  for (int c = 0; c < NC; ++c) P[c][0] += __shfl_xor_sync(0xffffffffu, P[c][0], 1);
}

// Same over 4 records (lane l holds record k ^ m_l, m_l = (l >> 3) & 3): xor-16/8 exchanges
// without selects, then xor-4/2/1 butterflies; every lane ends with the warp sums of record
// m_l in P[c][0]. Half the live partials of the 8-record form for ~1.3x its shuffles.
template <int NC>
__device__ __forceinline__ void sym_reduce_scatter4(float (&P)[NC][4]) {
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int c = 0; c < NC; ++c) P[c][k] += __shfl_xor_sync(0xffffffffu, P[c][k + 2], 16);
#pragma unroll
  for (int c = 0; c < NC; ++c) P[c][0] += __shfl_xor_sync(0xffffffffu, P[c][1], 8);
#pragma unroll
  for (int o = 4; o >= 1; o >>= 1)
#pragma unroll
    for (int c = 0; c < NC; ++c) P[c][0] += __shfl_xor_sync(0xffffffffu, P[c][0], o);
}

// the fold's walk over a record's slots: own-cell tiles before its tile, then the tiles of
// cell c-1 whose seg2 reaches it; calls f(slot) in that fixed order
template <typename F>
__device__ __forceinline__ void sym_for_slots(int64_t p, const int32_t* __restrict__ cell_start,
                                              const int32_t* __restrict__ tile_start,
                                              const SymMeta* __restrict__ meta,
                                              const int64_t* __restrict__ off, int M, int TI,
                                              F&& f) {
  int lo = 0, hi = M;  // cell of p: largest c with cell_start[c] <= p
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(cell_start + mid) <= p) lo = mid; else hi = mid;
  }
  const int c = lo;
  const int rel = (int)(p - cell_start[c]);
  const int tc = tile_start[c];
  const int tp = tc + rel / TI;
  for (int t = tc; t < tp; ++t) f(off[t] + (rel - (t - tc + 1) * TI));
  const int cm = c == 0 ? M - 1 : c - 1;
  for (int t = tile_start[cm]; t < tile_start[cm + 1]; ++t) {
    const SymMeta m = meta[t];
    if (rel < m.len2) f(off[t] + max(m.len1, 0) + rel);
  }
}

// Layout of the symmetric path's scratch (all offsets 256-aligned):
//   tile_start i32[M+2] | meta SymMeta[Tmax] | off i64[Tmax+1] | flag i32 | Upart f32[nsplit][nc][n]
//   | Jslot f32[cap][nc]   (nc = 3 for the Landau sum, 4 for the blob (den, mu) sums)
struct SymScratch {
  int32_t* tile_start;
  SymMeta* meta;
  int64_t* off;
  int32_t* flag;
  float* Upart;
  float* Jslot;
  int64_t cap;
  size_t bytes;
};

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// m_occ: the cells the records occupy (M for a whole-grid call; a domain rank's target range
// plus its halo cells for a range call), which sets the per-cell size estimate
static inline SymScratch sym_layout(void* base, int64_t n, int M, int nsplit, int TI, int nc = 3,
                                    int m_occ = 0) {
  SymScratch s{};
  if (m_occ <= 0 || m_occ > M) m_occ = M;
  const int64_t Tmax = n / TI + M + 2;
  // slot estimate for a near-uniform ensemble: each tile's forward window ~ one cell plus a
  // sub-cell; 1.3x headroom (an exceeding ensemble runs the ordered path, see k_sym_tiles)
  const int64_t ncell = n / std::max(m_occ, 1);
  const int64_t Tocc = n / TI + m_occ + 2;
  int64_t cap = (int64_t)(1.3 * (double)Tocc * (double)(ncell + 2 * TI)) + 4096;
  // at most 16 GiB of slots (a near-uniform n = 2^24, M = 1024 ensemble needs ~7 GB); a
  // degenerate ensemble (e.g. one huge cell) beyond that takes the ordered path
  const int64_t cap_max = ((int64_t)16 << 30) / (int64_t)(sizeof(float) * nc);
  cap = std::min(cap, cap_max);
  if (const char* e = getenv("SPIC_SYM_CAP_SLOTS")) cap = atoll(e);  // tests: force the fallback
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o = align256(o + b);
    return (char*)base + at;
  };
  s.tile_start = (int32_t*)take(sizeof(int32_t) * (M + 2));
  s.meta = (SymMeta*)take(sizeof(SymMeta) * Tmax);
  s.off = (int64_t*)take(sizeof(int64_t) * (Tmax + 1));
  s.flag = (int32_t*)take(sizeof(int32_t) * 8);
  s.Upart = (float*)take(sizeof(float) * (size_t)nsplit * nc * n);
  s.Jslot = (float*)take(sizeof(float) * (size_t)cap * nc);
  s.cap = cap;
  s.bytes = o;
  return s;
}

}  // namespace spic
