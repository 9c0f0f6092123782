// pairs.cuh — shared machinery of the cell-stencil pair kernels (Landau collision, blob KDE):
// the j-window of a target tile (up to 3 contiguous segments of the cell-sorted records,
// culled to the sub-cells within eta of the tile), the per-cell target-tile table, and the
// bulk-copy (cp.async.bulk + mbarrier) helpers that stream j-records into shared memory.
#pragma once
#include <cstdlib>

#include "common.cuh"

namespace spic {

constexpr int kLandauNT = 128;  // threads per CTA
constexpr int kLandauR = 2;     // targets per thread
constexpr int kLandauTI = kLandauNT * kLandauR;
constexpr int kLandauTJ = 256;  // records per stage
constexpr int kLandauStages = 3;
constexpr float kEps2 = 1e-24f;  // ref: kernels.py:7 EPS_Z^2, collision.py:100

// ---- bulk copy / mbarrier helpers (sm_90+; UBLKCP + SYNCS in SASS) ----------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- j-window: up to 3 segments of sorted positions, each with an x shift ----------------
struct Window {
  int start[3], len[3];
  float shift[3];
  int nseg;
};

// Tile q of TJ records inside split [jlo, jhi) of the concatenated window.
struct TileDesc {
  int pos, cnt;
  float shift;
};

__device__ __forceinline__ int window_tiles(const Window& w, int jlo, int jhi) {
  int off = 0, nt = 0;
  for (int s = 0; s < w.nseg; ++s) {
    int a = max(jlo, off), b = min(jhi, off + w.len[s]);
    if (b > a) nt += (b - a + kLandauTJ - 1) / kLandauTJ;
    off += w.len[s];
  }
  return nt;
}

__device__ __forceinline__ TileDesc window_tile(const Window& w, int jlo, int jhi, int q) {
  int off = 0;
  TileDesc d{0, 0, 0.f};
  for (int s = 0; s < w.nseg; ++s) {
    int a = max(jlo, off), b = min(jhi, off + w.len[s]);
    if (b > a) {
      int nt = (b - a + kLandauTJ - 1) / kLandauTJ;
      if (q < nt) {
        int lo = a + q * kLandauTJ;
        d.pos = w.start[s] + (lo - off);
        d.cnt = min(kLandauTJ, b - lo);
        d.shift = w.shift[s];
        return d;
      }
      q -= nt;
    }
    off += w.len[s];
  }
  return d;
}

// Builds the window of cell c for the target range [t0, t1) (sorted positions).
static __device__ Window build_window(const int32_t* __restrict__ cell_start,
                               const int32_t* __restrict__ sub_start, int M, int S, int c, int t0,
                               int t1, float L) {
  Window w;
  w.nseg = 0;
  if (M <= 2) {  // deduplicated stencil, per-pair minimum image
    int cells[2] = {c, (c + 1) % M};
    int nc = M == 1 ? 1 : 2;
    for (int k = 0; k < nc; ++k) {
      w.start[w.nseg] = cell_start[cells[k]];
      w.len[w.nseg] = cell_start[cells[k] + 1] - cell_start[cells[k]];
      w.shift[w.nseg] = 0.f;
      ++w.nseg;
    }
    return w;
  }
  // local sub-cell coordinates u in [0, 3S): cell c-1 -> [0,S), c -> [S,2S), c+1 -> [2S,3S)
  int ulo = 0, uhi = 3 * S - 1;
  if (S > 1 && sub_start) {
    const int32_t* ss = sub_start + (size_t)c * S;
    int a = 0, b = 0;
    for (int k = 1; k < S; ++k) {  // S <= 64: linear scan is fine (one thread)
      if (ss[k] <= t0) a = k;
      if (ss[k] <= t1 - 1) b = k;
    }
    // cell c-1 from sub-cell a, cell c+1 through sub-cell b: beyond them every pair is
    // farther than eta apart (see k_sym_tiles)
    ulo = a;
    uhi = 2 * S + b;
  }
  for (int d = -1; d <= 1; ++d) {
    int u0 = (d + 1) * S, u1 = u0 + S - 1;
    int lo = max(ulo, u0) - u0, hi = min(uhi, u1) - u0;
    if (hi < lo) continue;
    int cd = c + d;
    float shift = cd < 0 ? -L : (cd >= M ? L : 0.f);
    cd = (cd + M) % M;
    int p0, p1;
    if (S > 1 && sub_start) {
      p0 = sub_start[(size_t)cd * S + lo];
      p1 = sub_start[(size_t)cd * S + hi + 1];
    } else {
      p0 = cell_start[cd];
      p1 = cell_start[cd + 1];
    }
    if (p1 > p0) {
      w.start[w.nseg] = p0;
      w.len[w.nseg] = p1 - p0;
      w.shift[w.nseg] = shift;
      ++w.nseg;
    }
  }
  return w;
}

static __global__ void k_landau_tiles(const int32_t* __restrict__ cell_start, int M, int TI,
                                      int32_t* __restrict__ tile_start, int c_lo = 0,
                                      int c_hi = 1 << 30) {
  // single CTA exclusive scan of ceil(count_c / TI)
  __shared__ int ws[33];
  int carry = 0;
  for (int base = 0; base < M; base += blockDim.x) {
    int c = base + threadIdx.x;
    // target cells outside [c_lo, c_hi) (halo cells of a domain rank) get no tiles
    int v = (c < M && c >= c_lo && c < c_hi) ? (cell_start[c + 1] - cell_start[c] + TI - 1) / TI : 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      int s = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0;
      int si = s;
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, si, o);
        if (lane >= o) si += t;
      }
      ws[lane] = si - s;
      if (lane == 31) ws[32] = si;
    }
    __syncthreads();
    if (c < M) tile_start[c] = carry + ws[wid] + inc - v;
    carry += ws[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tile_start[M] = carry;
    tile_start[M + 1] = 0;  // work-queue counter of the persistent pair kernels
  }
}

// j-split of a pair kernel: choose nsplit so the (tile, split) CTA count fills whole waves
// of the resident CTA slots (4 per SM); wave quantisation, not the pair count, sets the tail
static inline int pair_nsplit_slots(int64_t n, int M, int TI, int resident) {
  const double tiles = (double)(n / TI) + 0.5 * M > 1.0 ? (double)(n / TI) + 0.5 * M : 1.0;
  const double slots = (double)resident;
  const int64_t window = 2 * n / (M > 1 ? M : 1);  // records in a culled j-window (approx.)
  // at least min_split j-records per split (SPIC_PAIR_MIN_SPLIT, A/B): 128 lets small cells
  // (config 0: ~2k-record windows) split far enough to fill the SMs (c0 pair 0.241 -> 0.172 ms
  // against 1024); windows of the larger configs hit the 16-split cap either way
  static const int min_split = [] {
    const char* e = getenv("SPIC_PAIR_MIN_SPLIT");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : 128;
  }();
  int cap = (int)(window / min_split);
  cap = cap < 1 ? 1 : (cap > 16 ? 16 : cap);
  int best = 1;
  double best_eff = -1.0;
  for (int ns = 1; ns <= cap; ++ns) {
    const double waves = tiles * ns / slots;
    double eff = waves < 1.0 ? waves : waves / ceil(waves);
    eff -= 0.004 * (ns - 1);  // each split re-reads targets and writes a partial
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = ns;
    }
  }
  return best;
}

static inline int pair_nsplit(int64_t n, int M, int TI) {
  return pair_nsplit_slots(n, M, TI, 4 * kNumSMs);
}

}  // namespace spic
