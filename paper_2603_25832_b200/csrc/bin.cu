// bin.cu — bit-exact cell binning: a stable, deterministic counting sort by
// key = (cell, sub-cell) with the fused gather into cell-sorted float4 records.
//
// Replaces Grid.cell_of (ref: pic.py:27-30) and build_cell_index (ref: collision.py:39-46,
// np.argsort(kind="stable") + searchsorted). With S == 1 the permutation equals the
// reference's concat(bins) exactly; with S > 1 particles are additionally ordered by
// sub-cell inside each cell (cell membership and cell_start are unchanged), which lets the
// pair kernels cull j-ranges that lie farther than eta from a target tile.
//
// Passes (all deterministic, no float atomics):
//   1. k_bin_count   — per tile of T pid-ordered particles: smem histogram of keys,
//                      written key-major: counts[key * n_tiles + tile].
//   2. exclusive scan of counts (3 small kernels)  -> global offset of (key, tile).
//   3. k_bin_starts  — cell_start / sub_start from the scanned counts.
//   4. k_bin_scatter — per tile, W warps each own a contiguous sub-chunk; per-warp key
//                      histograms are prefix-summed across warps, then each warp replays its
//                      sub-chunk in lane order with __match_any_sync ranks. Position order is
//                      therefore (key, tile, warp, group, lane) = (key, pid): stable.
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "pairs.cuh"

namespace spic {

struct BinPlan {
  int K, W, G, T, n_tiles;
  size_t counts_elems, nb_scan;
};

constexpr int kScanThreads = 1024;
constexpr int kScanPerThread = 16;
constexpr int kScanChunk = kScanThreads * kScanPerThread;

static BinPlan bin_plan(int64_t n, int M, int S) {
  BinPlan p;
  p.K = M * S;
  int W = 32768 / p.K;
  p.W = W < 1 ? 1 : (W > 8 ? 8 : W);
  // about one tile per SM: the (key, tile) count table then stays ~K x 148 entries (small
  // next to n) and the scatter kernel runs one wave
  long long per = (long long)p.W * 32 * kNumSMs;
  long long G = (n + per - 1) / per;
  p.G = (int)(G < 4 ? 4 : (G > 8192 ? 8192 : G));
  p.T = p.W * 32 * p.G;
  p.n_tiles = (int)((n + p.T - 1) / p.T);
  if (p.n_tiles < 1) p.n_tiles = 1;
  p.counts_elems = (size_t)p.K * p.n_tiles;
  p.nb_scan = (p.counts_elems + kScanChunk - 1) / kScanChunk;
  return p;
}

__global__ void k_cell_of(const float* __restrict__ x, int64_t n, double eta, int M,
                          int32_t* __restrict__ cell) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cell[i] = cell_key(x[i], eta, M, 1).cell;
}

__global__ void k_bin_count(const float* __restrict__ x, int64_t n, double eta, int M, int S,
                            int T, int n_tiles, int32_t* __restrict__ counts) {
  extern __shared__ int hist[];
  const int K = M * S;
  for (int k = threadIdx.x; k < K; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * T;
  const int64_t end = min((int64_t)n, base + T);
  for (int64_t i0 = base + threadIdx.x; i0 < end; i0 += 8 * (int64_t)blockDim.x) {
    float xs[8];  // loads of eight strides issued before their keys
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + u * (int64_t)blockDim.x;
      xs[u] = i < end ? x[i] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u * (int64_t)blockDim.x < end) {
        CellKey ck = cell_key(xs[u], eta, M, S);
        atomicAdd(&hist[ck.cell * S + ck.sub], 1);
      }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    counts[(size_t)k * n_tiles + blockIdx.x] = hist[k];
}

// ---- exclusive scan of int32 (in place), three launches --------------------------------
__global__ void k_scan_reduce(const int32_t* __restrict__ a, size_t n, int32_t* __restrict__ bsum) {
  __shared__ int ws[32];
  size_t base = (size_t)blockIdx.x * kScanChunk + (size_t)threadIdx.x * kScanPerThread;
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k)
    if (base + k < n) s += a[base + k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    int t = ws[threadIdx.x];
    t = warp_sum(t);
    if (threadIdx.x == 0) bsum[blockIdx.x] = t;
  }
}

// block-wide exclusive scan of one value per thread (blockDim.x == 1024)
__device__ __forceinline__ int block_excl_scan(int v, int* ws, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) ws[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = ws[lane];
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += t;
    }
    ws[lane] = si - s;  // exclusive warp offsets
    if (lane == 31) ws[32] = si;
  }
  __syncthreads();
  int out = ws[wid] + inc - v;
  if (total) *total = ws[32];
  __syncthreads();
  return out;
}

__global__ void k_scan_blocksums(int32_t* __restrict__ bsum, size_t nb) {
  __shared__ int ws[33];
  int carry = 0;
  for (size_t base = 0; base < nb; base += blockDim.x) {
    size_t i = base + threadIdx.x;
    int v = i < nb ? bsum[i] : 0;
    int tot;
    int ex = block_excl_scan(v, ws, &tot);
    if (i < nb) bsum[i] = carry + ex;
    carry += tot;
  }
}

__global__ void k_scan_apply(int32_t* __restrict__ a, size_t n, const int32_t* __restrict__ bsum) {
  __shared__ int ws[33];
  size_t base = (size_t)blockIdx.x * kScanChunk + (size_t)threadIdx.x * kScanPerThread;
  int vals[kScanPerThread];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    vals[k] = base + k < n ? a[base + k] : 0;
    s += vals[k];
  }
  int off = block_excl_scan(s, ws, nullptr) + bsum[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    if (base + k < n) a[base + k] = off;
    off += vals[k];
  }
}

__global__ void k_bin_starts(const int32_t* __restrict__ scanned, int M, int S, int n_tiles,
                             int32_t n, int32_t* __restrict__ cell_start,
                             int32_t* __restrict__ sub_start) {
  const int K = M * S;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= K; k += gridDim.x * blockDim.x) {
    int32_t v = k < K ? scanned[(size_t)k * n_tiles] : n;
    if (sub_start) sub_start[k] = v;
    if (k % S == 0) cell_start[k / S] = v;
  }
}

__global__ void __launch_bounds__(256) k_bin_scatter(
    const float* __restrict__ x, const float* __restrict__ v, int64_t ldv,
    const float* __restrict__ w, int64_t n, int dv, double eta, double L, int M, int S, int W,
    int G, int n_tiles, const int32_t* __restrict__ scanned, int32_t* __restrict__ perm,
    float4* __restrict__ xv, float4* __restrict__ sw) {
  extern __shared__ int hist[];  // [W][K]
  const int K = M * S;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < W * K; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  const int T = W * 32 * G;
  const int64_t wbase = (int64_t)blockIdx.x * T + (int64_t)wid * 32 * G;
  int* my = hist + wid * K;
  // pass 1: per-warp histogram of its sub-chunk (positions loaded kPF groups ahead: the
  // sweep is latency-bound, one warp per key-histogram slice)
  constexpr int kPF = 8;
  for (int g0 = 0; g0 < G; g0 += kPF) {
    float xs[kPF];
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
      const int64_t i = wbase + (int64_t)(g0 + u) * 32 + lane;
      xs[u] = (g0 + u < G && i < n) ? x[i] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
      const int64_t i = wbase + (int64_t)(g0 + u) * 32 + lane;
      if (g0 + u < G && i < n) {
        CellKey ck = cell_key(xs[u], eta, M, S);
        atomicAdd(&my[ck.cell * S + ck.sub], 1);
      }
    }
  }
  __syncthreads();
  // pass 2: per key, exclusive prefix across warps, seeded with the global (key, tile) offset
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    int run = scanned[(size_t)k * n_tiles + blockIdx.x];
    for (int q = 0; q < W; ++q) {
      int t = hist[q * K + k];
      hist[q * K + k] = run;
      run += t;
    }
  }
  __syncthreads();
  // pass 3: replay in pid order, rank within 32-groups by key (record fields loaded kPF
  // groups ahead; the key ranks are the only serial dependency)
  for (int g0 = 0; g0 < G; g0 += kPF) {
    float xs[kPF], v0[kPF], v1[kPF], v2[kPF], ws[kPF];
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
      const int64_t i = wbase + (int64_t)(g0 + u) * 32 + lane;
      const bool ok = g0 + u < G && i < n;
      xs[u] = ok ? x[i] : 0.f;
      v0[u] = (ok && xv) ? v[i] : 0.f;
      v1[u] = (ok && xv) ? v[ldv + i] : 0.f;
      v2[u] = (ok && xv && dv > 2) ? v[2 * ldv + i] : 0.f;
      ws[u] = (ok && w) ? w[i] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
      const int64_t i = wbase + (int64_t)(g0 + u) * 32 + lane;
      const bool valid = g0 + u < G && i < n;
      const unsigned active = __ballot_sync(0xffffffffu, valid);
      if (valid) {
        const float xi = xs[u];
        CellKey ck = cell_key(xi, eta, M, S);
        int key = ck.cell * S + ck.sub;
        unsigned peers = __match_any_sync(active, key);
        int rank = __popc(peers & lanemask_lt());
        int basepos = my[key];
        __syncwarp(active);
        if (rank == 0) my[key] = basepos + __popc(peers);
        int pos = basepos + rank;
        if (perm) perm[pos] = (int32_t)i;
        if (xv) {
          float4 r;
          r.x = ck.wrapped ? (float)((double)xi - L) : xi;
          r.y = v0[u];
          r.z = v1[u];
          r.w = v2[u];
          xv[pos] = r;
        }
        if (sw) sw[pos] = make_float4(0.f, 0.f, 0.f, ws[u]);
      }
      __syncwarp();
    }
  }
}

// ---- LSD radix path: two stable 8/7-bit digit passes with many small tiles --------------
// The single-pass scatter above ranks keys with one warp per K-entry histogram slice, so for
// K = M*S up to 32768 only 1-2 warps fit per SM and the sweep is latency-bound. The radix path
// sorts the same (key, pid) order with <= 256 buckets per pass: 8 warps per tile, thousands
// of tiles, and the counts table stays 256 x tiles. Key word: bits 0-14 key, bit 15 the
// "x rounds onto L" flag (stored x - L).
constexpr int kRxW = 8, kRxG = 8, kRxT = kRxW * 32 * kRxG;  // tile = 2048 records
constexpr int kRxB = 256;

struct RadixPlan {
  int bits, passes, n_tiles;
  size_t counts_elems, nb_scan;
};

static RadixPlan radix_plan(int64_t n, int M, int S) {
  RadixPlan r;
  const int K = M * S;
  r.bits = 1;
  while ((1 << r.bits) < K) ++r.bits;
  r.passes = r.bits <= 8 ? 1 : 2;
  r.n_tiles = (int)std::max<int64_t>(1, (n + kRxT - 1) / kRxT);
  r.counts_elems = (size_t)kRxB * r.n_tiles;
  r.nb_scan = (size_t)kRxB * ((r.n_tiles + 63) / 64);  // column-scan block sums (kRxR = 64)
  return r;
}

__device__ __forceinline__ uint32_t key_word(float xf, double eta, int M, int S) {
  const CellKey ck = cell_key(xf, eta, M, S);
  return (uint32_t)(ck.cell * S + ck.sub) | (ck.wrapped ? 0x8000u : 0u);
}

// histogram of one digit per tile (keys from x on the first pass, else from key_in)
template <bool FROM_X>
__global__ void __launch_bounds__(256) k_radix_count(const float* __restrict__ x,
                                                     const uint32_t* __restrict__ key_in,
                                                     uint32_t* __restrict__ key_out, int64_t n,
                                                     double eta, int M, int S, int shift,
                                                     int mask, int n_tiles,
                                                     int32_t* __restrict__ counts) {
  __shared__ int hist[kRxB];
  for (int k = threadIdx.x; k < kRxB; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRxT;
#pragma unroll
  for (int u = 0; u < kRxT / 256; ++u) {
    const int64_t i = base + u * 256 + threadIdx.x;
    if (i < n) {
      uint32_t kw;
      if (FROM_X) {
        kw = key_word(x[i], eta, M, S);
        key_out[i] = kw;
      } else {
        kw = key_in[i];
      }
      atomicAdd(&hist[(kw >> shift) & mask], 1);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kRxB; k += blockDim.x)
    counts[(size_t)blockIdx.x * kRxB + k] = hist[k];  // tile-major row: one coalesced store
}

// Stable scatter of one digit pass: warp w of a tile owns records [32 G w, 32 G (w+1)); per-warp
// digit counts, prefix across warps seeded with the scanned (digit, tile) offset, then each
// warp replays its records in order ranking equal digits with __match_any_sync. The record
// payload (pid, (x', v), w) travels with the key, so every pass reads its input in order:
//   MODE 0: first of two passes   planes (pid order) -> key1, idx1, rec1, w1 (by low digit)
//   MODE 1: second of two passes  key1, idx1, rec1, w1 -> perm, sorted keys, xv, sw
//   MODE 2: the only pass         planes (pid order) -> perm, sorted keys, xv, sw
template <int MODE>
__global__ void __launch_bounds__(kRxW * 32) k_radix_scatter(
    const uint32_t* __restrict__ key_in, const int32_t* __restrict__ idx_in,
    const float4* __restrict__ rec_in, const float* __restrict__ w_in, int64_t n, int shift,
    int mask, int n_tiles, const int32_t* __restrict__ scanned, uint32_t* __restrict__ key_out,
    int32_t* __restrict__ idx_out, float4* __restrict__ rec_out, float* __restrict__ w_out,
    const float* __restrict__ x, const float* __restrict__ v, int64_t ldv,
    const float* __restrict__ w, int dv, double L) {
  __shared__ int hist[kRxW][kRxB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < kRxW * kRxB; k += blockDim.x) (&hist[0][0])[k] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * kRxT + (int64_t)wid * 32 * kRxG;
  uint32_t kw[kRxG];
#pragma unroll
  for (int g = 0; g < kRxG; ++g) {
    const int64_t i = wbase + g * 32 + lane;
    kw[g] = i < n ? key_in[i] : 0u;
  }
#pragma unroll
  for (int g = 0; g < kRxG; ++g)
    if (wbase + g * 32 + lane < n) atomicAdd(&hist[wid][(kw[g] >> shift) & mask], 1);
  __syncthreads();
  for (int k = threadIdx.x; k < kRxB; k += blockDim.x) {
    int run = scanned[(size_t)blockIdx.x * kRxB + k];
#pragma unroll
    for (int q = 0; q < kRxW; ++q) {
      const int t = hist[q][k];
      hist[q][k] = run;
      run += t;
    }
  }
  __syncthreads();
  int* my = hist[wid];
#pragma unroll 2
  for (int g = 0; g < kRxG; ++g) {
    const int64_t i = wbase + g * 32 + lane;
    const bool valid = i < n;
    // payload of this record (coalesced loads, issued before the ranking)
    int32_t pid = 0;
    float4 rec = make_float4(0.f, 0.f, 0.f, 0.f);
    float wv = 0.f;
    if (valid) {
      if (MODE == 1) {
        pid = idx_in[i];
        rec = rec_in[i];
        wv = w_in ? w_in[i] : 0.f;
      } else {
        pid = (int32_t)i;
        const float xi = x[i];
        rec.x = (kw[g] & 0x8000u) ? (float)((double)xi - L) : xi;
        rec.y = v[i];
        rec.z = v[ldv + i];
        rec.w = dv > 2 ? v[2 * ldv + i] : 0.f;
        wv = w ? w[i] : 0.f;
      }
    }
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      const int dg = (int)((kw[g] >> shift) & mask);
      const unsigned peers = __match_any_sync(active, dg);
      const int rank = __popc(peers & lanemask_lt());
      const int basepos = my[dg];
      __syncwarp(active);
      if (rank == 0) my[dg] = basepos + __popc(peers);
      const int pos = basepos + rank;
      key_out[pos] = kw[g];
      if (idx_out) idx_out[pos] = pid;
      if (rec_out) rec_out[pos] = rec;
      if (MODE == 0) {
        if (w_out) w_out[pos] = wv;
      } else if (w_out) {  // the sw record: scores are filled in later, w in lane 3
        reinterpret_cast<float4*>(w_out)[pos] = make_float4(0.f, 0.f, 0.f, wv);
      }
    }
    __syncwarp();
  }
}

// Staged variant of k_radix_scatter: the same ranks, but each tile is first reordered in
// shared memory (tile-local position = digit's offset in the tile + rank), then written out
// with consecutive threads on consecutive tile positions, so every digit run of the tile
// leaves as one coalesced burst instead of 32 scattered stores per warp instruction (the
// scattered form writes partial sectors: ncu counted ~1.7x the payload in DRAM traffic).
constexpr size_t kRxStagedSmem =
    sizeof(int) * (kRxW * kRxB + 2 * kRxB + 32) +
    (size_t)kRxT * (sizeof(uint32_t) + sizeof(int32_t) + sizeof(float4) + sizeof(float));

template <int MODE>
__global__ void __launch_bounds__(kRxW * 32) k_radix_scatter_s(
    const uint32_t* __restrict__ key_in, const int32_t* __restrict__ idx_in,
    const float4* __restrict__ rec_in, const float* __restrict__ w_in, int64_t n, int shift,
    int mask, int n_tiles, const int32_t* __restrict__ scanned, uint32_t* __restrict__ key_out,
    int32_t* __restrict__ idx_out, float4* __restrict__ rec_out, float* __restrict__ w_out,
    const float* __restrict__ x, const float* __restrict__ v, int64_t ldv,
    const float* __restrict__ w, int dv, double L) {
  extern __shared__ __align__(16) unsigned char s_dyn_rx[];
  float4* s_rec = reinterpret_cast<float4*>(s_dyn_rx);                     // [kRxT]
  uint32_t* s_key = reinterpret_cast<uint32_t*>(s_rec + kRxT);             // [kRxT]
  int32_t* s_idx = reinterpret_cast<int32_t*>(s_key + kRxT);               // [kRxT]
  float* s_w = reinterpret_cast<float*>(s_idx + kRxT);                     // [kRxT]
  int* hist = reinterpret_cast<int*>(s_w + kRxT);                          // [kRxW][kRxB]
  int* s_lb = hist + kRxW * kRxB;                                          // [kRxB]
  int* s_gb = s_lb + kRxB;                                                 // [kRxB]
  int* s_ws = s_gb + kRxB;                                                 // [32]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < kRxW * kRxB; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  const int64_t tbase = (int64_t)blockIdx.x * kRxT;
  const int cnt = n - tbase < kRxT ? (int)(n - tbase) : kRxT;
  const int64_t wbase = tbase + (int64_t)wid * 32 * kRxG;
  uint32_t kw[kRxG];
#pragma unroll
  for (int g = 0; g < kRxG; ++g) {
    const int64_t i = wbase + g * 32 + lane;
    kw[g] = i < n ? key_in[i] : 0u;
  }
#pragma unroll
  for (int g = 0; g < kRxG; ++g)
    if (wbase + g * 32 + lane < n) atomicAdd(&hist[wid * kRxB + ((kw[g] >> shift) & mask)], 1);
  __syncthreads();
  // digit d = threadIdx.x: tile total, exclusive scan over digits -> local base; per-warp
  // running offsets start at local base + earlier warps' counts
  {
    const int d = threadIdx.x;  // blockDim.x == kRxB
    int tot = 0;
#pragma unroll
    for (int q = 0; q < kRxW; ++q) tot += hist[q * kRxB + d];
    int inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_ws[wid] = inc;
    __syncthreads();
    int wpre = 0;
    for (int q = 0; q < wid; ++q) wpre += s_ws[q];
    const int lb = wpre + inc - tot;
    s_lb[d] = lb;
    s_gb[d] = scanned[(size_t)blockIdx.x * kRxB + d];
    int run = lb;
#pragma unroll
    for (int q = 0; q < kRxW; ++q) {
      const int t = hist[q * kRxB + d];
      hist[q * kRxB + d] = run;
      run += t;
    }
  }
  __syncthreads();
  int* my = hist + wid * kRxB;
#pragma unroll 2
  for (int g = 0; g < kRxG; ++g) {
    const int64_t i = wbase + g * 32 + lane;
    const bool valid = i < n;
    int32_t pid = 0;
    float4 rec = make_float4(0.f, 0.f, 0.f, 0.f);
    float wv = 0.f;
    if (valid) {
      if (MODE == 1) {
        pid = idx_in[i];
        rec = rec_in[i];
        wv = w_in ? w_in[i] : 0.f;
      } else {
        pid = (int32_t)i;
        const float xi = x[i];
        rec.x = (kw[g] & 0x8000u) ? (float)((double)xi - L) : xi;
        rec.y = v[i];
        rec.z = v[ldv + i];
        rec.w = dv > 2 ? v[2 * ldv + i] : 0.f;
        wv = w ? w[i] : 0.f;
      }
    }
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      const int dg = (int)((kw[g] >> shift) & mask);
      const unsigned peers = __match_any_sync(active, dg);
      const int rank = __popc(peers & lanemask_lt());
      const int basepos = my[dg];
      __syncwarp(active);
      if (rank == 0) my[dg] = basepos + __popc(peers);
      const int lp = basepos + rank;
      s_key[lp] = kw[g];
      s_idx[lp] = pid;
      s_rec[lp] = rec;
      s_w[lp] = wv;
    }
    __syncwarp();
  }
  __syncthreads();
  for (int l = threadIdx.x; l < cnt; l += blockDim.x) {
    const uint32_t k = s_key[l];
    const int dg = (int)((k >> shift) & mask);
    const int pos = s_gb[dg] + (l - s_lb[dg]);
    key_out[pos] = k;
    if (idx_out) idx_out[pos] = s_idx[l];
    if (rec_out) rec_out[pos] = s_rec[l];
    if (MODE == 0) {
      if (w_out) w_out[pos] = s_w[l];
    } else if (w_out) {
      reinterpret_cast<float4*>(w_out)[pos] = make_float4(0.f, 0.f, 0.f, s_w[l]);
    }
  }
}

// Bulk-copy variant of the staged scatter: the tile's keys and payload arrive in shared memory
// by cp.async.bulk (keys on one mbarrier, payload on a second, so the histogram and digit
// scan run while the payload is still in flight); the ranking only records each tile
// position's source index, and the write-out gathers the payload from shared memory. No
// thread waits on a global load (the direct-load form stalls on long scoreboards: 0.78 IPC).
// Needs 16-B aligned input ranges (the caller checks) and a tile length that is a multiple
// of 4 records; the partial last tile falls back to plain loads.
constexpr size_t kRxBulkSmem =
    128 + (size_t)kRxT * (4 /*key*/ + 4 /*idx or x*/ + 16 /*rec or v0..v2 + pad*/ + 4 /*w*/) +
    (size_t)kRxT * 2 /*src*/ + sizeof(int) * (kRxW * kRxB + 2 * kRxB + 32) + 2 * sizeof(uint64_t);

template <int MODE>
__global__ void __launch_bounds__(kRxW * 32) k_radix_scatter_b(
    const uint32_t* __restrict__ key_in, const int32_t* __restrict__ idx_in,
    const float4* __restrict__ rec_in, const float* __restrict__ w_in, int64_t n, int shift,
    int mask, int n_tiles, const int32_t* __restrict__ scanned, uint32_t* __restrict__ key_out,
    int32_t* __restrict__ idx_out, float4* __restrict__ rec_out, float* __restrict__ w_out,
    const float* __restrict__ x, const float* __restrict__ v, int64_t ldv,
    const float* __restrict__ w, int dv, double L) {
  extern __shared__ unsigned char s_dyn_rb[];
  unsigned char* sb = s_dyn_rb + ((128u - (uint32_t)((uintptr_t)s_dyn_rb & 127u)) & 127u);
  uint32_t* s_key = reinterpret_cast<uint32_t*>(sb);                      // [kRxT]
  int32_t* s_i = reinterpret_cast<int32_t*>(s_key + kRxT);                // idx (1) / x (0, 2)
  float4* s_rec = reinterpret_cast<float4*>(s_i + kRxT);                  // rec (1)
  float* s_pl = reinterpret_cast<float*>(s_rec);                          // v0, v1, v2 (0, 2)
  float* s_w = reinterpret_cast<float*>(s_rec + kRxT);                    // [kRxT]
  uint16_t* s_src = reinterpret_cast<uint16_t*>(s_w + kRxT);              // [kRxT]
  int* hist = reinterpret_cast<int*>(s_src + kRxT);                       // [kRxW][kRxB]
  int* s_lb = hist + kRxW * kRxB;
  int* s_gb = s_lb + kRxB;
  int* s_ws = s_gb + kRxB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_ws + 32);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t tbase = (int64_t)blockIdx.x * kRxT;
  const int cnt = n - tbase < kRxT ? (int)(n - tbase) : kRxT;
  const bool bulk = (cnt & 3) == 0;
  if (threadIdx.x == 0 && bulk) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    const uint32_t b4 = (uint32_t)cnt * 4;
    mbar_expect_tx(&bar[0], b4);
    bulk_g2s(s_key, key_in + tbase, b4, &bar[0]);
    uint32_t tot = 0;
    if (MODE == 1) {
      tot = b4 + 4 * b4 + (w_in ? b4 : 0);
      mbar_expect_tx(&bar[1], tot);
      bulk_g2s(s_i, idx_in + tbase, b4, &bar[1]);
      bulk_g2s(s_rec, rec_in + tbase, 4 * b4, &bar[1]);
      if (w_in) bulk_g2s(s_w, w_in + tbase, b4, &bar[1]);
    } else {
      tot = b4 * (1 + 2 + (dv > 2 ? 1 : 0) + (w ? 1 : 0));
      mbar_expect_tx(&bar[1], tot);
      bulk_g2s(s_i, x + tbase, b4, &bar[1]);
      bulk_g2s(s_pl, v + tbase, b4, &bar[1]);
      bulk_g2s(s_pl + kRxT, v + ldv + tbase, b4, &bar[1]);
      if (dv > 2) bulk_g2s(s_pl + 2 * kRxT, v + 2 * ldv + tbase, b4, &bar[1]);
      if (w) bulk_g2s(s_w, w + tbase, b4, &bar[1]);
    }
  }
  for (int k = threadIdx.x; k < kRxW * kRxB; k += blockDim.x) hist[k] = 0;
  if (!bulk) {  // partial last tile: plain loads into the same staging
    for (int l = threadIdx.x; l < cnt; l += blockDim.x) {
      const int64_t i = tbase + l;
      s_key[l] = key_in[i];
      if (MODE == 1) {
        s_i[l] = idx_in[i];
        s_rec[l] = rec_in[i];
        if (w_in) s_w[l] = w_in[i];
      } else {
        s_i[l] = __float_as_int(x[i]);
        s_pl[l] = v[i];
        s_pl[kRxT + l] = v[ldv + i];
        if (dv > 2) s_pl[2 * kRxT + l] = v[2 * ldv + i];
        if (w) s_w[l] = w[i];
      }
    }
  }
  __syncthreads();
  if (bulk) mbar_wait(&bar[0], 0);
  const int wl0 = wid * 32 * kRxG;  // this warp's first tile position
  uint32_t kw[kRxG];
#pragma unroll
  for (int g = 0; g < kRxG; ++g) {
    const int l = wl0 + g * 32 + lane;
    kw[g] = l < cnt ? s_key[l] : 0u;
    if (l < cnt) atomicAdd(&hist[wid * kRxB + ((kw[g] >> shift) & mask)], 1);
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // blockDim.x == kRxB
    int tot = 0;
#pragma unroll
    for (int q = 0; q < kRxW; ++q) tot += hist[q * kRxB + d];
    int inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_ws[wid] = inc;
    __syncthreads();
    int wpre = 0;
    for (int q = 0; q < wid; ++q) wpre += s_ws[q];
    const int lb = wpre + inc - tot;
    s_lb[d] = lb;
    s_gb[d] = scanned[(size_t)blockIdx.x * kRxB + d];
    int run = lb;
#pragma unroll
    for (int q = 0; q < kRxW; ++q) {
      const int t = hist[q * kRxB + d];
      hist[q * kRxB + d] = run;
      run += t;
    }
  }
  __syncthreads();
  int* my = hist + wid * kRxB;
#pragma unroll
  for (int g = 0; g < kRxG; ++g) {
    const int l = wl0 + g * 32 + lane;
    const bool valid = l < cnt;
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      const int dg = (int)((kw[g] >> shift) & mask);
      const unsigned peers = __match_any_sync(active, dg);
      const int rank = __popc(peers & lanemask_lt());
      const int basepos = my[dg];
      __syncwarp(active);
      if (rank == 0) my[dg] = basepos + __popc(peers);
      s_src[basepos + rank] = (uint16_t)l;
    }
    __syncwarp();
  }
  __syncthreads();
  if (bulk) mbar_wait(&bar[1], 0);
  for (int l = threadIdx.x; l < cnt; l += blockDim.x) {
    const int src = s_src[l];
    const uint32_t k = s_key[src];
    const int dg = (int)((k >> shift) & mask);
    const int pos = s_gb[dg] + (l - s_lb[dg]);
    key_out[pos] = k;
    float4 rec;
    int32_t pid;
    if (MODE == 1) {
      pid = s_i[src];
      rec = s_rec[src];
    } else {
      pid = (int32_t)(tbase + src);
      const float xi = __int_as_float(s_i[src]);
      rec.x = (k & 0x8000u) ? (float)((double)xi - L) : xi;
      rec.y = s_pl[src];
      rec.z = s_pl[kRxT + src];
      rec.w = dv > 2 ? s_pl[2 * kRxT + src] : 0.f;
    }
    const bool has_w = MODE == 1 ? (w_in != nullptr) : (w != nullptr);
    const float wv = has_w ? s_w[src] : 0.f;
    if (idx_out) idx_out[pos] = pid;
    if (rec_out) rec_out[pos] = rec;
    if (MODE == 0) {
      if (w_out) w_out[pos] = wv;
    } else if (w_out) {
      reinterpret_cast<float4*>(w_out)[pos] = make_float4(0.f, 0.f, 0.f, wv);
    }
  }
}

// Exclusive (digit, tile)-order scan of the tile-major radix count table c[tile][digit]:
//   offset[t][d] = sum_{d' < d} total[d'] + sum_{t' < t} c[t'][d].
// Two launches, every table access a coalesced 1-KB row: column sums per block of kRxR tiles,
// then per block the apply, which first derives its own prefix and the digit totals from all
// block sums (L2-resident, nb x 1 KB) and scans the totals over the digits in the CTA.
constexpr int kRxR = 64;  // tiles per column-scan block
__global__ void __launch_bounds__(kRxB) k_rx_colsum(const int32_t* __restrict__ c, int n_tiles,
                                                   int32_t* __restrict__ bsum) {
  const int d = threadIdx.x, t0 = blockIdx.x * kRxR, t1 = min(t0 + kRxR, n_tiles);
  int s = 0;
  for (int tb = t0; tb < t1; tb += 16) {
    int v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = tb + i < t1 ? c[(size_t)(tb + i) * kRxB + d] : 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += v[i];
  }
  bsum[(size_t)blockIdx.x * kRxB + d] = s;
}
__global__ void __launch_bounds__(kRxB) k_rx_colscan_apply(int32_t* __restrict__ c, int n_tiles,
                                                          const int32_t* __restrict__ bsum,
                                                          int nb) {
  __shared__ int ws[kRxB / 32];
  const int d = threadIdx.x, lane = d & 31, wid = d >> 5;
  int pre = 0, tot = 0;
  for (int bb = 0; bb < nb; bb += 16) {
    int v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = bb + i < nb ? bsum[(size_t)(bb + i) * kRxB + d] : 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      pre += bb + i < (int)blockIdx.x ? v[i] : 0;
      tot += v[i];
    }
  }
  int inc = tot;  // exclusive scan of the digit totals across the CTA
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) ws[wid] = inc;
  __syncthreads();
  int wpre = 0;
  for (int q = 0; q < wid; ++q) wpre += ws[q];
  int run = wpre + inc - tot + pre;
  const int t0 = blockIdx.x * kRxR, t1 = min(t0 + kRxR, n_tiles);
  for (int tb = t0; tb < t1; tb += 16) {  // 16 independent loads in flight, then the stores
    int v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = tb + i < t1 ? c[(size_t)(tb + i) * kRxB + d] : 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (tb + i < t1) c[(size_t)(tb + i) * kRxB + d] = run;
      run += v[i];
    }
  }
}

// cell_start / sub_start from the sorted key words: position k starts every key in
// (key[k-1], key[k]] (key[-1] = -1, key[n] = K)
__global__ void k_radix_starts(const uint32_t* __restrict__ key_sorted, int64_t n, int M, int S,
                               int32_t* __restrict__ cell_start, int32_t* __restrict__ sub_start) {
  const int K = M * S;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int cur = k < n ? (int)(key_sorted[k] & 0x7FFFu) : K;
    const int prev = k > 0 ? (int)(key_sorted[k - 1] & 0x7FFFu) : -1;
    for (int q = prev + 1; q <= cur; ++q) {
      if (sub_start) sub_start[q] = (int32_t)k;
      if (q % S == 0) cell_start[q / S] = (int32_t)k;
    }
  }
}

__global__ void k_gather_scores(const float* __restrict__ s, int64_t lds,
                                const int32_t* __restrict__ perm, int64_t n, int dv,
                                float4* __restrict__ sw, int32_t* flags) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int32_t i = perm[k];
    float4 r = sw[k];
    r.x = s[i];
    r.y = s[lds + i];
    r.z = dv > 2 ? s[2 * lds + i] : 0.f;
    if (!(isfinite(r.x) && isfinite(r.y) && isfinite(r.z))) raise_flag(flags, SPIC_FLAG_BAD_SCORE);
    sw[k] = r;
  }
}

}  // namespace spic

namespace spic {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace spic

using namespace spic;

extern "C" int spic_version(void) { return 1; }
extern "C" long long spic_launch_count(void) { return g_launches.load(); }
extern "C" int spic_num_sms(void) { return kNumSMs; }

extern "C" int spic_cell_of(const float* x, int64_t n, double eta, int32_t M, int32_t* cell,
                            void* stream) {
  if (n < 0 || M < 1 || !(eta > 0)) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  k_cell_of<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, n, eta, M, cell); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

// Path choice: the radix path (bulk-staged scatters) wins from ~2^20 records (2^20: 0.124 vs
// 0.138 ms, 2^22: 0.26 vs 0.81 ms, 2^24: 0.86 vs 5.15 ms); below that its 11 launches cost
// more than the single-pass sort saves (0.070 vs 0.050 ms at 2^16). SPIC_BIN_VARIANT=c / r
// forces a path (A/B tests).
static bool bin_use_counting(int64_t n) {
  const char* e = getenv("SPIC_BIN_VARIANT");
  if (e && e[0] == 'c') return true;
  if (e && e[0] == 'r') return false;
  return n < ((int64_t)1 << 20);
}

static size_t radix_scratch_bytes(int64_t n, int32_t M, int32_t S) {
  RadixPlan r = radix_plan(n, M, S);
  // key words (pid order), pass-1 (key, pid, record, w), sorted keys, counts + block sums
  return sizeof(int32_t) * (9 * (size_t)n + r.counts_elems + r.nb_scan + 64) + 8 * 256;
}

extern "C" size_t spic_bin_scratch_bytes(int64_t n, int32_t M, int32_t S) {
  if (M < 1 || S < 1) return 0;
  BinPlan p = bin_plan(n, M, S);
  size_t b = (p.counts_elems + p.nb_scan + 64) * sizeof(int32_t);
  if (!bin_use_counting(n)) b = std::max(b, radix_scratch_bytes(n, M, S));
  return b;
}

static int bin_radix(const float* x, const float* v, int64_t ldv, const float* w, int64_t n,
                     int32_t dv, double eta, int32_t M, int32_t S, int32_t* perm,
                     int32_t* cell_start, int32_t* sub_start, float* xv, float* sw,
                     void* scratch, cudaStream_t st) {
  RadixPlan r = radix_plan(n, M, S);
  auto align = [](void* p) { return (void*)(((uintptr_t)p + 255) & ~(uintptr_t)255); };
  uint32_t* key0 = (uint32_t*)align(scratch);
  uint32_t* key1 = (uint32_t*)align(key0 + n);
  int32_t* idx1 = (int32_t*)align(key1 + n);
  uint32_t* keyS = (uint32_t*)align(idx1 + n);
  float4* rec1 = (float4*)align(keyS + n);
  float* w1 = (float*)align(rec1 + n);
  int32_t* counts = (int32_t*)align(w1 + n);
  int32_t* bsum = counts + r.counts_elems;
  const double L = (double)M * eta;
  const unsigned nt = (unsigned)r.n_tiles;
  const int nbk = (r.n_tiles + kRxR - 1) / kRxR;
  auto scan = [&]() {
    k_rx_colsum<<<(unsigned)nbk, kRxB, 0, st>>>(counts, r.n_tiles, bsum);
    k_rx_colscan_apply<<<(unsigned)nbk, kRxB, 0, st>>>(counts, r.n_tiles, bsum, nbk);
    for (int k = 0; k < 2; ++k) spic::count_launch();
  };
  // "0": the direct-scatter kernels, "1": staged with plain loads, default: staged with bulk
  // copies when the input planes are 16-B aligned (A/B)
  const char* se = getenv("SPIC_RADIX_STAGED");
  const bool aligned = ((((uintptr_t)x) | ((uintptr_t)v) | ((uintptr_t)w)) & 15) == 0 &&
                       (ldv & 3) == 0;
  const bool bulkrx = !(se && (se[0] == '0' || se[0] == '1')) && aligned;
  const bool staged = !(se && se[0] == '0');
  if (staged) {
    cudaFuncSetAttribute(k_radix_scatter_s<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRxStagedSmem);
    cudaFuncSetAttribute(k_radix_scatter_s<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRxStagedSmem);
    cudaFuncSetAttribute(k_radix_scatter_s<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRxStagedSmem);
  }
  if (bulkrx) {
    cudaFuncSetAttribute(k_radix_scatter_b<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRxBulkSmem);
    cudaFuncSetAttribute(k_radix_scatter_b<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRxBulkSmem);
    cudaFuncSetAttribute(k_radix_scatter_b<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRxBulkSmem);
  }
  const size_t ssm = bulkrx ? kRxBulkSmem : (staged ? kRxStagedSmem : 0);
  auto sc0 = bulkrx ? k_radix_scatter_b<0> : (staged ? k_radix_scatter_s<0> : k_radix_scatter<0>);
  auto sc1 = bulkrx ? k_radix_scatter_b<1> : (staged ? k_radix_scatter_s<1> : k_radix_scatter<1>);
  auto sc2 = bulkrx ? k_radix_scatter_b<2> : (staged ? k_radix_scatter_s<2> : k_radix_scatter<2>);
  const int lo_bits = r.passes == 1 ? r.bits : 8;
  const int mask0 = (1 << lo_bits) - 1;
  k_radix_count<true><<<nt, 256, 0, st>>>(x, nullptr, key0, n, eta, M, S, 0, mask0, r.n_tiles,
                                          counts);
  spic::count_launch();
  scan();
  if (r.passes == 1) {
    sc2<<<nt, kRxW * 32, ssm, st>>>(key0, nullptr, nullptr, nullptr, n, 0, mask0,
                                                 r.n_tiles, counts, keyS, perm, (float4*)xv, sw,
                                                 x, v, ldv, w, dv, L);
    spic::count_launch();
  } else {
    sc0<<<nt, kRxW * 32, ssm, st>>>(key0, nullptr, nullptr, nullptr, n, 0, mask0,
                                                 r.n_tiles, counts, key1, idx1, rec1,
                                                 w ? w1 : nullptr, x, v, ldv, w, dv, L);
    spic::count_launch();
    const int mask1 = (1 << (r.bits - 8)) - 1;
    k_radix_count<false><<<nt, 256, 0, st>>>(nullptr, key1, nullptr, n, eta, M, S, 8, mask1,
                                             r.n_tiles, counts);
    spic::count_launch();
    scan();
    sc1<<<nt, kRxW * 32, ssm, st>>>(key1, idx1, rec1, w ? w1 : nullptr, n, 8, mask1,
                                                 r.n_tiles, counts, keyS, perm, (float4*)xv, sw,
                                                 nullptr, nullptr, 0, nullptr, dv, L);
    spic::count_launch();
  }
  const int sb = (int)std::min<int64_t>((n + 256) / 256, kNumSMs * 8);
  k_radix_starts<<<sb, 256, 0, st>>>(keyS, n, M, S, cell_start, sub_start);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_bin(const float* x, const float* v, int64_t ldv, const float* w, int64_t n,
                        int32_t dv, double eta, int32_t M, int32_t S, int32_t* perm,
                        int32_t* cell_start, int32_t* sub_start, float* xv, float* sw,
                        void* scratch, size_t scratch_bytes, void* stream) {
  if (n < 0 || n > INT32_MAX || M < 1 || S < 1 || !(eta > 0) || (dv != 2 && dv != 3))
    return SPIC_ERR_ARG;
  if ((int64_t)M * S > 32768) return SPIC_ERR_UNSUPPORTED;
  if (xv && !v) return SPIC_ERR_ARG;
  BinPlan p = bin_plan(n, M, S);
  if (scratch_bytes < spic_bin_scratch_bytes(n, M, S)) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* counts = (int32_t*)scratch;
  int32_t* bsum = counts + p.counts_elems;
  const double L = (double)M * eta;
  if (n == 0) {
    cudaMemsetAsync(cell_start, 0, sizeof(int32_t) * (M + 1), st);
    if (sub_start) cudaMemsetAsync(sub_start, 0, sizeof(int32_t) * ((size_t)M * S + 1), st);
    SPIC_CHECK_LAUNCH();
    return SPIC_OK;
  }
  if (!bin_use_counting(n))
    return bin_radix(x, v, ldv, w, n, dv, eta, M, S, perm, cell_start, sub_start, xv, sw, scratch,
                     st);
  size_t smem_count = sizeof(int) * p.K;
  if (smem_count > 48 * 1024)
    cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_count);
  k_bin_count<<<p.n_tiles, 256, smem_count, st>>>(x, n, eta, M, S, p.T, p.n_tiles, counts); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  k_scan_reduce<<<(unsigned)p.nb_scan, kScanThreads, 0, st>>>(counts, p.counts_elems, bsum); spic::count_launch();
  k_scan_blocksums<<<1, kScanThreads, 0, st>>>(bsum, p.nb_scan); spic::count_launch();
  k_scan_apply<<<(unsigned)p.nb_scan, kScanThreads, 0, st>>>(counts, p.counts_elems, bsum); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  int sb = (int)std::min<int64_t>(((int64_t)p.K + 256) / 256, 1024);
  k_bin_starts<<<sb, 256, 0, st>>>(counts, M, S, p.n_tiles, (int32_t)n, cell_start, sub_start); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  size_t smem_scatter = sizeof(int) * (size_t)p.W * p.K;
  if (smem_scatter > 48 * 1024)
    cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_scatter);
  k_bin_scatter<<<p.n_tiles, p.W * 32, smem_scatter, st>>>(
      x, v, ldv, w, n, dv, eta, L, M, S, p.W, p.G, p.n_tiles, counts, perm, (float4*)xv,
      (float4*)sw); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_gather_scores(const float* s, int64_t lds, const int32_t* perm, int64_t n,
                                  int32_t dv, float* sw, int32_t* flags, void* stream) {
  if (n < 0 || (dv != 2 && dv != 3)) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  k_gather_scores<<<blocks, 256, 0, (cudaStream_t)stream>>>(s, lds, perm, n, dv, (float4*)sw, flags); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}
