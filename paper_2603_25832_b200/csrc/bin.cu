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

#include "common.cuh"

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

extern "C" size_t spic_bin_scratch_bytes(int64_t n, int32_t M, int32_t S) {
  if (M < 1 || S < 1) return 0;
  BinPlan p = bin_plan(n, M, S);
  return (p.counts_elems + p.nb_scan + 64) * sizeof(int32_t);
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
