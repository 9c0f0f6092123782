// dist.cu — per-rank kernels of the cell-range domain decomposition (dist_engine.py,
// SURVEY.md section 8(e)); the reference has no distributed path (its operators are the
// single-process ones replaced elsewhere in this library).
//
// A rank owns cells [lo, hi). After the push its particles lie within a few cells of that
// range; they are binned as they are (records R0, used for the deposit and the score
// training: both are sums over particles, so any partition of the particles gives the same
// global sums). For the collision each rank needs every particle of the cells [lo-g, hi+g)
// (g = 1 halo cell for the Landau stencil, 2 when blob scores of the halo are evaluated
// locally). One fixed-capacity message per ring neighbour carries them: to the left the
// rank's records of the cyclic cell range [mid, lo+g) (everything that left on the left
// side plus the first g owned cells), to the right [hi-g, mid). Messages are fixed-size so
// the exchange needs no count round-trip; the header gives the row count.
//
// Message layout: float4 pairs; pair 0 = header (int32: rows, rows inside the receiver's
// owned range, rows that did not fit, 0), pair r+1 = row r = (x, v0, v1, v2), (w, gid, 0, 0).
#include <algorithm>

#include "common.cuh"

namespace spic {

namespace {

constexpr int kDistThreads = 256;

__device__ __forceinline__ int seg_len(const int32_t* cs, int c0, int c1) {
  return c1 > c0 ? cs[c1] - cs[c0] : 0;
}

__global__ void __launch_bounds__(kDistThreads) k_dist_pack(
    const float* __restrict__ x, const float* __restrict__ v, int64_t ldv, int dv,
    const float* __restrict__ w, float uniform_w, const int32_t* __restrict__ gid,
    const int32_t* __restrict__ perm, const int32_t* __restrict__ cs, int sa0, int sa1, int sb0,
    int sb1, int ra0, int ra1, int rb0, int rb1, int64_t cap, float4* __restrict__ msg) {
  const int la = seg_len(cs, sa0, sa1), lb = seg_len(cs, sb0, sb1);
  const int64_t total = (int64_t)la + lb;
  const int64_t rows = min(total, cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int4 h;
    h.x = (int)rows;
    h.y = seg_len(cs, ra0, ra1) + seg_len(cs, rb0, rb1);
    h.z = (int)(total - rows);
    h.w = 0;
    reinterpret_cast<int4*>(msg)[0] = h;
    reinterpret_cast<int4*>(msg)[1] = make_int4(0, 0, 0, 0);
  }
  const int a0 = la ? cs[sa0] : 0, b0 = lb ? cs[sb0] : 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int k = r < la ? a0 + (int)r : b0 + (int)(r - la);
    const int i = perm[k];
    float4 A, B;
    A.x = x[i];
    A.y = v[i];
    A.z = v[ldv + i];
    A.w = dv == 3 ? v[2 * ldv + i] : 0.f;
    B.x = w ? w[i] : uniform_w;
    B.y = __int_as_float(gid[i]);
    B.z = 0.f;
    B.w = 0.f;
    msg[2 * (r + 1)] = A;
    msg[2 * (r + 1) + 1] = B;
  }
}

__global__ void __launch_bounds__(kDistThreads) k_dist_unpack(
    const float4* __restrict__ msg, int64_t rows, int64_t at, float* __restrict__ x,
    float* __restrict__ v, int64_t ldv, int dv, float* __restrict__ w, int32_t* __restrict__ gid) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const float4 A = msg[2 * (r + 1)], B = msg[2 * (r + 1) + 1];
    const int64_t i = at + r;
    x[i] = A.x;
    v[i] = A.y;
    v[ldv + i] = A.z;
    if (dv == 3) v[2 * ldv + i] = A.w;
    if (w) w[i] = B.x;
    gid[i] = __float_as_int(B.y);
  }
}

// Collision epilogue over the owned sorted range [cs[lo], cs[hi)) (read on device) with the
// new own state compacted in sorted order: out_*[k - cs[lo]]. Partials per block:
// [H_dot, E_K, P0, P1, P2, sum w] (the diagnostics row's d[3:9]).
template <int DV>
__global__ void __launch_bounds__(kDistThreads) k_dist_epilogue(
    const float* __restrict__ Us, int64_t ldu, const float4* __restrict__ sw,
    const int32_t* __restrict__ perm, const int32_t* __restrict__ cs, int lo, int hi,
    float nu_dt, const float* __restrict__ x, const float* __restrict__ v, int64_t ldv,
    const float* __restrict__ w, const int32_t* __restrict__ gid, float* __restrict__ ox,
    float* __restrict__ ov, int64_t ldo, float* __restrict__ ow, int32_t* __restrict__ ogid,
    double* __restrict__ partials, int32_t* flags) {
  __shared__ double scratch[(kDistThreads / 32) * 6];
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  bool bad = false;
  const int64_t k0 = cs[lo], k1 = cs[hi];
  for (int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = perm[k];
    const float4 S = sw[k];
    const float sv[3] = {S.x, S.y, S.z};
    const int64_t o = k - k0;
    double hd = 0.0, ek = 0.0;
#pragma unroll
    for (int d = 0; d < DV; ++d) {
      const float U = Us[d * ldu + k];
      hd += (double)sv[d] * (double)U;
      const float vn = fmaf(-nu_dt, U, v[d * ldv + i]);
      bad |= !isfinite(vn);
      ov[d * ldo + o] = vn;
      ek += (double)vn * (double)vn;
      acc[2 + d] += (double)S.w * (double)vn;
    }
    ox[o] = x[i];
    if (ow) ow[o] = w[i];
    ogid[o] = gid[i];
    acc[0] += (double)S.w * hd;
    acc[1] += 0.5 * (double)S.w * ek;
    acc[5] += (double)S.w;
  }
  if (bad) raise_flag(flags, SPIC_FLAG_NONFINITE_V);
  block_sum<6>(acc, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) partials[(size_t)blockIdx.x * 6 + q] = acc[q];
}

__global__ void k_dist_reduce(const double* __restrict__ part, int rows, int cols,
                              double* __restrict__ out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int col = wid; col < cols; col += nw) {
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += part[(size_t)r * cols + col];
    s = warp_sum(s);
    if (lane == 0) out[col] = s;
  }
}

constexpr int kDistEpiBlocks = 2 * kNumSMs;

}  // namespace

}  // namespace spic

using namespace spic;

extern "C" int spic_dist_pack(const float* x, const float* v, int64_t ldv, int32_t dv,
                              const float* w, float uniform_w, const int32_t* gid,
                              const int32_t* perm, const int32_t* cell_start, int32_t M,
                              const int32_t* send_cells, const int32_t* recv_cells, int64_t cap,
                              float* msg, void* stream) {
  if ((dv != 2 && dv != 3) || M < 1 || cap < 0 || !send_cells || !recv_cells) return SPIC_ERR_ARG;
  for (int k = 0; k < 4; ++k)
    if (send_cells[k] < 0 || send_cells[k] > M || recv_cells[k] < 0 || recv_cells[k] > M)
      return SPIC_ERR_ARG;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((cap + kDistThreads - 1) / kDistThreads,
                                                                  4 * kNumSMs));
  k_dist_pack<<<blocks, kDistThreads, 0, (cudaStream_t)stream>>>(
      x, v, ldv, dv, w, uniform_w, gid, perm, cell_start, send_cells[0], send_cells[1],
      send_cells[2], send_cells[3], recv_cells[0], recv_cells[1], recv_cells[2], recv_cells[3],
      cap, (float4*)msg);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_dist_unpack(const float* msg, int64_t rows, int64_t at, float* x, float* v,
                                int64_t ldv, int32_t dv, float* w, int32_t* gid, void* stream) {
  if ((dv != 2 && dv != 3) || rows < 0 || at < 0) return SPIC_ERR_ARG;
  if (rows == 0) return SPIC_OK;
  const int blocks = (int)std::min<int64_t>((rows + kDistThreads - 1) / kDistThreads, 4 * kNumSMs);
  k_dist_unpack<<<blocks, kDistThreads, 0, (cudaStream_t)stream>>>((const float4*)msg, rows, at, x,
                                                                    v, ldv, dv, w, gid);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" size_t spic_dist_epilogue_scratch_bytes(void) {
  return sizeof(double) * kDistEpiBlocks * 6;
}

extern "C" int spic_dist_epilogue(const float* U_sorted, int64_t ldu, const float* sw,
                                  const int32_t* perm, const int32_t* cell_start, int32_t lo,
                                  int32_t hi, int32_t dv, float nu_dt, const float* x,
                                  const float* v, int64_t ldv, const float* w,
                                  const int32_t* gid, float* out_x, float* out_v, int64_t ldo,
                                  float* out_w, int32_t* out_gid, double* red_out,
                                  int32_t* flags, void* scratch, size_t scratch_bytes,
                                  void* stream) {
  if ((dv != 2 && dv != 3) || lo < 0 || hi < lo) return SPIC_ERR_ARG;
  if (scratch_bytes < spic_dist_epilogue_scratch_bytes()) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)scratch;
  if (dv == 3)
    k_dist_epilogue<3><<<kDistEpiBlocks, kDistThreads, 0, st>>>(
        U_sorted, ldu, (const float4*)sw, perm, cell_start, lo, hi, nu_dt, x, v, ldv, w, gid,
        out_x, out_v, ldo, out_w, out_gid, part, flags);
  else
    k_dist_epilogue<2><<<kDistEpiBlocks, kDistThreads, 0, st>>>(
        U_sorted, ldu, (const float4*)sw, perm, cell_start, lo, hi, nu_dt, x, v, ldv, w, gid,
        out_x, out_v, ldo, out_w, out_gid, part, flags);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  k_dist_reduce<<<1, 256, 0, st>>>(part, kDistEpiBlocks, 6, red_out);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}
