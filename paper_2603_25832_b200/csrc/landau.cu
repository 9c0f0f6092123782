// landau.cu — the binned pairwise Landau collision velocity and its epilogue.
//
// Replaces _collision_cell (ref: collision.py:49-89), collision_force (collision.py:92-110)
// and collision_push (collision.py:113-116). For target i in cell c and every neighbour j in
// the periodic stencil {c-1, c, c+1}:
//     U_i += w_j psi(dx) |z|^(gamma+2) [ u - (z.u/|z|^2) z ],  z = v_i - v_j, u = s_i - s_j,
// with psi(dx) = max(0, 1 - |dx|/eta)/eta (the reference's |dx| >= eta skip) and pairs with
// |z|^2 <= 1e-24 contributing nothing (the reference's eps2 skip, incl. the self pair).
//
// Work decomposition (B200): one CTA per (cell, target tile of TI = NT*R targets, j-split).
// Targets live in registers (R per thread). The j-window — the stencil's sub-cells within
// eta of the target tile, up to 3 contiguous segments of the cell-sorted records — is
// streamed through shared memory in TJ-record stages by the bulk-copy engine
// (cp.async.bulk + mbarrier, NSTAGE-deep ring), and every thread sweeps every staged record
// (shared-memory broadcast). Periodic images are handled per segment by shifting the
// targets (x_i - shift) so the inner loop has no min-image code for M >= 3; M <= 2 uses the
// per-pair minimum image like the reference. Accumulation is float32 per (target, split) in
// a fixed order; splits are summed in a fixed order by the epilogue: deterministic.
#include <algorithm>

#include "pairs.cuh"

namespace spic {

// GMODE: 0 -> gamma = -3 (coef = 1/|z|), 1 -> gamma = -2 (coef = 1), 2 -> generic pow.
template <int DV, bool MINIMG, int GMODE, bool UNIFORM_W>
__global__ void __launch_bounds__(kLandauNT, 4)
    k_landau(const float4* __restrict__ xv, const float4* __restrict__ sw,
             const int32_t* __restrict__ cell_start, const int32_t* __restrict__ sub_start,
             const int32_t* __restrict__ tile_start, int M, int S, float L, float ie, float ie2,
             float wie, float wie2, float half_pow, int nsplit, float* __restrict__ Uout,
             int64_t ldu) {
  __shared__ alignas(128) float4 s_xv[kLandauStages][kLandauTJ];
  __shared__ alignas(128) float4 s_sw[kLandauStages][kLandauTJ];
  __shared__ alignas(8) uint64_t s_bar[kLandauStages];
  __shared__ int s_cell;

  const int bx = blockIdx.x;
  if (threadIdx.x == 0) {
    int lo = 0, hi = M;  // largest c with tile_start[c] <= bx
    if (bx >= tile_start[M]) {
      s_cell = -1;
    } else {
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (tile_start[mid] <= bx) lo = mid; else hi = mid;
      }
      s_cell = lo;
    }
    for (int s = 0; s < kLandauStages; ++s) mbar_init(&s_bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int c = s_cell;
  if (c < 0) return;
  const int cs = cell_start[c], ce = cell_start[c + 1];
  const int t0 = cs + (bx - tile_start[c]) * kLandauTI;
  const int t1 = min(t0 + kLandauTI, ce);
  Window win = build_window(cell_start, sub_start, M, S, c, t0, t1, L);
  int wlen = 0;
  for (int s = 0; s < win.nseg; ++s) wlen += win.len[s];
  const int jlo = (int)(((long long)wlen * blockIdx.y) / nsplit);
  const int jhi = (int)(((long long)wlen * (blockIdx.y + 1)) / nsplit);
  const int ntiles = window_tiles(win, jlo, jhi);

  // targets
  float xi[kLandauR], vi0[kLandauR], vi1[kLandauR], vi2[kLandauR];
  float si0[kLandauR], si1[kLandauR], si2[kLandauR];
  float a0[kLandauR], a1[kLandauR], a2[kLandauR];
#pragma unroll
  for (int r = 0; r < kLandauR; ++r) {
    int p = t0 + threadIdx.x + r * kLandauNT;
    float4 A = make_float4(1e30f, 0.f, 0.f, 0.f), B = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p < t1) {
      A = xv[p];
      B = sw[p];
    }
    xi[r] = A.x; vi0[r] = A.y; vi1[r] = A.z; vi2[r] = A.w;
    si0[r] = B.x; si1[r] = B.y; si2[r] = B.z;
    a0[r] = a1[r] = a2[r] = 0.f;
  }
  const float invL = 1.0f / L;

  auto issue = [&](int q) {
    TileDesc d = window_tile(win, jlo, jhi, q);
    int st = q % kLandauStages;
    mbar_expect_tx(&s_bar[st], (uint32_t)(2 * d.cnt * sizeof(float4)));
    bulk_g2s(&s_xv[st][0], xv + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
    bulk_g2s(&s_sw[st][0], sw + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
  };
  if (threadIdx.x == 0) {
    fence_proxy_async();
    for (int q = 0; q < min(ntiles, kLandauStages); ++q) issue(q);
  }

  for (int q = 0; q < ntiles; ++q) {
    const int st = q % kLandauStages;
    TileDesc d = window_tile(win, jlo, jhi, q);
    float xa[kLandauR];
#pragma unroll
    for (int r = 0; r < kLandauR; ++r) xa[r] = xi[r] - d.shift;
    mbar_wait(&s_bar[st], (uint32_t)((q / kLandauStages) & 1));
    const float4* __restrict__ P = s_xv[st];
    const float4* __restrict__ Q = s_sw[st];
#pragma unroll 4
    for (int jj = 0; jj < d.cnt; ++jj) {
      const float4 A = P[jj];
      const float4 B = Q[jj];
#pragma unroll
      for (int r = 0; r < kLandauR; ++r) {
        float dx = xa[r] - A.x;
        if (MINIMG) dx = fmaf(-L, rintf(dx * invL), dx);
        float cpsi;
        if (UNIFORM_W)
          cpsi = fmaxf(fmaf(-fabsf(dx), wie2, wie), 0.f);
        else
          cpsi = fmaxf(fmaf(-fabsf(dx), ie2, ie), 0.f) * B.w;
        const float z0 = vi0[r] - A.y, z1 = vi1[r] - A.z;
        const float u0 = si0[r] - B.x, u1 = si1[r] - B.y;
        float zz = fmaf(z1, z1, z0 * z0);
        float zu = fmaf(z1, u1, z0 * u0);
        float z2 = 0.f, u2 = 0.f;
        if (DV == 3) {
          z2 = vi2[r] - A.w;
          u2 = si2[r] - B.z;
          zz = fmaf(z2, z2, zz);
          zu = fmaf(z2, u2, zu);
        }
        const bool live = zz > kEps2;
        float cw, q2;
        if (GMODE == 0) {
          float rr = live ? rsqrtf(zz) : 0.f;
          cw = cpsi * rr;
          q2 = zu * (rr * rr);
        } else if (GMODE == 1) {
          float iz = live ? __frcp_rn(zz) : 0.f;
          cw = live ? cpsi : 0.f;
          q2 = zu * iz;
        } else {
          float iz = live ? __frcp_rn(zz) : 0.f;
          cw = live ? cpsi * exp2f(half_pow * __log2f(zz)) : 0.f;
          q2 = zu * iz;
        }
        a0[r] = fmaf(cw, fmaf(-q2, z0, u0), a0[r]);
        a1[r] = fmaf(cw, fmaf(-q2, z1, u1), a1[r]);
        if (DV == 3) a2[r] = fmaf(cw, fmaf(-q2, z2, u2), a2[r]);
      }
    }
    __syncthreads();  // everyone is done with stage st
    if (threadIdx.x == 0 && q + kLandauStages < ntiles) {
      fence_proxy_async();
      issue(q + kLandauStages);
    }
  }

  float* out = Uout + (size_t)blockIdx.y * DV * ldu;
#pragma unroll
  for (int r = 0; r < kLandauR; ++r) {
    int p = t0 + threadIdx.x + r * kLandauNT;
    if (p < t1) {
      out[p] = a0[r];
      out[ldu + p] = a1[r];
      if (DV == 3) out[2 * ldu + p] = a2[r];
    }
  }
}

// Epilogue: sum splits in order, scatter U to pid order, collision push, H_dot/E_K/P partials.
template <int DV>
__global__ void __launch_bounds__(256) k_collision_epilogue(
    const float* __restrict__ Us, int nsplit, int64_t n, const float4* __restrict__ sw,
    const int32_t* __restrict__ perm, float nu_dt, float* __restrict__ v, int64_t ldv,
    float* __restrict__ Upid, int64_t ldu, double* __restrict__ partials, int32_t* flags) {
  __shared__ double scratch[8 * 5];
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  bool bad = false;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    float U[3] = {0.f, 0.f, 0.f};
    for (int s = 0; s < nsplit; ++s)
#pragma unroll
      for (int d = 0; d < DV; ++d) U[d] += Us[((size_t)s * DV + d) * n + k];
    const int32_t i = perm[k];
    const float4 B = sw[k];
    const float sv[3] = {B.x, B.y, B.z};
    double hd = 0.0, ek = 0.0;
#pragma unroll
    for (int d = 0; d < DV; ++d) {
      if (Upid) Upid[d * ldu + i] = U[d];
      hd += (double)sv[d] * (double)U[d];
      float vn = v[d * ldv + i];
      if (nu_dt != 0.f) {
        vn = fmaf(-nu_dt, U[d], vn);
        v[d * ldv + i] = vn;
      }
      bad |= !isfinite(vn);
      ek += (double)vn * (double)vn;
      acc[2 + d] += (double)B.w * (double)vn;
    }
    acc[0] += (double)B.w * hd;
    acc[1] += 0.5 * (double)B.w * ek;
  }
  if (bad) raise_flag(flags, SPIC_FLAG_NONFINITE_V);
  block_sum<5>(acc, scratch);
  if (threadIdx.x == 0)
    for (int k = 0; k < 5; ++k) partials[(size_t)blockIdx.x * 5 + k] = acc[k];
}

// Deterministic column sums of a [rows][cols] float64 matrix (one warp per column).
__global__ void k_reduce_rows(const double* __restrict__ part, int rows, int cols,
                              double* __restrict__ out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int col = wid; col < cols; col += nw) {
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += part[(size_t)r * cols + col];
    s = warp_sum(s);
    if (lane == 0) out[col] = s;
  }
}

__global__ void k_count_live(const float4* __restrict__ xv, const int32_t* __restrict__ cell_start,
                             int M, float L, float eta, unsigned long long* count) {
  // one CTA per cell, threads over targets; full stencil with the same shifts as k_landau
  const int c = blockIdx.x;
  Window win = build_window(cell_start, nullptr, M, 1, c, 0, 0, L);
  unsigned long long local = 0;
  for (int t = cell_start[c] + threadIdx.x; t < cell_start[c + 1]; t += blockDim.x) {
    const float xi = xv[t].x;
    for (int s = 0; s < win.nseg; ++s) {
      const float xa = xi - win.shift[s];
      for (int j = win.start[s]; j < win.start[s] + win.len[s]; ++j) {
        float dx = xa - __ldg(&xv[j].x);
        if (M <= 2) dx = fmaf(-L, rintf(dx / L), dx);
        local += fabsf(dx) < eta;
      }
    }
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

constexpr int kEpiBlocks = 2 * kNumSMs;

template <int DV, bool MINIMG, int GMODE, bool UW>
static void launch_landau(dim3 grid, cudaStream_t st, const float4* xv, const float4* sw,
                          const int32_t* cs, const int32_t* ss, const int32_t* ts, int M, int S,
                          float L, float ie, float ie2, float wie, float wie2, float hp, int nsplit,
                          float* U, int64_t ldu) {
  k_landau<DV, MINIMG, GMODE, UW><<<grid, kLandauNT, 0, st>>>(xv, sw, cs, ss, ts, M, S, L, ie, ie2,
                                                              wie, wie2, hp, nsplit, U, ldu); spic::count_launch();
}

template <int DV, bool MINIMG, int GMODE>
static void dispatch_w(bool uw, dim3 g, cudaStream_t st, const float4* xv, const float4* sw,
                       const int32_t* cs, const int32_t* ss, const int32_t* ts, int M, int S,
                       float L, float ie, float ie2, float wie, float wie2, float hp, int ns,
                       float* U, int64_t ldu) {
  if (uw)
    launch_landau<DV, MINIMG, GMODE, true>(g, st, xv, sw, cs, ss, ts, M, S, L, ie, ie2, wie, wie2,
                                           hp, ns, U, ldu);
  else
    launch_landau<DV, MINIMG, GMODE, false>(g, st, xv, sw, cs, ss, ts, M, S, L, ie, ie2, wie, wie2,
                                            hp, ns, U, ldu);
}

template <int DV, bool MINIMG>
static void dispatch_g(int gm, bool uw, dim3 g, cudaStream_t st, const float4* xv,
                       const float4* sw, const int32_t* cs, const int32_t* ss, const int32_t* ts,
                       int M, int S, float L, float ie, float ie2, float wie, float wie2, float hp,
                       int ns, float* U, int64_t ldu) {
  if (gm == 0)
    dispatch_w<DV, MINIMG, 0>(uw, g, st, xv, sw, cs, ss, ts, M, S, L, ie, ie2, wie, wie2, hp, ns, U, ldu);
  else if (gm == 1)
    dispatch_w<DV, MINIMG, 1>(uw, g, st, xv, sw, cs, ss, ts, M, S, L, ie, ie2, wie, wie2, hp, ns, U, ldu);
  else
    dispatch_w<DV, MINIMG, 2>(uw, g, st, xv, sw, cs, ss, ts, M, S, L, ie, ie2, wie, wie2, hp, ns, U, ldu);
}

static int auto_nsplit(int64_t n, int M) {
  int64_t tiles = n / kLandauTI + (M + 1) / 2;
  if (tiles < 1) tiles = 1;
  int64_t want = (4 * kNumSMs + tiles - 1) / tiles;
  int64_t window = 3 * n / std::max(M, 1);  // records per window (upper bound)
  int64_t cap = std::max<int64_t>(1, window / 512);
  want = std::min<int64_t>(want, cap);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, 16));
}

__global__ void k_fold_splits(const float* __restrict__ part, int nsplit, int dv, int64_t n,
                              float* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n * dv;
       k += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < nsplit; ++q) s += part[(size_t)q * dv * n + k];
    out[k] = s;
  }
}

}  // namespace spic

using namespace spic;

extern "C" size_t spic_landau_scratch_bytes(int64_t n, int32_t M, int32_t dv, int32_t nsplit) {
  if (nsplit <= 0) nsplit = auto_nsplit(n, M);
  size_t b = sizeof(int32_t) * (size_t)(M + 1 + 31);
  if (nsplit > 1) b += sizeof(float) * (size_t)nsplit * dv * n + 256;
  return b;
}

extern "C" int spic_landau(const float* xv, const float* sw, int64_t n, int32_t dv,
                           const int32_t* cell_start, const int32_t* sub_start, int32_t M,
                           int32_t S, double eta, double gamma, float uniform_w, int32_t nsplit,
                           float* U_sorted, void* scratch, size_t scratch_bytes, void* stream) {
  if (n < 0 || n > INT32_MAX || M < 1 || S < 1 || !(eta > 0) || (dv != 2 && dv != 3))
    return SPIC_ERR_ARG;
  if (nsplit <= 0) nsplit = auto_nsplit(n, M);
  if (scratch_bytes < spic_landau_scratch_bytes(n, M, dv, nsplit)) return SPIC_ERR_SCRATCH;
  if (n == 0) return SPIC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* tile_start = (int32_t*)scratch;
  float* Upart = U_sorted;
  if (nsplit > 1) {
    uintptr_t p = (uintptr_t)(tile_start + M + 1 + 31);
    p = (p + 255) & ~(uintptr_t)255;
    Upart = (float*)p;
  }
  k_landau_tiles<<<1, 1024, 0, st>>>(cell_start, M, kLandauTI, tile_start); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  const double L = (double)M * eta;
  const float ie = (float)(1.0 / eta), ie2 = (float)(1.0 / (eta * eta));
  const float wie = (float)((double)uniform_w / eta), wie2 = (float)((double)uniform_w / (eta * eta));
  int gm = gamma == -3.0 ? 0 : (gamma == -2.0 ? 1 : 2);
  const float hp = (float)((gamma + 2.0) / 2.0);
  const bool minimg = M <= 2;
  const bool uw = uniform_w > 0.f;
  dim3 grid((unsigned)(n / kLandauTI + M + 1), (unsigned)nsplit);
  if (dv == 3) {
    if (minimg)
      dispatch_g<3, true>(gm, uw, grid, st, (const float4*)xv, (const float4*)sw, cell_start,
                          sub_start, tile_start, M, S, (float)L, ie, ie2, wie, wie2, hp, nsplit,
                          Upart, n);
    else
      dispatch_g<3, false>(gm, uw, grid, st, (const float4*)xv, (const float4*)sw, cell_start,
                           sub_start, tile_start, M, S, (float)L, ie, ie2, wie, wie2, hp, nsplit,
                           Upart, n);
  } else {
    if (minimg)
      dispatch_g<2, true>(gm, uw, grid, st, (const float4*)xv, (const float4*)sw, cell_start,
                          sub_start, tile_start, M, S, (float)L, ie, ie2, wie, wie2, hp, nsplit,
                          Upart, n);
    else
      dispatch_g<2, false>(gm, uw, grid, st, (const float4*)xv, (const float4*)sw, cell_start,
                           sub_start, tile_start, M, S, (float)L, ie, ie2, wie, wie2, hp, nsplit,
                           Upart, n);
  }
  SPIC_CHECK_LAUNCH();
  if (nsplit > 1) {  // fold the splits into U_sorted in a fixed order
    int blocks = (int)std::min<int64_t>((n * dv + 255) / 256, kNumSMs * 8);
    k_fold_splits<<<blocks, 256, 0, st>>>(Upart, nsplit, dv, n, U_sorted); spic::count_launch();
    SPIC_CHECK_LAUNCH();
  }
  return SPIC_OK;
}


extern "C" int spic_landau_fold(const float* U_part, int32_t nsplit, int32_t dv, int64_t n,
                                float* U_sorted, void* stream) {
  int blocks = (int)std::min<int64_t>((n * dv + 255) / 256, kNumSMs * 8);
  if (blocks < 1) return SPIC_OK;
  k_fold_splits<<<blocks, 256, 0, (cudaStream_t)stream>>>(U_part, nsplit, dv, n, U_sorted); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_collision_epilogue(const float* U_sorted, const float* sw, const int32_t* perm,
                                       int64_t n, int32_t dv, float nu_dt, float* v, int64_t ldv,
                                       float* U_pid, int64_t ldu, double* red_out, int32_t* flags,
                                       void* scratch, size_t scratch_bytes, void* stream) {
  if (n < 0 || (dv != 2 && dv != 3)) return SPIC_ERR_ARG;
  if (scratch_bytes < sizeof(double) * kEpiBlocks * 5) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)scratch;
  if (dv == 3)
    k_collision_epilogue<3><<<kEpiBlocks, 256, 0, st>>>(U_sorted, 1, n, (const float4*)sw, perm,
                                                        nu_dt, v, ldv, U_pid, ldu, part, flags);
  else
    k_collision_epilogue<2><<<kEpiBlocks, 256, 0, st>>>(U_sorted, 1, n, (const float4*)sw, perm,
                                                        nu_dt, v, ldv, U_pid, ldu, part, flags);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  if (red_out) {
    k_reduce_rows<<<1, 256, 0, st>>>(part, kEpiBlocks, 5, red_out); spic::count_launch();
    SPIC_CHECK_LAUNCH();
  }
  return SPIC_OK;
}

extern "C" int spic_count_live_pairs(const float* xv, int64_t n, const int32_t* cell_start,
                                     int32_t M, double eta, unsigned long long* count,
                                     void* stream) {
  if (n < 0 || M < 1) return SPIC_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
  if (n == 0) return SPIC_OK;
  k_count_live<<<M, 256, 0, st>>>((const float4*)xv, cell_start, M, (float)(M * eta), (float)eta,
                                  count); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}
