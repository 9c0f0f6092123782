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
#include <cstdlib>

#include "pairs.cuh"
#include "f32x2.cuh"

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
          float iz = live ? fast_rcp(zz) : 0.f;
          cw = live ? cpsi : 0.f;
          q2 = zu * iz;
        } else {
          float iz = live ? fast_rcp(zz) : 0.f;
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

// ---- packed-FP32 (f32x2, sm_100) variant of the dominant case ---------------------------
// DV = 3, M >= 3, gamma = -3. Each thread owns 2*RP targets held as (even, odd) pairs in
// 64-bit registers so every arithmetic step is one FFMA2/FADD2/FMUL2 for two pairs; the
// broadcast j-record enters as a scalar operand. |dx| is taken with FMNMX (ALU pipe) and
// the eps2 test with FSETP+FSEL, keeping the FMA pipe for the 21 packed ops per two pairs.
template <int RP, int MINB, bool UNIFORM_W, bool MINIMG, int UNR = 2>
__global__ void __launch_bounds__(kLandauNT, MINB)
    k_landau_x2(const float4* __restrict__ xv, const float4* __restrict__ sw,
                const int32_t* __restrict__ cell_start, const int32_t* __restrict__ sub_start,
                int32_t* __restrict__ tile_start, int M, int S, float L, float ie, float ie2,
                float wie, float wie2, int nsplit, float* __restrict__ Uout, int64_t ldu) {
  // One CTA per work item (target tile, j-split): blockIdx.x = tile, blockIdx.y = split.
  // (A persistent atomic-queue variant raised register pressure past 128/thread and cost
  // more in register moves than it saved in tail; the host picks nsplit for full waves.)
  constexpr int TI = kLandauNT * 2 * RP;
  __shared__ alignas(128) float4 s_xv[kLandauStages][kLandauTJ];
  __shared__ alignas(128) float4 s_sw[kLandauStages][kLandauTJ];
  __shared__ alignas(8) uint64_t s_bar[kLandauStages];
  const int tile = blockIdx.x, split = blockIdx.y;
  if (tile >= tile_start[M]) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLandauStages; ++s) mbar_init(&s_bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const f2 W1c = UNIFORM_W ? mk2(wie, wie) : mk2(ie, ie);
  const f2 nW2 = UNIFORM_W ? mk2(-wie2, -wie2) : mk2(-ie2, -ie2);
  const f2 invL2 = mk2(1.0f / L, 1.0f / L), negL2 = mk2(-L, -L);
  const int qg = 0;
  {
    int lo = 0, hi = M;  // cell of this tile: largest c with tile_start[c] <= tile
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(tile_start + mid) <= tile) lo = mid; else hi = mid;
    }
    const int c = lo;
    const int cs = cell_start[c], ce = cell_start[c + 1];
    const int t0 = cs + (tile - tile_start[c]) * TI;
    const int t1 = min(t0 + TI, ce);
    Window win = build_window(cell_start, sub_start, M, S, c, t0, t1, L);
    int wlen = 0;
    for (int s = 0; s < win.nseg; ++s) wlen += win.len[s];
    const int jlo = (int)(((long long)wlen * split) / nsplit);
    const int jhi = (int)(((long long)wlen * (split + 1)) / nsplit);
    const int ntiles = window_tiles(win, jlo, jhi);

    f2 X[RP], V0[RP], V1[RP], V2[RP], S0[RP], S1[RP], S2[RP], A0[RP], A1[RP], A2[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      float4 Ae = make_float4(1e30f, 0.f, 0.f, 0.f), Be = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 Ao = Ae, Bo = Be;
      const int pe = t0 + threadIdx.x + (2 * r) * kLandauNT;
      const int po = pe + kLandauNT;
      if (pe < t1) { Ae = xv[pe]; Be = sw[pe]; }
      if (po < t1) { Ao = xv[po]; Bo = sw[po]; }
      X[r] = mk2(Ae.x, Ao.x);
      V0[r] = mk2(Ae.y, Ao.y); V1[r] = mk2(Ae.z, Ao.z); V2[r] = mk2(Ae.w, Ao.w);
      S0[r] = mk2(Be.x, Bo.x); S1[r] = mk2(Be.y, Bo.y); S2[r] = mk2(Be.z, Bo.z);
      A0[r] = A1[r] = A2[r] = mk2(0.f, 0.f);
    }
    auto issue = [&](int q) {
      TileDesc d = window_tile(win, jlo, jhi, q);
      const int st = (qg + q) % kLandauStages;
      mbar_expect_tx(&s_bar[st], (uint32_t)(2 * d.cnt * sizeof(float4)));
      bulk_g2s(&s_xv[st][0], xv + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
      bulk_g2s(&s_sw[st][0], sw + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
    };
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (int q = 0; q < min(ntiles, kLandauStages); ++q) issue(q);
    }
    for (int q = 0; q < ntiles; ++q) {
      const int st = (qg + q) % kLandauStages;
      TileDesc d = window_tile(win, jlo, jhi, q);
      f2 XA[RP];
      const f2 sh = mk2(d.shift, d.shift);
#pragma unroll
      for (int r = 0; r < RP; ++r) XA[r] = sub2(X[r], sh);
      mbar_wait(&s_bar[st], (uint32_t)(((qg + q) / kLandauStages) & 1));
      const float4* __restrict__ P = s_xv[st];
      const float4* __restrict__ Q = s_sw[st];
#pragma unroll UNR
      for (int jj = 0; jj < d.cnt; ++jj) {
        const float4 A = P[jj];
        const float4 B = Q[jj];
        const f2 xj = mk2(A.x, A.x), vj0 = mk2(A.y, A.y), vj1 = mk2(A.z, A.z), vj2 = mk2(A.w, A.w);
        const f2 sj0 = mk2(B.x, B.x), sj1 = mk2(B.y, B.y), sj2 = mk2(B.z, B.z);
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          f2 dx = sub2(XA[r], xj);
          if (MINIMG) dx = fma2(rint2(mul2(dx, invL2)), negL2, dx);  // M <= 2: minimum image
          // w psi(dx) = max(0, w/eta - |dx| w/eta^2)
          float ce, co;
          un2(fma2(abs2(dx), nW2, W1c), ce, co);
          ce = fmaxf(ce, 0.f);
          co = fmaxf(co, 0.f);
          if (!UNIFORM_W) {
            ce *= B.w;
            co *= B.w;
          }
          const f2 z0 = sub2(V0[r], vj0), z1 = sub2(V1[r], vj1), z2 = sub2(V2[r], vj2);
          const f2 u0 = sub2(S0[r], sj0), u1 = sub2(S1[r], sj1), u2 = sub2(S2[r], sj2);
          const f2 zz = fma2(z2, z2, fma2(z1, z1, mul2(z0, z0)));
          const f2 zu = fma2(z2, u2, fma2(z1, u1, mul2(z0, u0)));
          float zze, zzo;
          un2(zz, zze, zzo);
          const float qe = rsqrtf(zze), qo = rsqrtf(zzo);
          // 1/|z|, or 0 for the eps2-skipped pairs (incl. the self pair)
          const f2 rp = mk2(zze > kEps2 ? qe : 0.f, zzo > kEps2 ? qo : 0.f);
          const f2 cw = mul2(mk2(ce, co), rp);           // w psi / |z|
          const f2 q = mul2(mul2(rp, rp), zu);    // -(z.u)/|z|^2
          A0[r] = fma2(cw, fnms2(q, z0, u0), A0[r]);
          A1[r] = fma2(cw, fnms2(q, z1, u1), A1[r]);
          A2[r] = fma2(cw, fnms2(q, z2, u2), A2[r]);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && q + kLandauStages < ntiles) {
        fence_proxy_async();
        issue(q + kLandauStages);
      }
    }
    float* out = Uout + (size_t)split * 3 * ldu;
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      float a0e, a0o, a1e, a1o, a2e, a2o;
      un2(A0[r], a0e, a0o);
      un2(A1[r], a1e, a1o);
      un2(A2[r], a2e, a2o);
      const int pe = t0 + threadIdx.x + (2 * r) * kLandauNT;
      const int po = pe + kLandauNT;
      if (pe < t1) { out[pe] = a0e; out[ldu + pe] = a1e; out[2 * ldu + pe] = a2e; }
      if (po < t1) { out[po] = a0o; out[ldu + po] = a1o; out[2 * ldu + po] = a2o; }
    }
  }
}

// resident CTAs per SM of a kernel (cached) x SM count
template <typename K>
static int persistent_grid_unused(K kernel, int threads) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = kNumSMs;
  }
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0);
  return std::max(1, per) * sms;
}

// Epilogue: sum splits in order, scatter U to pid order, collision push, H_dot/E_K/P partials.
template <int DV>
__global__ void __launch_bounds__(256) k_collision_epilogue(
    const float* __restrict__ Us, int nsplit, int64_t n, const float4* __restrict__ sw,
    const int32_t* __restrict__ perm, float nu_dt, float* __restrict__ v, int64_t ldv,
    float* __restrict__ Upid, int64_t ldu, double* __restrict__ partials, int32_t* flags,
    int64_t k0, int64_t k1) {
  __shared__ double scratch[8 * 5];
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  bool bad = false;
  for (int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1;
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
constexpr int kLandauRP = 2;  // packed pairs per thread in k_landau_x2 (4 targets)

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

static int auto_nsplit(int64_t n, int M, int dv) {
  return pair_nsplit(n, M, dv == 3 ? kLandauNT * 2 * 2 : kLandauTI);
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

// antisymmetric (unordered-pair) path, landau_sym.cu
size_t spic_landau_sym_scratch_bytes(int64_t n, int32_t M, int32_t nsplit, int32_t m_occ);
int spic_landau_sym_run(const float* xv, const float* sw, int64_t n, const int32_t* cell_start,
                        const int32_t* sub_start, int32_t M, int32_t S, double eta,
                        float uniform_w, int32_t nsplit, int32_t c_lo, int32_t c_hi,
                        float* U_sorted, void* scratch, size_t scratch_bytes, void* stream);

// SPIC_LANDAU_VARIANT: unset -> antisymmetric kernel where eligible, 'o' -> ordered packed
// kernel, 's' -> ordered scalar kernel (A/B checks)
static char landau_variant() {
  const char* var = getenv("SPIC_LANDAU_VARIANT");
  return var ? var[0] : 0;
}

extern "C" size_t spic_landau_range_scratch_bytes(int64_t n, int32_t M, int32_t dv,
                                                   int32_t nsplit, int32_t c_lo, int32_t c_hi) {
  const int32_t ns = nsplit <= 0 ? auto_nsplit(n, M, dv) : nsplit;
  size_t b = sizeof(int32_t) * (size_t)(M + 1 + 31);
  if (ns > 1) b += sizeof(float) * (size_t)ns * dv * n + 256;
  const int32_t m_occ = (c_hi - c_lo) < M ? std::min<int32_t>(M, (c_hi - c_lo) + 3) : M;
  if (dv == 3 && landau_variant() == 0)
    b = std::max(b, spic_landau_sym_scratch_bytes(n, M, nsplit, m_occ));
  return b;
}

extern "C" size_t spic_landau_scratch_bytes(int64_t n, int32_t M, int32_t dv, int32_t nsplit) {
  return spic_landau_range_scratch_bytes(n, M, dv, nsplit, 0, M);
}

extern "C" int spic_landau_range(const float* xv, const float* sw, int64_t n, int32_t dv,
                                 const int32_t* cell_start, const int32_t* sub_start, int32_t M,
                                 int32_t S, double eta, double gamma, float uniform_w,
                                 int32_t nsplit, int32_t c_lo, int32_t c_hi, float* U_sorted,
                                 void* scratch, size_t scratch_bytes, void* stream);

extern "C" int spic_landau(const float* xv, const float* sw, int64_t n, int32_t dv,
                           const int32_t* cell_start, const int32_t* sub_start, int32_t M,
                           int32_t S, double eta, double gamma, float uniform_w, int32_t nsplit,
                           float* U_sorted, void* scratch, size_t scratch_bytes, void* stream) {
  return spic_landau_range(xv, sw, n, dv, cell_start, sub_start, M, S, eta, gamma, uniform_w,
                           nsplit, 0, M, U_sorted, scratch, scratch_bytes, stream);
}

extern "C" int spic_landau_range(const float* xv, const float* sw, int64_t n, int32_t dv,
                                 const int32_t* cell_start, const int32_t* sub_start, int32_t M,
                                 int32_t S, double eta, double gamma, float uniform_w,
                                 int32_t nsplit, int32_t c_lo, int32_t c_hi, float* U_sorted,
                                 void* scratch, size_t scratch_bytes, void* stream) {
  if (c_lo < 0 || c_hi > M || c_lo > c_hi) return SPIC_ERR_ARG;
  if (n < 0 || n > INT32_MAX || M < 1 || S < 1 || !(eta > 0) || (dv != 2 && dv != 3))
    return SPIC_ERR_ARG;
  if (scratch_bytes < spic_landau_range_scratch_bytes(n, M, dv, nsplit, c_lo, c_hi))
    return SPIC_ERR_SCRATCH;
  if (n == 0) return SPIC_OK;
  const char var = landau_variant();
  if (dv == 3 && gamma == -3.0 && uniform_w > 0.f && var == 0 &&
      (M >= 3 || (c_lo == 0 && c_hi == M)))
    return spic_landau_sym_run(xv, sw, n, cell_start, sub_start, M, S, eta, uniform_w, nsplit,
                               c_lo, c_hi, U_sorted, scratch, scratch_bytes, stream);
  if (nsplit <= 0) nsplit = auto_nsplit(n, M, dv);
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* tile_start = (int32_t*)scratch;
  float* Upart = U_sorted;
  if (nsplit > 1) {
    uintptr_t p = (uintptr_t)(tile_start + M + 1 + 31);
    p = (p + 255) & ~(uintptr_t)255;
    Upart = (float*)p;
  }
  const double L = (double)M * eta;
  const float ie = (float)(1.0 / eta), ie2 = (float)(1.0 / (eta * eta));
  const float wie = (float)((double)uniform_w / eta), wie2 = (float)((double)uniform_w / (eta * eta));
  int gm = gamma == -3.0 ? 0 : (gamma == -2.0 ? 1 : 2);
  const float hp = (float)((gamma + 2.0) / 2.0);
  const bool minimg = M <= 2;
  const bool uw = uniform_w > 0.f;
  // packed f32x2 kernel for the dominant case (dv = 3, M >= 3, Coulomb gamma = -3)
  // SPIC_LANDAU_VARIANT=s forces the scalar kernel (A/B checks); the packed configuration
  // (2 packed pairs per thread, 4 CTAs/SM, 2-way j unroll) won a sweep of RP 1..3, 2..8
  // CTAs/SM and unroll 1/2/4 on config 2
  const bool packed = dv == 3 && gm == 0 && var != 's';
  constexpr int rp = kLandauRP;
  const int TI = packed ? kLandauNT * 2 * rp : kLandauTI;
  k_landau_tiles<<<1, 1024, 0, st>>>(cell_start, M, TI, tile_start, c_lo, c_hi); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  dim3 grid((unsigned)(n / TI + M + 1), (unsigned)nsplit);
  if (packed) {
#define SPIC_X2(MINIMG_, UW_)                                                                 \
  k_landau_x2<kLandauRP, 4, UW_, MINIMG_, 2><<<grid, kLandauNT, 0, st>>>(                     \
      (const float4*)xv, (const float4*)sw, cell_start, sub_start, tile_start, M, S, (float)L, \
      ie, ie2, wie, wie2, nsplit, Upart, n)
    if (minimg) {
      if (uw) SPIC_X2(true, true); else SPIC_X2(true, false);
    } else {
      if (uw) SPIC_X2(false, true); else SPIC_X2(false, false);
    }
#undef SPIC_X2
    spic::count_launch();
  } else if (dv == 3) {
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

extern "C" int spic_collision_epilogue_range(const float* U_sorted, const float* sw,
                                             const int32_t* perm, int64_t n, int32_t dv,
                                             int64_t k0, int64_t k1, float nu_dt, float* v,
                                             int64_t ldv, float* U_pid, int64_t ldu,
                                             double* red_out, int32_t* flags, void* scratch,
                                             size_t scratch_bytes, void* stream) {
  if (n < 0 || (dv != 2 && dv != 3) || k0 < 0 || k1 > n || k0 > k1) return SPIC_ERR_ARG;
  if (scratch_bytes < sizeof(double) * kEpiBlocks * 5) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)scratch;
  if (dv == 3)
    k_collision_epilogue<3><<<kEpiBlocks, 256, 0, st>>>(U_sorted, 1, n, (const float4*)sw, perm,
                                                        nu_dt, v, ldv, U_pid, ldu, part, flags, k0, k1);
  else
    k_collision_epilogue<2><<<kEpiBlocks, 256, 0, st>>>(U_sorted, 1, n, (const float4*)sw, perm,
                                                        nu_dt, v, ldv, U_pid, ldu, part, flags, k0, k1);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  if (red_out) {
    k_reduce_rows<<<1, 256, 0, st>>>(part, kEpiBlocks, 5, red_out); spic::count_launch();
    SPIC_CHECK_LAUNCH();
  }
  return SPIC_OK;
}

extern "C" int spic_collision_epilogue(const float* U_sorted, const float* sw, const int32_t* perm,
                                       int64_t n, int32_t dv, float nu_dt, float* v, int64_t ldv,
                                       float* U_pid, int64_t ldu, double* red_out, int32_t* flags,
                                       void* scratch, size_t scratch_bytes, void* stream) {
  return spic_collision_epilogue_range(U_sorted, sw, perm, n, dv, 0, n, nu_dt, v, ldv, U_pid, ldu,
                                       red_out, flags, scratch, scratch_bytes, stream);
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
