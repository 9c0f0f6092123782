// blob.cu — the blob (Gaussian KDE) score estimator on the cell stencil.
//
// Replaces _blob_cell (ref: score.py:453-490), silverman_bandwidth (score.py:493-500) and
// blob_score (score.py:503-523):
//     den_i = sum_j w_j psi(dx) exp(-|v_i - v_j|^2 / 2h^2),  mu_i = sum_j (same) v_j,
//     s_i = (mu_i / den_i - v_i) / h^2,
// with h fixed or Silverman's rule per cell over the (deduplicated) stencil velocities.
// Pair sweep as in landau.cu (bulk-copied j-tiles, targets in registers, sub-cell culling);
// the exponential is one MUFU.EX2. Splits of the j-window write (den, mu) partials that a
// fold kernel sums in a fixed order before forming s and checking den > 0 (isolated
// particle -> flag + the smallest (cell, pid) offender, matching the reference's choice).
#include <algorithm>

#include "pairs.cuh"
#include "f32x2.cuh"

namespace spic {

// per cell: count and sum of v (float64)
__global__ void k_blob_cellsum(const float4* __restrict__ xv, const int32_t* __restrict__ cell_start,
                               int dv, double* __restrict__ S1) {
  __shared__ double red[8 * 3];
  const int c = blockIdx.x;
  double a[3] = {0.0, 0.0, 0.0};
  for (int p = cell_start[c] + threadIdx.x; p < cell_start[c + 1]; p += blockDim.x) {
    const float4 A = xv[p];
    a[0] += A.y;
    a[1] += A.z;
    a[2] += A.w;
  }
  block_sum<3>(a, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) S1[c * 3 + k] = a[k];
}

// per cell: Silverman bandwidth over the deduplicated stencil (two-pass, float64)
__global__ void k_blob_silverman(const float4* __restrict__ xv, const int32_t* __restrict__ cell_start,
                                 int M, int dv, const double* __restrict__ S1,
                                 float* __restrict__ h_cell) {
  __shared__ double red[8 * 3];
  const int c = blockIdx.x;
  int cells[3], nc = 0;
  for (int d = -1; d <= 1; ++d) {
    int cd = ((c + d) % M + M) % M;
    bool dup = false;
    for (int q = 0; q < nc; ++q) dup |= cells[q] == cd;
    if (!dup) cells[nc++] = cd;
  }
  long long m = 0;
  double mean[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < nc; ++q) {
    m += cell_start[cells[q] + 1] - cell_start[cells[q]];
    for (int k = 0; k < 3; ++k) mean[k] += S1[cells[q] * 3 + k];
  }
  for (int k = 0; k < 3; ++k) mean[k] /= (double)(m > 0 ? m : 1);
  double ss[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < nc; ++q)
    for (int p = cell_start[cells[q]] + threadIdx.x; p < cell_start[cells[q] + 1]; p += blockDim.x) {
      const float4 A = xv[p];
      const double d0 = A.y - mean[0], d1 = A.z - mean[1], d2 = A.w - mean[2];
      ss[0] += d0 * d0;
      ss[1] += d1 * d1;
      ss[2] += d2 * d2;
    }
  block_sum<3>(ss, red);
  if (threadIdx.x == 0) {
    double sigma = 0.0;
    if (m > 1) {
      for (int k = 0; k < dv; ++k) sigma += sqrt(ss[k] / (double)(m - 1));
      sigma /= (double)dv;
    }
    double h = sigma * pow(4.0 / ((double)(dv + 2) * (double)m), 1.0 / (double)(dv + 4));
    h_cell[c] = (float)((h > 0.0 && isfinite(h)) ? h : 1.0);
  }
}

template <int DV, bool MINIMG, bool UNIFORM_W>
__global__ void __launch_bounds__(kLandauNT, 4)
    k_blob_pairs(const float4* __restrict__ xv, const float4* __restrict__ sw,
                 const int32_t* __restrict__ cell_start, const int32_t* __restrict__ sub_start,
                 const int32_t* __restrict__ tile_start, int M, int S, float L, float ie, float ie2,
                 float wie, float wie2, const float* __restrict__ h_cell, float h_fixed,
                 int nsplit, float* __restrict__ part, int64_t n) {
  __shared__ alignas(128) float4 s_xv[kLandauStages][kLandauTJ];
  __shared__ alignas(128) float4 s_sw[UNIFORM_W ? 1 : kLandauStages][kLandauTJ];
  __shared__ alignas(8) uint64_t s_bar[kLandauStages];
  __shared__ int s_cell;
  const int bx = blockIdx.x;
  if (threadIdx.x == 0) {
    int lo = 0, hi = M;
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
  const float h = h_cell ? h_cell[c] : h_fixed;
  const float kexp = -1.4426950408889634f * (0.5f / (h * h));  // exp(-q2/2h^2) = 2^(kexp q2)

  float xi[kLandauR], vi0[kLandauR], vi1[kLandauR], vi2[kLandauR];
  float den[kLandauR], m0[kLandauR], m1[kLandauR], m2[kLandauR];
#pragma unroll
  for (int r = 0; r < kLandauR; ++r) {
    int p = t0 + threadIdx.x + r * kLandauNT;
    float4 A = make_float4(1e30f, 0.f, 0.f, 0.f);
    if (p < t1) A = xv[p];
    xi[r] = A.x; vi0[r] = A.y; vi1[r] = A.z; vi2[r] = A.w;
    den[r] = m0[r] = m1[r] = m2[r] = 0.f;
  }
  const float invL = 1.0f / L;
  auto issue = [&](int q) {
    TileDesc d = window_tile(win, jlo, jhi, q);
    int st = q % kLandauStages;
    mbar_expect_tx(&s_bar[st], (uint32_t)((UNIFORM_W ? 1 : 2) * d.cnt * sizeof(float4)));
    bulk_g2s(&s_xv[st][0], xv + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
    if (!UNIFORM_W) bulk_g2s(&s_sw[st][0], sw + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
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
    const float4* __restrict__ Q = s_sw[UNIFORM_W ? 0 : st];
#pragma unroll 4
    for (int jj = 0; jj < d.cnt; ++jj) {
      const float4 A = P[jj];
      float wj = 0.f;
      if (!UNIFORM_W) wj = Q[jj].w;
#pragma unroll
      for (int r = 0; r < kLandauR; ++r) {
        float dx = xa[r] - A.x;
        if (MINIMG) dx = fmaf(-L, rintf(dx * invL), dx);
        float cpsi = UNIFORM_W ? fmaxf(fmaf(-fabsf(dx), wie2, wie), 0.f)
                               : fmaxf(fmaf(-fabsf(dx), ie2, ie), 0.f) * wj;
        const float z0 = vi0[r] - A.y, z1 = vi1[r] - A.z;
        float q2 = fmaf(z1, z1, z0 * z0);
        if (DV == 3) {
          const float z2 = vi2[r] - A.w;
          q2 = fmaf(z2, z2, q2);
        }
        const float kw = cpsi * exp2f(kexp * q2);
        den[r] += kw;
        m0[r] = fmaf(kw, A.y, m0[r]);
        m1[r] = fmaf(kw, A.z, m1[r]);
        if (DV == 3) m2[r] = fmaf(kw, A.w, m2[r]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && q + kLandauStages < ntiles) {
      fence_proxy_async();
      issue(q + kLandauStages);
    }
  }
  float* out = part + (size_t)blockIdx.y * 4 * n;
#pragma unroll
  for (int r = 0; r < kLandauR; ++r) {
    int p = t0 + threadIdx.x + r * kLandauNT;
    if (p < t1) {
      out[p] = den[r];
      out[n + p] = m0[r];
      out[2 * n + p] = m1[r];
      out[3 * n + p] = m2[r];
    }
  }
}

// Packed-FP32 blob sweep (dv = 3): 4 targets per thread as two f32x2 pairs, the j record
// broadcast in the B/C operand slots; one MUFU.EX2 per pair. Same partial layout as above.
template <bool MINIMG, bool UNIFORM_W>
__global__ void __launch_bounds__(kLandauNT, 4)
    k_blob_x2(const float4* __restrict__ xv, const float4* __restrict__ sw,
              const int32_t* __restrict__ cell_start, const int32_t* __restrict__ sub_start,
              const int32_t* __restrict__ tile_start, int M, int S, float L, float ie, float ie2,
              float wie, float wie2, const float* __restrict__ h_cell, float h_fixed, int nsplit,
              float* __restrict__ part, int64_t n) {
  constexpr int RP = 2;
  constexpr int TI = kLandauNT * 2 * RP;
  __shared__ alignas(128) float4 s_xv[kLandauStages][kLandauTJ];
  __shared__ alignas(128) float4 s_sw[UNIFORM_W ? 1 : kLandauStages][kLandauTJ];
  __shared__ alignas(8) uint64_t s_bar[kLandauStages];
  const int tile = blockIdx.x, split = blockIdx.y;
  if (tile >= tile_start[M]) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLandauStages; ++s) mbar_init(&s_bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  int lo = 0, hi = M;
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
  const float h = h_cell ? h_cell[c] : h_fixed;
  const float kexp = -1.4426950408889634f * (0.5f / (h * h));  // exp(-q2/2h^2) = 2^(kexp q2)

  f2 X[RP], V0[RP], V1[RP], V2[RP], DEN[RP], M0[RP], M1[RP], M2[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    float4 Ae = make_float4(1e30f, 0.f, 0.f, 0.f), Ao = Ae;
    const int pe = t0 + threadIdx.x + (2 * r) * kLandauNT, po = pe + kLandauNT;
    if (pe < t1) Ae = xv[pe];
    if (po < t1) Ao = xv[po];
    X[r] = mk2(Ae.x, Ao.x);
    V0[r] = mk2(Ae.y, Ao.y); V1[r] = mk2(Ae.z, Ao.z); V2[r] = mk2(Ae.w, Ao.w);
    DEN[r] = M0[r] = M1[r] = M2[r] = mk2(0.f, 0.f);
  }
  auto issue = [&](int q) {
    TileDesc d = window_tile(win, jlo, jhi, q);
    const int st = q % kLandauStages;
    mbar_expect_tx(&s_bar[st], (uint32_t)((UNIFORM_W ? 1 : 2) * d.cnt * sizeof(float4)));
    bulk_g2s(&s_xv[st][0], xv + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
    if (!UNIFORM_W) bulk_g2s(&s_sw[st][0], sw + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
  };
  if (threadIdx.x == 0) {
    fence_proxy_async();
    for (int q = 0; q < min(ntiles, kLandauStages); ++q) issue(q);
  }
  const f2 W1c = UNIFORM_W ? mk2(wie, wie) : mk2(ie, ie);
  const f2 nW2 = UNIFORM_W ? mk2(-wie2, -wie2) : mk2(-ie2, -ie2);
  const f2 invL2 = mk2(1.0f / L, 1.0f / L), negL2 = mk2(-L, -L), kx2 = mk2(kexp, kexp);
  for (int q = 0; q < ntiles; ++q) {
    const int st = q % kLandauStages;
    TileDesc d = window_tile(win, jlo, jhi, q);
    f2 XA[RP];
    const f2 sh = mk2(d.shift, d.shift);
#pragma unroll
    for (int r = 0; r < RP; ++r) XA[r] = sub2(X[r], sh);
    mbar_wait(&s_bar[st], (uint32_t)((q / kLandauStages) & 1));
    const float4* __restrict__ P = s_xv[st];
    const float4* __restrict__ Q = s_sw[UNIFORM_W ? 0 : st];
#pragma unroll 2
    for (int jj = 0; jj < d.cnt; ++jj) {
      const float4 A = P[jj];
      const float wj = UNIFORM_W ? 1.f : Q[jj].w;
      const f2 xj = mk2(A.x, A.x), vj0 = mk2(A.y, A.y), vj1 = mk2(A.z, A.z), vj2 = mk2(A.w, A.w);
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        f2 dx = sub2(XA[r], xj);
        if (MINIMG) dx = fma2(rint2(mul2(dx, invL2)), negL2, dx);
        float ce, co;
        un2(fma2(abs2(dx), nW2, W1c), ce, co);
        ce = fmaxf(ce, 0.f);
        co = fmaxf(co, 0.f);
        if (!UNIFORM_W) {
          ce *= wj;
          co *= wj;
        }
        const f2 z0 = sub2(V0[r], vj0), z1 = sub2(V1[r], vj1), z2 = sub2(V2[r], vj2);
        float ee, eo;
        un2(mul2(fma2(z2, z2, fma2(z1, z1, mul2(z0, z0))), kx2), ee, eo);
        const f2 kw = mul2(mk2(ce, co), mk2(exp2f(ee), exp2f(eo)));
        DEN[r] = add2(DEN[r], kw);
        M0[r] = fma2(kw, vj0, M0[r]);
        M1[r] = fma2(kw, vj1, M1[r]);
        M2[r] = fma2(kw, vj2, M2[r]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && q + kLandauStages < ntiles) {
      fence_proxy_async();
      issue(q + kLandauStages);
    }
  }
  float* out = part + (size_t)split * 4 * n;
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    float de, dn, m0e, m0o, m1e, m1o, m2e, m2o;
    un2(DEN[r], de, dn);
    un2(M0[r], m0e, m0o);
    un2(M1[r], m1e, m1o);
    un2(M2[r], m2e, m2o);
    const int pe = t0 + threadIdx.x + (2 * r) * kLandauNT, po = pe + kLandauNT;
    if (pe < t1) { out[pe] = de; out[n + pe] = m0e; out[2 * n + pe] = m1e; out[3 * n + pe] = m2e; }
    if (po < t1) { out[po] = dn; out[n + po] = m0o; out[2 * n + po] = m1o; out[3 * n + po] = m2o; }
  }
}

// fold splits (fixed order), form s, isolated-particle check
__global__ void k_blob_fold(const float* __restrict__ part, int nsplit, int64_t n, int dv,
                            const float4* __restrict__ xv, float4* __restrict__ sw,
                            const int32_t* __restrict__ perm, const int32_t* __restrict__ cell_start,
                            int M, const float* __restrict__ h_cell, float h_fixed,
                            long long* bad_pid, int32_t* flags) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    float den = 0.f, m0 = 0.f, m1 = 0.f, m2 = 0.f;
    for (int q = 0; q < nsplit; ++q) {
      const float* pp = part + (size_t)q * 4 * n;
      den += pp[k];
      m0 += pp[n + k];
      m1 += pp[2 * n + k];
      m2 += pp[3 * n + k];
    }
    // cell of sorted position k (binary search; only needed for h and the error order)
    int lo = 0, hi = M;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (cell_start[mid] <= k) lo = mid; else hi = mid;
    }
    const float h = h_cell ? h_cell[lo] : h_fixed;
    const float ih2 = 1.f / (h * h);
    const float4 A = xv[k];
    float4 r = sw[k];
    bool bad = !(den > 0.f);
    if (!bad) {
      const float id = 1.f / den;
      r.x = (m0 * id - A.y) * ih2;
      r.y = (m1 * id - A.z) * ih2;
      r.z = dv > 2 ? (m2 * id - A.w) * ih2 : 0.f;
      bad = !(isfinite(r.x) && isfinite(r.y) && isfinite(r.z));
    } else {
      r.x = r.y = r.z = 0.f;
    }
    sw[k] = r;
    if (bad) {
      raise_flag(flags, SPIC_FLAG_ISOLATED);
      if (bad_pid) atomicMin(bad_pid, ((long long)lo << 32) | (long long)perm[k]);
    }
  }
}

static int blob_nsplit(int64_t n, int M, int dv) {
  return pair_nsplit(n, M, dv == 3 ? kLandauNT * 4 : kLandauTI);
}

}  // namespace spic

using namespace spic;

// symmetric (unordered-pair) path, blob_sym.cu
size_t spic_blob_sym_scratch_bytes(int64_t n, int32_t M);
int spic_blob_sym_run(const float4* xv, float4* sw, const int32_t* perm, int64_t n,
                      const int32_t* cell_start, const int32_t* sub_start, int32_t M, int32_t S,
                      double eta, const float* h_cell, float h_fixed, float uniform_w,
                      long long* bad_pid, int32_t* flags, void* scratch, size_t scratch_bytes,
                      cudaStream_t st);

// SPIC_BLOB_VARIANT=o selects the ordered sweep (A/B checks)
static bool blob_ordered_forced() {
  const char* e = getenv("SPIC_BLOB_VARIANT");
  return e && e[0] == 'o';
}

static size_t blob_s1_bytes(int32_t M) { return (sizeof(double) * 3 * (size_t)M + 255) & ~(size_t)255; }

extern "C" size_t spic_blob_scratch_bytes(int64_t n, int32_t M, int32_t dv) {
  int ns = blob_nsplit(n, M, dv);
  size_t b = sizeof(float) * (size_t)ns * 4 * n + sizeof(double) * 3 * (size_t)M +
             sizeof(int32_t) * (M + 1) + 1024;
  if (dv == 3 && !blob_ordered_forced())
    b = std::max(b, blob_s1_bytes(M) + spic_blob_sym_scratch_bytes(n, M) + 256);
  return b;
}

extern "C" int spic_blob(const float* xv, float* sw, const int32_t* perm, int64_t n, int32_t dv,
                         const int32_t* cell_start, const int32_t* sub_start, int32_t M, int32_t S,
                         double eta, double bandwidth, float uniform_w, float* h_cell,
                         long long* bad_pid, int32_t* flags, void* scratch, size_t scratch_bytes,
                         void* stream) {
  if (n < 0 || n > INT32_MAX || M < 1 || S < 1 || !(eta > 0) || (dv != 2 && dv != 3))
    return SPIC_ERR_ARG;
  if (scratch_bytes < spic_blob_scratch_bytes(n, M, dv)) return SPIC_ERR_SCRATCH;
  if (bandwidth <= 0 && !h_cell) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int ns = blob_nsplit(n, M, dv);
  const bool symp = dv == 3 && uniform_w > 0.f && !blob_ordered_forced();
  float* part = (float*)scratch;
  uintptr_t pp = (uintptr_t)(part + (size_t)ns * 4 * n);
  pp = (pp + 255) & ~(uintptr_t)255;
  if (symp) pp = ((uintptr_t)scratch + 255) & ~(uintptr_t)255;  // S1 first, then the sym region
  double* S1 = (double*)pp;
  int32_t* tile_start = (int32_t*)(S1 + 3 * (size_t)M);
  const float4* xv4 = (const float4*)xv;
  const float* hc = nullptr;
  if (bandwidth <= 0) {
    k_blob_cellsum<<<M, 256, 0, st>>>(xv4, cell_start, dv, S1); spic::count_launch();
    k_blob_silverman<<<M, 256, 0, st>>>(xv4, cell_start, M, dv, S1, h_cell); spic::count_launch();
    SPIC_CHECK_LAUNCH();
    hc = h_cell;
  }
  if (symp) {
    char* sr = (char*)S1 + blob_s1_bytes(M);
    const size_t used = (size_t)(sr - (char*)scratch);
    return spic_blob_sym_run(xv4, (float4*)sw, perm, n, cell_start, sub_start, M, S, eta, hc,
                             (float)bandwidth, uniform_w, bad_pid, flags, sr,
                             scratch_bytes > used ? scratch_bytes - used : 0, st);
  }
  const bool packed = dv == 3;
  const int TI = packed ? kLandauNT * 4 : kLandauTI;
  k_landau_tiles<<<1, 1024, 0, st>>>(cell_start, M, TI, tile_start); spic::count_launch();
  const double L = (double)M * eta;
  const float ie = (float)(1.0 / eta), ie2 = (float)(1.0 / (eta * eta));
  const float wie = (float)((double)uniform_w / eta), wie2 = (float)((double)uniform_w / (eta * eta));
  dim3 grid((unsigned)(n / TI + M + 1), (unsigned)ns);
  const bool mi = M <= 2, uw = uniform_w > 0.f;
  const float hf = (float)bandwidth;
  if (packed) {
#define SPIC_BLOBX(MI_, UW_)                                                                   \
  k_blob_x2<MI_, UW_><<<grid, kLandauNT, 0, st>>>(xv4, (const float4*)sw, cell_start, sub_start, \
                                                  tile_start, M, S, (float)L, ie, ie2, wie, wie2, \
                                                  hc, hf, ns, part, n)
    if (mi) { if (uw) SPIC_BLOBX(true, true); else SPIC_BLOBX(true, false); }
    else { if (uw) SPIC_BLOBX(false, true); else SPIC_BLOBX(false, false); }
#undef SPIC_BLOBX
    spic::count_launch();
  } else {
#define SPIC_BLOB(DV_, MI_, UW_)                                                             \
  do {                                                                                       \
    k_blob_pairs<DV_, MI_, UW_><<<grid, kLandauNT, 0, st>>>(                                 \
        xv4, (const float4*)sw, cell_start, sub_start, tile_start, M, S, (float)L, ie, ie2, \
        wie, wie2, hc, hf, ns, part, n);                                                     \
    spic::count_launch();                                                                    \
  } while (0)
    if (mi) { if (uw) SPIC_BLOB(2, true, true); else SPIC_BLOB(2, true, false); }
    else { if (uw) SPIC_BLOB(2, false, true); else SPIC_BLOB(2, false, false); }
#undef SPIC_BLOB
  }
  SPIC_CHECK_LAUNCH();
  int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  k_blob_fold<<<blocks, 256, 0, st>>>(part, ns, n, dv, xv4, (float4*)sw, perm, cell_start, M, hc,
                                      hf, bad_pid, flags); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}
