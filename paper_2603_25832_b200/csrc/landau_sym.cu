// landau_sym.cu — antisymmetric (unordered-pair) form of the binned Landau collision sum.
//
// Same operator as landau.cu (ref: collision.py:49-110): U_i = sum_j w_j T_ij with
//     T_ij = psi(dx) |z|^-1 [ u - (z.u/|z|^2) z ],  z = v_i - v_j, u = s_i - s_j.
// T is antisymmetric (T_ji = -T_ij: z and u both flip sign), so one evaluation of an
// unordered pair {i, j} serves both targets: U_i += w T, U_j -= w T (uniform weights).
// That halves the pair work of the ordered kernel (41 FLOP per unordered pair instead of
// 2 x 38 for the two ordered ones).
//
// Enumeration (M >= 3, dv = 3, gamma = -3, uniform w). Records are sorted by (cell, sub-cell).
// A target tile [t0, t1) of cell c owns the pairs it forms with its FORWARD window:
//   seg0 = [t0, t1)            the diagonal block, evaluated one-sided (both orders),
//   seg1 = [t1, ce)            the rest of cell c (every pair in a cell is within eta),
//   seg2 = prefix of cell c+1  through the sub-cell of the tile's last record (periodic
//                              shift +L for c = M-1); later sub-cells are beyond eta.
// Every unordered pair of the 3-cell stencil is thus evaluated exactly once: pairs inside a
// cell by the tile of the earlier record, pairs across the c|c+1 border by the tile in c.
//
// Accumulation is deterministic. The register (i) side sums in a fixed order per thread as
// in the ordered kernel. The streamed (j) side of each record is reduced over the CTA's
// threads (warp reduce-scatter over 8 records + fixed-order combine of the warps in shared
// memory) and written once per (tile, record) into a slot buffer; k_sym_fold sums a record's
// slots in a fixed order (tiles of its own cell before it, then the tiles of cell c-1 whose
// seg2 reaches it). The slot count is data dependent (~ n * n_cell / TI); if it exceeds the
// caller's scratch, the tile table clears a device flag and the same kernels run the ordered
// (full-stencil, one-sided) enumeration instead — graph-safe, no host synchronisation.
#include "sym.cuh"

namespace spic {

// |minimum image of dx| for M <= 2 (ref: collision.py:62-66) from a = |dx| (|dx| < L + ulp:
// positions lie in [0, L), quirk records at x - L): min(a, |L - a|), where L - a is exact
// for a >= L/2 (Sterbenz) — one packed subtract instead of the rint-based fold. A NaN
// padding record stays NaN (both operands NaN), so its weight max(NaN, 0) is still 0.
__device__ __forceinline__ f2 minimg_abs2(f2 a, f2 L2) {
  const f2 b = abs2(sub2(L2, a));
  float a0, a1, b0, b1;
  un2(a, a0, a1);
  un2(b, b0, b1);
  return mk2(fminf(a0, b0), fminf(a1, b1));
}

__device__ __forceinline__ bool sym_tile_cell(int c, int M, int c_lo, int c_hi, bool partial) {
  if (c >= c_lo && c < c_hi) return true;
  return partial && c == (c_lo - 1 + M) % M;
}

// Single CTA: tile_start[0..M] (targets tiles per cell, incl. the halo cell c_lo-1 of a
// partial range), per-tile SymMeta, slot offsets off[0..T], the symmetric-path flag.
__global__ void __launch_bounds__(1024) k_sym_tiles(
    const int32_t* __restrict__ cell_start, const int32_t* __restrict__ sub_start, int M, int S,
    int TI, int c_lo, int c_hi, int64_t cap_slots, int32_t* __restrict__ tile_start,
    SymMeta* __restrict__ meta, int64_t* __restrict__ off, int32_t* __restrict__ symflag) {
  __shared__ long long ws[33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool partial = (c_hi - c_lo) < M;
  // phase 1: tiles per cell, exclusive scan
  long long carry = 0;
  for (int base = 0; base < M; base += blockDim.x) {
    const int c = base + threadIdx.x;
    long long v = 0;
    if (c < M && sym_tile_cell(c, M, c_lo, c_hi, partial))
      v = (cell_start[c + 1] - cell_start[c] + TI - 1) / TI;
    long long inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      long long t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      long long s = lane < nw ? ws[lane] : 0;
      long long si = s;
      for (int o = 1; o < 32; o <<= 1) {
        long long t = __shfl_up_sync(0xffffffffu, si, o);
        if (lane >= o) si += t;
      }
      ws[lane] = si - s;
      if (lane == 31) ws[32] = si;
    }
    __syncthreads();
    if (c < M) tile_start[c] = (int)(carry + ws[wid] + inc - v);
    carry += ws[32];
    __syncthreads();
  }
  const int T = (int)carry;
  if (threadIdx.x == 0) {
    tile_start[M] = T;
    tile_start[M + 1] = 0;
  }
  __syncthreads();
  // phase 2: per-tile forward-window lengths and their exclusive scan
  long long ocarry = 0;
  for (int base = 0; base < T; base += blockDim.x) {
    const int t = base + threadIdx.x;
    long long F = 0;
    if (t < T) {
      int lo = 0, hi = M;  // largest c with tile_start[c] <= t
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (tile_start[mid] <= t) lo = mid; else hi = mid;
      }
      const int c = lo;
      const int cs = cell_start[c], ce = cell_start[c + 1];
      const int t1 = min(cs + (t - tile_start[c] + 1) * TI, ce);
      const bool halo = !(c >= c_lo && c < c_hi);
      const int cn = (c + 1) % M;
      int len2;
      if (M <= 2) {  // deduplicated stencil (per-pair minimum image): cell 0 pairs with cell 1
        len2 = (M == 2 && c == 0) ? cell_start[2] - cell_start[1] : 0;
      } else if (S > 1 && sub_start) {
        const int32_t* ss = sub_start + (size_t)c * S;
        int b = 0;  // sub-cell of the tile's last record
        for (int k = 1; k < S; ++k)
          if (ss[k] <= t1 - 1) b = k;
        // next-cell records at sub-cell offsets > b lie farther than eta from every target of
        // the tile (x_j - x_i > eta on the binning's own float64 cell coordinates; at a sub-cell
        // boundary the float64 rounding of x / eta can only misplace a pair whose weight is
        // ~1e-16 of psi(0)), so the prefix ends with sub-cell b
        len2 = sub_start[(size_t)cn * S + b + 1] - cell_start[cn];
      } else {
        len2 = cell_start[cn + 1] - cell_start[cn];
      }
      SymMeta m;
      m.len1 = halo ? -1 : ce - t1;
      m.len2 = len2;
      meta[t] = m;
      F = (long long)max(m.len1, 0) + len2;
    }
    long long inc = F;
    for (int o = 1; o < 32; o <<= 1) {
      long long x = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += x;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      long long s = lane < nw ? ws[lane] : 0;
      long long si = s;
      for (int o = 1; o < 32; o <<= 1) {
        long long x = __shfl_up_sync(0xffffffffu, si, o);
        if (lane >= o) si += x;
      }
      ws[lane] = si - s;
      if (lane == 31) ws[32] = si;
    }
    __syncthreads();
    if (t < T) off[t] = ocarry + ws[wid] + inc - F;
    ocarry += ws[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    off[T] = ocarry;
    *symflag = ocarry <= cap_slots ? 1 : 0;
  }
}

// One CTA per (target tile, j-split). NT threads, 4 targets per thread as two packed
// (even, odd) pairs; j records broadcast from shared memory (one-sided stages) or read in a
// per-lane XOR order inside groups of 8 (two-sided stages, so the warp reduce-scatter of the
// j-side needs no selects: lane l holds record (k ^ m_l), m_l = (l >> 2) & 7).
template <int NT, int RP, int MINB, bool MINIMG, int G>
__global__ void __launch_bounds__(NT, MINB)
    k_landau_sym(const float4* __restrict__ xv, const float4* __restrict__ sw,
                 const int32_t* __restrict__ cell_start, const int32_t* __restrict__ sub_start,
                 const int32_t* __restrict__ tile_start, const SymMeta* __restrict__ meta,
                 const int64_t* __restrict__ off, const int32_t* __restrict__ symflag, int M,
                 int S, float L, float wie, float wie2, int nsplit, int split_fast,
                 float* __restrict__ Upart,
                 float* __restrict__ Jslot, int64_t n) {
  constexpr int TI = NT * 2 * RP;
  constexpr int NW = NT / 32;
  // dynamic shared memory (128-aligned by hand): stages of [xv records | sw records] (the sw
  // half at a fixed byte offset), the double-buffered per-warp j-side sums, the mbarriers
  extern __shared__ unsigned char s_dyn[];
  unsigned char* s_base = s_dyn + ((128u - (uint32_t)((uintptr_t)s_dyn & 127u)) & 127u);
  auto s_rec = reinterpret_cast<float4(*)[2][kSymTJ]>(s_base);
  auto s_jp = reinterpret_cast<float(*)[NW][kSymTJ * 3]>(s_base + sizeof(float4) * kSymStages * 2 * kSymTJ);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_base + sizeof(float4) * kSymStages * 2 * kSymTJ +
                                                sizeof(float) * 2 * NW * kSymTJ * 3);
  // split_fast: grid (nsplit, tiles) — a tile's j-splits are dispatched together, tiles in
  // order, so the long windows (first tiles of a cell) start before the short ones
  const int tile = split_fast ? blockIdx.y : blockIdx.x;
  const int split = split_fast ? blockIdx.x : blockIdx.y;
  if (tile >= tile_start[M]) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // zero the stage buffers once (padding records beyond a stage's count must be finite)
  for (int k = threadIdx.x; k < kSymStages * 2 * kSymTJ; k += NT)
    (&s_rec[0][0][0])[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSymStages; ++s) mbar_init(&s_bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const f2 W1c = mk2(wie, wie), nW2 = mk2(-wie2, -wie2);
  const f2 L2 = mk2(L, L);
  int lo = 0, hi = M;  // cell of this tile
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(tile_start + mid) <= tile) lo = mid; else hi = mid;
  }
  const int c = lo;
  const int cs = cell_start[c], ce = cell_start[c + 1];
  const int t0 = cs + (tile - tile_start[c]) * TI;
  const int t1 = min(t0 + TI, ce);
  const bool sym = *symflag != 0;
  const SymWindow win =
      sym_build_window(sym, meta, cell_start, sub_start, M, S, c, tile, t0, t1, L, MINIMG);
  const int64_t slot0 = sym ? off[tile] : 0;
  int wlen = 0;
  for (int s = 0; s < win.nseg; ++s) wlen += win.len[s];
  const int jlo = (int)(((long long)wlen * split) / nsplit);
  const int jhi = (int)(((long long)wlen * (split + 1)) / nsplit);
  const int ntiles = sym_window_tiles(win, jlo, jhi);

  f2 X[RP], V0[RP], V1[RP], V2[RP], S0[RP], S1[RP], S2[RP], A0[RP], A1[RP], A2[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    // padding targets: x = NaN -> max(NaN, 0) = 0 weight (also under the minimum image,
    // which would fold a merely distant x back into the box), so they add nothing to the
    // j-side sums
    float4 Ae = make_float4(__int_as_float(0x7fffffff), 0.f, 0.f, 0.f), Be = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 Ao = Ae, Bo = Be;
    const int pe = t0 + threadIdx.x + (2 * r) * NT;
    const int po = pe + NT;
    if (pe < t1) { Ae = xv[pe]; Be = sw[pe]; }
    if (po < t1) { Ao = xv[po]; Bo = sw[po]; }
    X[r] = mk2(Ae.x, Ao.x);
    V0[r] = mk2(Ae.y, Ao.y); V1[r] = mk2(Ae.z, Ao.z); V2[r] = mk2(Ae.w, Ao.w);
    S0[r] = mk2(Be.x, Bo.x); S1[r] = mk2(Be.y, Bo.y); S2[r] = mk2(Be.z, Bo.z);
    A0[r] = A1[r] = A2[r] = mk2(0.f, 0.f);
  }
  auto issue = [&](int q) {
    const SymTileDesc d = sym_window_tile(win, jlo, jhi, q);
    const int st = q % kSymStages;
    // padding records up to the next group of 8: x = NaN -> zero weight (see the targets)
    const int ru = min(kSymTJ, (d.cnt + 7) & ~7);
    for (int j = d.cnt; j < ru; ++j) s_rec[st][0][j].x = __int_as_float(0x7fffffff);
    mbar_expect_tx(&s_bar[st], (uint32_t)(2 * d.cnt * sizeof(float4)));
    bulk_g2s(&s_rec[st][0][0], xv + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
    bulk_g2s(&s_rec[st][1][0], sw + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
  };
  if (threadIdx.x == 0) {
    fence_proxy_async();
    for (int q = 0; q < min(ntiles, kSymStages); ++q) issue(q);
  }
  __syncthreads();  // padding writes of the prologue stages
  // two-sided stages: groups of G records, lane l reads record k ^ m_l of each group
  constexpr int kLpr = 32 / G;  // lanes per record after the reduce-scatter
  const int m_l = (lane / kLpr) & (G - 1);
  const uint32_t mofs = (uint32_t)(m_l * sizeof(float4));
  constexpr uint32_t kSwOfs = kSymTJ * sizeof(float4);

  for (int q = 0; q < ntiles; ++q) {
    const int st = q % kSymStages;
    const SymTileDesc d = sym_window_tile(win, jlo, jhi, q);
    f2 XA[RP];
    const f2 sh = mk2(d.shift, d.shift);
#pragma unroll
    for (int r = 0; r < RP; ++r) XA[r] = sub2(X[r], sh);
    mbar_wait(&s_bar[st], (uint32_t)((q / kSymStages) & 1));
    const uint32_t sbase = smem_u32(&s_rec[st][0][0]);
    if (!d.two) {
      // one-sided: broadcast records, i-side only (the diagonal block / ordered fallback)
      const float4* __restrict__ P = s_rec[st][0];
      const float4* __restrict__ Q = s_rec[st][1];
#pragma unroll 2
      for (int jj = 0; jj < d.cnt; ++jj) {
        const float4 A = P[jj];
        const float4 B = Q[jj];
        const f2 xj = mk2(A.x, A.x), vj0 = mk2(A.y, A.y), vj1 = mk2(A.z, A.z), vj2 = mk2(A.w, A.w);
        const f2 sj0 = mk2(B.x, B.x), sj1 = mk2(B.y, B.y), sj2 = mk2(B.z, B.z);
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          f2 adx = abs2(sub2(XA[r], xj));
          if (MINIMG) adx = minimg_abs2(adx, L2);
          float ce_, co_;
          un2(fma2(adx, nW2, W1c), ce_, co_);
          ce_ = fmaxf(ce_, 0.f);
          co_ = fmaxf(co_, 0.f);
          const f2 z0 = sub2(V0[r], vj0), z1 = sub2(V1[r], vj1), z2 = sub2(V2[r], vj2);
          const f2 u0 = sub2(S0[r], sj0), u1 = sub2(S1[r], sj1), u2 = sub2(S2[r], sj2);
          const f2 zz = fma2(z2, z2, fma2(z1, z1, mul2(z0, z0)));
          const f2 zu = fma2(z2, u2, fma2(z1, u1, mul2(z0, u0)));
          float zze, zzo;
          un2(zz, zze, zzo);
          const float qe = rsqrtf(zze), qo = rsqrtf(zzo);
          const f2 rp = mk2(zze > kEps2 ? qe : 0.f, zzo > kEps2 ? qo : 0.f);
          const f2 cw = mul2(mk2(ce_, co_), rp);
          const f2 q = mul2(mul2(rp, rp), zu);
          A0[r] = fma2(cw, fnms2(q, z0, u0), A0[r]);
          A1[r] = fma2(cw, fnms2(q, z1, u1), A1[r]);
          A2[r] = fma2(cw, fnms2(q, z2, u2), A2[r]);
        }
      }
    } else {
      float* jp = &s_jp[q & 1][wid][0];
      for (int jb = 0; jb < d.cnt; jb += G) {
        float P0[G], P1[G], P2[G];
        const uint32_t gb = (sbase + (uint32_t)jb * sizeof(float4)) | mofs;
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const uint32_t a = gb ^ (uint32_t)(k * sizeof(float4));
          const float4 A = lds128(a);
          const float4 B = lds128(a + kSwOfs);
          const f2 xj = mk2(A.x, A.x), vj0 = mk2(A.y, A.y), vj1 = mk2(A.z, A.z), vj2 = mk2(A.w, A.w);
          const f2 sj0 = mk2(B.x, B.x), sj1 = mk2(B.y, B.y), sj2 = mk2(B.z, B.z);
          f2 J0, J1, J2;
#pragma unroll
          for (int r = 0; r < RP; ++r) {
            f2 adx = abs2(sub2(XA[r], xj));
            if (MINIMG) adx = minimg_abs2(adx, L2);
            float ce_, co_;
            un2(fma2(adx, nW2, W1c), ce_, co_);
            ce_ = fmaxf(ce_, 0.f);
            co_ = fmaxf(co_, 0.f);
            const f2 z0 = sub2(V0[r], vj0), z1 = sub2(V1[r], vj1), z2 = sub2(V2[r], vj2);
            const f2 u0 = sub2(S0[r], sj0), u1 = sub2(S1[r], sj1), u2 = sub2(S2[r], sj2);
            const f2 zz = fma2(z2, z2, fma2(z1, z1, mul2(z0, z0)));
            const f2 zu = fma2(z2, u2, fma2(z1, u1, mul2(z0, u0)));
            float zze, zzo;
            un2(zz, zze, zzo);
            const float qe = rsqrtf(zze), qo = rsqrtf(zzo);
            const f2 rp = mk2(zze > kEps2 ? qe : 0.f, zzo > kEps2 ? qo : 0.f);
            const f2 cw = mul2(mk2(ce_, co_), rp);
            const f2 q = mul2(mul2(rp, rp), zu);
            const f2 d0 = fnms2(q, z0, u0), d1 = fnms2(q, z1, u1), d2 = fnms2(q, z2, u2);
            A0[r] = fma2(cw, d0, A0[r]);
            A1[r] = fma2(cw, d1, A1[r]);
            A2[r] = fma2(cw, d2, A2[r]);
            if (r == 0) {
              J0 = mul2(cw, d0); J1 = mul2(cw, d1); J2 = mul2(cw, d2);
            } else {
              J0 = fma2(cw, d0, J0); J1 = fma2(cw, d1, J1); J2 = fma2(cw, d2, J2);
            }
          }
          float e, o;
          un2(J0, e, o); P0[k] = e + o;
          un2(J1, e, o); P1[k] = e + o;
          un2(J2, e, o); P2[k] = e + o;
        }
        float PP[3][G];
#pragma unroll
        for (int k = 0; k < G; ++k) { PP[0][k] = P0[k]; PP[1][k] = P1[k]; PP[2][k] = P2[k]; }
        if constexpr (G == 8) sym_reduce_scatter8<3>(PP); else sym_reduce_scatter4<3>(PP);
        P0[0] = PP[0][0]; P1[0] = PP[1][0]; P2[0] = PP[2][0];
        const int cc = lane & (kLpr - 1);
        if (cc < 3) jp[(jb + m_l) * 3 + cc] = cc == 0 ? P0[0] : (cc == 1 ? P1[0] : P2[0]);
      }
    }
    __syncthreads();  // stage st consumed; warp slices of a two-sided stage complete
    if (threadIdx.x == 0 && q + kSymStages < ntiles) {
      fence_proxy_async();
      issue(q + kSymStages);
    }
    if (d.two) {  // fixed-order combine of the warps' j-side sums: U_j -= w T
      const float* jb = &s_jp[q & 1][0][0];
      float* dst = Jslot + (size_t)(slot0 + d.wofs) * 3;
      for (int k = threadIdx.x; k < d.cnt * 3; k += NT) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += jb[w * kSymTJ * 3 + k];
        dst[k] = -s;
      }
    }
  }
  float* out = Upart + (size_t)split * 3 * n;
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    float a0e, a0o, a1e, a1o, a2e, a2o;
    un2(A0[r], a0e, a0o);
    un2(A1[r], a1e, a1o);
    un2(A2[r], a2e, a2o);
    const int pe = t0 + threadIdx.x + (2 * r) * NT;
    const int po = pe + NT;
    if (pe < t1) { out[pe] = a0e; out[n + pe] = a1e; out[2 * n + pe] = a2e; }
    if (po < t1) { out[po] = a0o; out[n + po] = a1o; out[2 * n + po] = a2o; }
  }
}

// U_sorted[d][p] = sum_split Upart + (symmetric path) the record's j-side slots, all in a
// fixed order: tiles of its own cell before its tile, then the tiles of cell c-1 whose seg2
// reaches it. Sorted positions [k0, k1) only (a domain rank's owned targets).
__global__ void __launch_bounds__(256) k_sym_fold(
    const float* __restrict__ Upart, int nsplit, int64_t n, const int32_t* __restrict__ cell_start,
    const int32_t* __restrict__ tile_start, const SymMeta* __restrict__ meta,
    const int64_t* __restrict__ off, const int32_t* __restrict__ symflag, int M, int TI,
    const float* __restrict__ Jslot, int c_lo, int c_hi, float* __restrict__ U) {
  const bool sym = *symflag != 0;
  const int64_t k0 = cell_start[c_lo], k1 = cell_start[c_hi];
  for (int64_t p = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < k1;
       p += (int64_t)gridDim.x * blockDim.x) {
    float u0 = 0.f, u1 = 0.f, u2 = 0.f;
    for (int s = 0; s < nsplit; ++s) {
      const float* P = Upart + (size_t)s * 3 * n;
      u0 += P[p]; u1 += P[n + p]; u2 += P[2 * n + p];
    }
    if (sym)
      sym_for_slots(p, cell_start, tile_start, meta, off, M, TI, [&](int64_t sl) {
        u0 += Jslot[sl * 3]; u1 += Jslot[sl * 3 + 1]; u2 += Jslot[sl * 3 + 2];
      });
    U[p] = u0; U[n + p] = u1; U[2 * n + p] = u2;
  }
}

}  // namespace spic

using namespace spic;

namespace {

constexpr size_t sym_smem_bytes(int NT) {
  return 128 + sizeof(float4) * kSymStages * 2 * kSymTJ + sizeof(float) * 2 * (NT / 32) * kSymTJ * 3 +
         sizeof(uint64_t) * kSymStages;
}

// kernel configuration: threads per CTA, packed target pairs per thread, resident CTAs per SM
struct SymCfg {
  int nt, rp, minb, g;  // g: records per j-side reduce-scatter group
  int ti() const { return nt * 2 * rp; }
};
constexpr SymCfg kSymCfgs[] = {{128, 2, 4, 8}, {128, 2, 3, 8}, {128, 3, 3, 8}, {256, 2, 2, 8},
                               {128, 3, 2, 8}, {128, 2, 5, 8}, {128, 2, 4, 4}, {128, 2, 5, 4},
                               {128, 2, 6, 4}, {128, 4, 3, 8}, {64, 4, 6, 8}, {64, 5, 5, 8},
                               {64, 5, 6, 8}, {64, 6, 5, 8}, {64, 5, 5, 4}, {128, 5, 3, 8}};
// default: 64 threads x 10 targets (5 packed pairs) per thread. ptxas settles at 168 registers
// under __launch_bounds__(64, 5), so six CTAs (12 warps) are resident per SM; the j-side
// reduce-scatter and the even + odd adds are amortised over 10 targets instead of 4, and a
// two-warp CTA loses less at its per-stage barriers (config 4: 298.3 -> 282.9 ms, config 2:
// 9.82 -> 9.38 ms; sweep in profiles/r2_pair_kernel_experiments.json)
constexpr int kSymDefault = 11;
constexpr int kNumSymCfgs = sizeof(kSymCfgs) / sizeof(kSymCfgs[0]);

SymCfg sym_cfg(int M) {
  if (M <= 2) return kSymCfgs[0];
  const char* e = getenv("SPIC_SYM_CFG");
  const int k = e ? atoi(e) : kSymDefault;
  return kSymCfgs[(k >= 0 && k < kNumSymCfgs) ? k : kSymDefault];
}

}  // namespace

extern "C" int spic_landau_tile_targets(int32_t M) { return sym_cfg(M).ti(); }

// nsplit for the symmetric kernel: whole waves of (CTAs per SM) x SMs
int spic_landau_sym_nsplit(int64_t n, int32_t M, int32_t m_occ) {
  const SymCfg c = sym_cfg(M);
  return pair_nsplit_slots(n, m_occ > 0 ? m_occ : M, c.ti(), c.minb * kNumSMs);
}

size_t spic_landau_sym_scratch_bytes(int64_t n, int32_t M, int32_t nsplit, int32_t m_occ) {
  if (nsplit <= 0) nsplit = spic_landau_sym_nsplit(n, M, m_occ);
  return sym_layout(nullptr, n, M, nsplit, sym_cfg(M).ti(), 3, m_occ).bytes + 256;
}

template <int NT, int RP, int MINB, bool MINIMG, int G = 8>
static void launch_sym(dim3 grid, cudaStream_t st, const float* xv, const float* sw,
                       const int32_t* cell_start, const int32_t* ssp, const SymScratch& s, int M,
                       int S, float L, float wie, float wie2, int nsplit, int split_fast,
                       int64_t n) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_landau_sym<NT, RP, MINB, MINIMG, G>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym_smem_bytes(NT));
    attr = true;
  }
  k_landau_sym<NT, RP, MINB, MINIMG, G><<<grid, NT, sym_smem_bytes(NT), st>>>(
      (const float4*)xv, (const float4*)sw, cell_start, ssp, s.tile_start, s.meta, s.off, s.flag,
      M, S, L, wie, wie2, nsplit, split_fast, s.Upart, s.Jslot, n);
}

int spic_landau_sym_run(const float* xv, const float* sw, int64_t n, const int32_t* cell_start,
                        const int32_t* sub_start, int32_t M, int32_t S, double eta,
                        float uniform_w, int32_t nsplit, int32_t c_lo, int32_t c_hi,
                        float* U_sorted, void* scratch, size_t scratch_bytes, void* stream) {
  const SymCfg cfg = sym_cfg(M);
  const int TI = cfg.ti();
  const int m_occ = (c_hi - c_lo) < M ? std::min<int>(M, (c_hi - c_lo) + 3) : M;
  if (nsplit <= 0) nsplit = spic_landau_sym_nsplit(n, M, m_occ);
  uintptr_t b = ((uintptr_t)scratch + 255) & ~(uintptr_t)255;
  SymScratch s = sym_layout((void*)b, n, M, nsplit, TI, 3, m_occ);
  if (s.bytes + (b - (uintptr_t)scratch) > scratch_bytes) return SPIC_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  const double L = (double)M * eta;
  const float wie = (float)((double)uniform_w / eta), wie2 = (float)((double)uniform_w / (eta * eta));
  k_sym_tiles<<<1, 1024, 0, st>>>(cell_start, (S > 1 && M >= 3) ? sub_start : nullptr, M, S, TI, c_lo, c_hi,
                                  s.cap, s.tile_start, s.meta, s.off, s.flag);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  const bool partial = (c_hi - c_lo) < M;
  const int64_t ncells = (c_hi - c_lo) + (partial ? 1 : 0);
  const int64_t ntile_grid = n / TI + ncells + 1;
  const char* sf = getenv("SPIC_SYM_ORDER");  // "t": tile-fastest grid (A/B)
  const int split_fast = (ntile_grid <= 65535 && !(sf && sf[0] == 't')) ? 1 : 0;
  dim3 grid = split_fast ? dim3((unsigned)nsplit, (unsigned)ntile_grid)
                         : dim3((unsigned)ntile_grid, (unsigned)nsplit);
  const int32_t* ssp = (S > 1 && M >= 3) ? sub_start : nullptr;
  const float Lf = (float)L;
  if (M <= 2)
    launch_sym<128, 2, 4, true>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
#define SPIC_SYM_CASE(NT_, RP_, MB_, G_)                                                        \
  else if (cfg.nt == NT_ && cfg.rp == RP_ && cfg.minb == MB_ && cfg.g == G_)                    \
    launch_sym<NT_, RP_, MB_, false, G_>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie,   \
                                         wie2, nsplit, split_fast, n);
  SPIC_SYM_CASE(64, 5, 5, 8)
  SPIC_SYM_CASE(64, 4, 6, 8)
  SPIC_SYM_CASE(64, 5, 6, 8)
  SPIC_SYM_CASE(64, 6, 5, 8)
  SPIC_SYM_CASE(64, 5, 5, 4)
  SPIC_SYM_CASE(128, 5, 3, 8)
#undef SPIC_SYM_CASE
  else if (cfg.rp == 4 && cfg.nt == 128)
    launch_sym<128, 4, 3, false>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.g == 4 && cfg.minb == 4)
    launch_sym<128, 2, 4, false, 4>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.g == 4 && cfg.minb == 5)
    launch_sym<128, 2, 5, false, 4>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.g == 4 && cfg.minb == 6)
    launch_sym<128, 2, 6, false, 4>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.minb == 5)
    launch_sym<128, 2, 5, false>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.nt == 256)
    launch_sym<256, 2, 2, false>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.rp == 3 && cfg.minb == 3)
    launch_sym<128, 3, 3, false>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.rp == 3)
    launch_sym<128, 3, 2, false>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else if (cfg.minb == 3)
    launch_sym<128, 2, 3, false>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  else
    launch_sym<128, 2, 4, false>(grid, st, xv, sw, cell_start, ssp, s, M, S, Lf, wie, wie2, nsplit, split_fast, n);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  if (blocks > 0) {  // owned sorted range [cell_start[c_lo], cell_start[c_hi]) read on device
    k_sym_fold<<<blocks, 256, 0, st>>>(s.Upart, nsplit, n, cell_start, s.tile_start, s.meta,
                                       s.off, s.flag, M, TI, s.Jslot, c_lo, c_hi, U_sorted);
    spic::count_launch();
    SPIC_CHECK_LAUNCH();
  }
  return SPIC_OK;
}
