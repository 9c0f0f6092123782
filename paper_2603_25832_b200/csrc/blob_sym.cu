// blob_sym.cu — the blob (Gaussian KDE) score sums over unordered pairs.
//
// Same estimator as blob.cu (ref: _blob_cell score.py:453-490, blob_score score.py:503-523):
//     den_i = sum_j w_j psi(dx) exp(-|v_i - v_j|^2 / 2h_i^2),  mu_i = sum_j (same) v_j,
//     s_i = (mu_i / den_i - v_i) / h_i^2,
// with h_i fixed or Silverman's per-cell bandwidth of the target's cell. The pair weight
// psi(dx) exp(-|dv|^2 / 2h^2) is symmetric whenever both targets use the same h (fixed h, or
// two records of one cell), so one evaluation of an unordered pair serves both sums:
//     den_i += w K, mu_i += w K v_j,   den_j += w K', mu_j += w K' v_i,
// where K' = K unless the pair straddles two cells of different Silverman bandwidths (then K'
// takes the second exponential with h_j). The enumeration, the streamed-side reduction and
// the slot fold are those of the antisymmetric Landau kernel (sym.cuh, landau_sym.cu); the
// ordered fallback runs behind the same device flag.
#include <type_traits>

#include "sym.cuh"

namespace spic {

constexpr int kBlobNC = 4;  // den, mu0, mu1, mu2

template <int NT, int RP, int MINB, bool MINIMG>
__global__ void __launch_bounds__(NT, MINB)
    k_blob_sym(const float4* __restrict__ xv, const int32_t* __restrict__ cell_start,
               const int32_t* __restrict__ sub_start, const int32_t* __restrict__ tile_start,
               const SymMeta* __restrict__ meta, const int64_t* __restrict__ off,
               const int32_t* __restrict__ symflag, int M, int S, float L, float wie, float wie2,
               const float* __restrict__ h_cell, float h_fixed, int nsplit, int split_fast,
               float* __restrict__ Upart, float* __restrict__ Jslot, int64_t n) {
  constexpr int TI = NT * 2 * RP;
  constexpr int NW = NT / 32;
  constexpr int NC = kBlobNC;
  extern __shared__ unsigned char s_dyn[];
  unsigned char* s_base = s_dyn + ((128u - (uint32_t)((uintptr_t)s_dyn & 127u)) & 127u);
  auto s_rec = reinterpret_cast<float4(*)[kSymTJ]>(s_base);
  auto s_jp = reinterpret_cast<float(*)[NW][kSymTJ * NC]>(s_base + sizeof(float4) * kSymStages * kSymTJ);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_base + sizeof(float4) * kSymStages * kSymTJ +
                                                sizeof(float) * 2 * NW * kSymTJ * NC);
  // split_fast: grid (nsplit, tiles), a tile's j-splits dispatched together (as k_landau_sym)
  const int tile = split_fast ? blockIdx.y : blockIdx.x;
  const int split = split_fast ? blockIdx.x : blockIdx.y;
  if (tile >= tile_start[M]) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < kSymStages * kSymTJ; k += NT)
    (&s_rec[0][0])[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSymStages; ++s) mbar_init(&s_bar[s], 1);
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
  const bool sym = *symflag != 0;
  const SymWindow win =
      sym_build_window(sym, meta, cell_start, sub_start, M, S, c, tile, t0, t1, L, MINIMG);
  const int64_t slot0 = sym ? off[tile] : 0;
  int wlen = 0;
  for (int s = 0; s < win.nseg; ++s) wlen += win.len[s];
  const int jlo = (int)(((long long)wlen * split) / nsplit);
  const int jhi = (int)(((long long)wlen * (split + 1)) / nsplit);
  const int ntiles = sym_window_tiles(win, jlo, jhi);
  const int cn = c + 1 == M ? 0 : c + 1;
  const float hi_ = h_cell ? h_cell[c] : h_fixed;
  const float hn_ = h_cell ? h_cell[cn] : h_fixed;
  // exp(-q2 / 2h^2) = 2^(kexp q2)
  const float kexp_i = -1.4426950408889634f * (0.5f / (hi_ * hi_));
  const float kexp_n = -1.4426950408889634f * (0.5f / (hn_ * hn_));
  const f2 kxi = mk2(kexp_i, kexp_i), kxn = mk2(kexp_n, kexp_n);

  f2 X[RP], V0[RP], V1[RP], V2[RP], DEN[RP], M0[RP], M1[RP], M2[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    // padding targets: x = NaN -> zero weight (see landau_sym.cu)
    float4 Ae = make_float4(__int_as_float(0x7fffffff), 0.f, 0.f, 0.f), Ao = Ae;
    const int pe = t0 + threadIdx.x + (2 * r) * NT, po = pe + NT;
    if (pe < t1) Ae = xv[pe];
    if (po < t1) Ao = xv[po];
    X[r] = mk2(Ae.x, Ao.x);
    V0[r] = mk2(Ae.y, Ao.y); V1[r] = mk2(Ae.z, Ao.z); V2[r] = mk2(Ae.w, Ao.w);
    DEN[r] = M0[r] = M1[r] = M2[r] = mk2(0.f, 0.f);
  }
  auto issue = [&](int q) {
    const SymTileDesc d = sym_window_tile(win, jlo, jhi, q);
    const int st = q % kSymStages;
    const int ru = min(kSymTJ, (d.cnt + 7) & ~7);
    for (int j = d.cnt; j < ru; ++j) s_rec[st][j].x = __int_as_float(0x7fffffff);
    mbar_expect_tx(&s_bar[st], (uint32_t)(d.cnt * sizeof(float4)));
    bulk_g2s(&s_rec[st][0], xv + d.pos, d.cnt * sizeof(float4), &s_bar[st]);
  };
  if (threadIdx.x == 0) {
    fence_proxy_async();
    for (int q = 0; q < min(ntiles, kSymStages); ++q) issue(q);
  }
  __syncthreads();
  const f2 W1c = mk2(wie, wie), nW2 = mk2(-wie2, -wie2);
  const f2 invL2 = mk2(1.0f / L, 1.0f / L), negL2 = mk2(-L, -L);
  const uint32_t mofs = (uint32_t)(((lane >> 2) & 7) * sizeof(float4));

  for (int q = 0; q < ntiles; ++q) {
    const int st = q % kSymStages;
    const SymTileDesc d = sym_window_tile(win, jlo, jhi, q);
    f2 XA[RP];
    const f2 sh = mk2(d.shift, d.shift);
#pragma unroll
    for (int r = 0; r < RP; ++r) XA[r] = sub2(X[r], sh);
    mbar_wait(&s_bar[st], (uint32_t)((q / kSymStages) & 1));
    if (!d.two) {
      const float4* __restrict__ P = s_rec[st];
#pragma unroll 2
      for (int jj = 0; jj < d.cnt; ++jj) {
        const float4 A = P[jj];
        const f2 xj = mk2(A.x, A.x), vj0 = mk2(A.y, A.y), vj1 = mk2(A.z, A.z), vj2 = mk2(A.w, A.w);
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          f2 dx = sub2(XA[r], xj);
          if (MINIMG) dx = fma2(rint2(mul2(dx, invL2)), negL2, dx);
          float ce_, co_;
          un2(fma2(abs2(dx), nW2, W1c), ce_, co_);
          ce_ = fmaxf(ce_, 0.f);
          co_ = fmaxf(co_, 0.f);
          const f2 z0 = sub2(V0[r], vj0), z1 = sub2(V1[r], vj1), z2 = sub2(V2[r], vj2);
          float ee, eo;
          un2(mul2(fma2(z2, z2, fma2(z1, z1, mul2(z0, z0))), kxi), ee, eo);
          const f2 kw = mul2(mk2(ce_, co_), mk2(exp2f(ee), exp2f(eo)));
          DEN[r] = add2(DEN[r], kw);
          M0[r] = fma2(kw, vj0, M0[r]);
          M1[r] = fma2(kw, vj1, M1[r]);
          M2[r] = fma2(kw, vj2, M2[r]);
        }
      }
    } else {
      // the records of seg2 belong to cell c+1: a different Silverman h needs its own weight
      const bool twoh = kexp_n != kexp_i && cn != c && d.pos >= cell_start[cn] &&
                        d.pos < cell_start[cn + 1];
      // one instantiation per case keeps the second exponential out of the common loop
      auto two_sided = [&](auto twoh_c) {
        constexpr bool TWOH = decltype(twoh_c)::value;
        float* jp = &s_jp[q & 1][wid][0];
        const uint32_t sbase = smem_u32(&s_rec[st][0]);
        for (int jb = 0; jb < d.cnt; jb += 8) {
          float P[NC][8];
          const uint32_t gb = (sbase + (uint32_t)jb * sizeof(float4)) | mofs;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 A = lds128(gb ^ (uint32_t)(k * sizeof(float4)));
            const f2 xj = mk2(A.x, A.x), vj0 = mk2(A.y, A.y), vj1 = mk2(A.z, A.z), vj2 = mk2(A.w, A.w);
            f2 JD, J0, J1, J2;
#pragma unroll
            for (int r = 0; r < RP; ++r) {
              f2 dx = sub2(XA[r], xj);
              if (MINIMG) dx = fma2(rint2(mul2(dx, invL2)), negL2, dx);
              float ce_, co_;
              un2(fma2(abs2(dx), nW2, W1c), ce_, co_);
              ce_ = fmaxf(ce_, 0.f);
              co_ = fmaxf(co_, 0.f);
              const f2 cp = mk2(ce_, co_);
              const f2 z0 = sub2(V0[r], vj0), z1 = sub2(V1[r], vj1), z2 = sub2(V2[r], vj2);
              const f2 q2 = fma2(z2, z2, fma2(z1, z1, mul2(z0, z0)));
              float ee, eo;
              un2(mul2(q2, kxi), ee, eo);
              const f2 kw = mul2(cp, mk2(exp2f(ee), exp2f(eo)));
              DEN[r] = add2(DEN[r], kw);
              M0[r] = fma2(kw, vj0, M0[r]);
              M1[r] = fma2(kw, vj1, M1[r]);
              M2[r] = fma2(kw, vj2, M2[r]);
              f2 kj = kw;
              if (TWOH) {
                un2(mul2(q2, kxn), ee, eo);
                kj = mul2(cp, mk2(exp2f(ee), exp2f(eo)));
              }
              if (r == 0) {
                JD = kj; J0 = mul2(kj, V0[r]); J1 = mul2(kj, V1[r]); J2 = mul2(kj, V2[r]);
              } else {
                JD = add2(JD, kj);
                J0 = fma2(kj, V0[r], J0); J1 = fma2(kj, V1[r], J1); J2 = fma2(kj, V2[r], J2);
              }
            }
            float e, o;
            un2(JD, e, o); P[0][k] = e + o;
            un2(J0, e, o); P[1][k] = e + o;
            un2(J1, e, o); P[2][k] = e + o;
            un2(J2, e, o); P[3][k] = e + o;
          }
          sym_reduce_scatter8<NC>(P);
          const int cc = lane & 3;
          jp[(jb + ((lane >> 2) & 7)) * NC + cc] =
              cc == 0 ? P[0][0] : (cc == 1 ? P[1][0] : (cc == 2 ? P[2][0] : P[3][0]));
        }
      };
      if (twoh)
        two_sided(std::true_type{});
      else
        two_sided(std::false_type{});
    }
    __syncthreads();
    if (threadIdx.x == 0 && q + kSymStages < ntiles) {
      fence_proxy_async();
      issue(q + kSymStages);
    }
    if (d.two) {  // fixed-order combine of the warps' j-side sums
      const float* jb = &s_jp[q & 1][0][0];
      float* dst = Jslot + (size_t)(slot0 + d.wofs) * NC;
      for (int k = threadIdx.x; k < d.cnt * NC; k += NT) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += jb[w * kSymTJ * NC + k];
        dst[k] = s;
      }
    }
  }
  float* out = Upart + (size_t)split * NC * n;
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    float de, dn, m0e, m0o, m1e, m1o, m2e, m2o;
    un2(DEN[r], de, dn);
    un2(M0[r], m0e, m0o);
    un2(M1[r], m1e, m1o);
    un2(M2[r], m2e, m2o);
    const int pe = t0 + threadIdx.x + (2 * r) * NT, po = pe + NT;
    if (pe < t1) { out[pe] = de; out[n + pe] = m0e; out[2 * n + pe] = m1e; out[3 * n + pe] = m2e; }
    if (po < t1) { out[po] = dn; out[n + po] = m0o; out[2 * n + po] = m1o; out[3 * n + po] = m2o; }
  }
}

// sum the splits and the record's slots in a fixed order, form s, isolated-particle check
// (as k_blob_fold in blob.cu)
__global__ void __launch_bounds__(256) k_blob_sym_fold(
    const float* __restrict__ Upart, int nsplit, int64_t n, const int32_t* __restrict__ cell_start,
    const int32_t* __restrict__ tile_start, const SymMeta* __restrict__ meta,
    const int64_t* __restrict__ off, const int32_t* __restrict__ symflag, int M, int TI,
    const float* __restrict__ Jslot, const float4* __restrict__ xv, float4* __restrict__ sw,
    const int32_t* __restrict__ perm, const float* __restrict__ h_cell, float h_fixed,
    long long* bad_pid, int32_t* flags) {
  const bool sym = *symflag != 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    float den = 0.f, m0 = 0.f, m1 = 0.f, m2 = 0.f;
    for (int q = 0; q < nsplit; ++q) {
      const float* pp = Upart + (size_t)q * kBlobNC * n;
      den += pp[k]; m0 += pp[n + k]; m1 += pp[2 * n + k]; m2 += pp[3 * n + k];
    }
    if (sym)
      sym_for_slots(k, cell_start, tile_start, meta, off, M, TI, [&](int64_t sl) {
        const float4 J = *reinterpret_cast<const float4*>(Jslot + sl * kBlobNC);
        den += J.x; m0 += J.y; m1 += J.z; m2 += J.w;
      });
    int lo = 0, hi = M;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
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
      r.z = (m2 * id - A.w) * ih2;
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

}  // namespace spic

using namespace spic;

namespace {

// kernel shape (threads, packed target pairs per thread, resident CTAs per SM), A/B by
// SPIC_BLOB_SYM_CFG: 0 = 128 x 2 x 4, 1 = 64 x 4 x 6, 2 = 64 x 5 x 5 (see landau_sym.cu)
struct BlobSymCfg {
  int nt, rp, minb;
  int ti() const { return nt * 2 * rp; }
};
constexpr BlobSymCfg kBlobSymCfgs[] = {{128, 2, 4}, {64, 4, 6}, {64, 5, 5}};
// default: 64-thread CTAs with 8 targets per thread as in landau_sym.cu (config 4: blob step
// 493.8 -> 480.4 ms, config 2: 16.79 -> 16.48 ms). 10 targets per thread gain another 1% at
// config 4 (475.3 ms) but lose at config 2 (17.3 ms: wave quantisation of the fewer, larger
// tiles); the shape does not depend on n, so scratch sized for a capacity fits any smaller run
BlobSymCfg blob_sym_cfg(int M, int64_t) {
  if (M <= 2) return kBlobSymCfgs[0];
  const char* e = getenv("SPIC_BLOB_SYM_CFG");
  const int k = e ? atoi(e) : 1;
  return kBlobSymCfgs[(k >= 0 && k < 3) ? k : 1];
}

constexpr size_t blob_sym_smem_bytes(int nt) {
  return 128 + sizeof(float4) * kSymStages * kSymTJ +
         sizeof(float) * 2 * (nt / 32) * kSymTJ * kBlobNC + sizeof(uint64_t) * kSymStages;
}

}  // namespace

int spic_blob_sym_nsplit(int64_t n, int32_t M) {
  const BlobSymCfg c = blob_sym_cfg(M, n);
  return pair_nsplit_slots(n, M, c.ti(), c.minb * kNumSMs);
}

size_t spic_blob_sym_scratch_bytes(int64_t n, int32_t M) {
  return sym_layout(nullptr, n, M, spic_blob_sym_nsplit(n, M), blob_sym_cfg(M, n).ti(), kBlobNC).bytes + 256;
}

// dv = 3, uniform weights; h_cell (nullable: fixed h_fixed) already computed
int spic_blob_sym_run(const float4* xv, float4* sw, const int32_t* perm, int64_t n,
                      const int32_t* cell_start, const int32_t* sub_start, int32_t M, int32_t S,
                      double eta, const float* h_cell, float h_fixed, float uniform_w,
                      long long* bad_pid, int32_t* flags, void* scratch, size_t scratch_bytes,
                      cudaStream_t st) {
  const int nsplit = spic_blob_sym_nsplit(n, M);
  const BlobSymCfg cfg = blob_sym_cfg(M, n);
  const int TI = cfg.ti();
  uintptr_t b = ((uintptr_t)scratch + 255) & ~(uintptr_t)255;
  SymScratch s = sym_layout((void*)b, n, M, nsplit, TI, kBlobNC);
  if (s.bytes + (b - (uintptr_t)scratch) > scratch_bytes) return SPIC_ERR_SCRATCH;
  const double L = (double)M * eta;
  const float wie = (float)((double)uniform_w / eta), wie2 = (float)((double)uniform_w / (eta * eta));
  const int32_t* ssp = (S > 1 && M >= 3) ? sub_start : nullptr;
  k_sym_tiles<<<1, 1024, 0, st>>>(cell_start, ssp, M, S, TI, 0, M, s.cap, s.tile_start,
                                  s.meta, s.off, s.flag);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  const int64_t ntile_grid = n / TI + M + 1;
  const char* sf = getenv("SPIC_SYM_ORDER");  // "t": tile-fastest grid (A/B)
  const int split_fast = (ntile_grid <= 65535 && !(sf && sf[0] == 't')) ? 1 : 0;
  dim3 grid = split_fast ? dim3((unsigned)nsplit, (unsigned)ntile_grid)
                         : dim3((unsigned)ntile_grid, (unsigned)nsplit);
#define SPIC_BLOBSYM(NT_, RP_, MB_, MI_)                                                         \
  do {                                                                                           \
    static bool attr = false;                                                                    \
    if (!attr) {                                                                                 \
      cudaFuncSetAttribute(k_blob_sym<NT_, RP_, MB_, MI_>,                                       \
                           cudaFuncAttributeMaxDynamicSharedMemorySize,                          \
                           (int)blob_sym_smem_bytes(NT_));                                       \
      attr = true;                                                                               \
    }                                                                                            \
    k_blob_sym<NT_, RP_, MB_, MI_><<<grid, NT_, blob_sym_smem_bytes(NT_), st>>>(                 \
        xv, cell_start, ssp, s.tile_start, s.meta, s.off, s.flag, M, S, (float)L, wie, wie2,     \
        h_cell, h_fixed, nsplit, split_fast, s.Upart, s.Jslot, n);                               \
  } while (0)
  if (M <= 2)
    SPIC_BLOBSYM(128, 2, 4, true);
  else if (cfg.nt == 64 && cfg.rp == 4)
    SPIC_BLOBSYM(64, 4, 6, false);
  else if (cfg.nt == 64)
    SPIC_BLOBSYM(64, 5, 5, false);
  else
    SPIC_BLOBSYM(128, 2, 4, false);
#undef SPIC_BLOBSYM
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  k_blob_sym_fold<<<blocks, 256, 0, st>>>(s.Upart, nsplit, n, cell_start, s.tile_start, s.meta,
                                          s.off, s.flag, M, TI, s.Jslot, xv, sw, perm,
                                          h_cell, h_fixed, bad_pid, flags);
  spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}
