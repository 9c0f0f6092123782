// sbtm.cu — the SBTM score network on device: forward pass, implicit-score-matching (ISM)
// loss + gradient partials, and the deterministic reduction + AdamW finalize.
//
// Replaces mlp_forward (ref: score.py:80-86), _ism_kernel_shared (score.py:128-187),
// _ism_kernel_perparticle (score.py:190-251), _mse_kernel (score.py:254-300),
// ism_loss_and_grad (score.py:303-338), AdamW.step (score.py:371-386) and the per-step body
// of sbtm_update incl. its restore-and-halve recovery (score.py:547-588).
//
// Network: s(u) = W2 softsign(W1 u + b1) + b2, u = [x/L; v], W1 [H][1+dv], W2 [dv][H].
// The GEMMs have K = 1+dv = 4 and N = dv = 3, far below any tensor-core tile, so the math
// runs on the FP32 pipes: one thread per particle for the forward sweep over h, and one
// thread per hidden unit (x particle group) for the backward/outer-product reductions over
// a 256-particle chunk staged in shared memory. Chunk sums are float32 and are promoted to
// float64 per chunk; block partials are float64 and are reduced in a fixed order by a
// single-CTA finalize that also applies the divergence-coefficient terms and AdamW (float64
// master parameters). Deterministic for a given (n, grid).
#include <algorithm>

#include "adamw.cuh"
#include "common.cuh"
#include "f32x2.cuh"

namespace spic {

constexpr int kIsmNT = 256;     // threads per block == particles per chunk
constexpr int kIsmBlocksMax = 4 * kNumSMs;
constexpr int kIsmAcc = 10;     // per (h, group): gW1[4], gb1, gW2[3], Phi, pad

__host__ __device__ inline int64_t n_params(int H, int dv) {
  return (int64_t)H * (1 + dv) + H + (int64_t)dv * H + dv;
}

// params32 -> packed smem records per hidden unit: Wp[h] = (W1[h,0..3]),
// Bp[h] = (b1[h], W2[0,h], W2[1,h], W2[2,h]); pad lanes are zero for dv == 2.
__device__ __forceinline__ void load_packed(const float* __restrict__ p, int H, int dv,
                                            float4* Wp, float4* Bp, float* b2) {
  const float* W1 = p;
  const float* b1 = W1 + H * (1 + dv);
  const float* W2 = b1 + H;
  const float* bb2 = W2 + dv * H;
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    float4 a, b;
    a.x = W1[h * (1 + dv) + 0];
    a.y = W1[h * (1 + dv) + 1];
    a.z = W1[h * (1 + dv) + 2];
    a.w = dv > 2 ? W1[h * (1 + dv) + 3] : 0.f;
    b.x = b1[h];
    b.y = W2[h];
    b.z = W2[H + h];
    b.w = dv > 2 ? W2[2 * H + h] : 0.f;
    Wp[h] = a;
    Bp[h] = b;
  }
  if (threadIdx.x < 3) b2[threadIdx.x] = threadIdx.x < dv ? bb2[threadIdx.x] : 0.f;
}

// ------------------------------------------------------------------------------------------
// forward: s = W2 softsign(W1 [x*x_scale; v] + b1) + b2
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_mlp_forward(
    const float* __restrict__ params, int H, int dv, const float4* __restrict__ xv,
    const float* __restrict__ x, const float* __restrict__ v, int64_t ldv, int64_t n,
    float x_scale, float L, float4* __restrict__ sw, float* __restrict__ s, int64_t lds) {
  extern __shared__ float4 smem4[];
  float4* Wp = smem4;
  float4* Bp = smem4 + H;
  __shared__ float b2[3];
  load_packed(params, H, dv, Wp, Bp, b2);
  __syncthreads();
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    float xn, v0, v1, v2;
    if (xv) {
      float4 A = xv[p];
      xn = A.x < 0.f ? A.x + L : A.x;  // % M quirk records carry x - L
      v0 = A.y; v1 = A.z; v2 = A.w;
    } else {
      xn = x[p];
      v0 = v[p];
      v1 = v[ldv + p];
      v2 = dv > 2 ? v[2 * ldv + p] : 0.f;
    }
    xn *= x_scale;
    float s0 = b2[0], s1 = b2[1], s2 = b2[2];
#pragma unroll 4
    for (int h = 0; h < H; ++h) {
      const float4 a = Wp[h];
      const float4 b = Bp[h];
      float z = fmaf(a.w, v2, fmaf(a.z, v1, fmaf(a.y, v0, fmaf(a.x, xn, b.x))));
      float act = z * fast_rcp(1.f + fabsf(z));
      s0 = fmaf(b.y, act, s0);
      s1 = fmaf(b.z, act, s1);
      s2 = fmaf(b.w, act, s2);
    }
    if (sw) {
      float4 r = sw[p];
      r.x = s0; r.y = s1; r.z = dv > 2 ? s2 : 0.f;
      sw[p] = r;
    } else {
      s[p] = s0;
      s[lds + p] = s1;
      if (dv > 2) s[2 * lds + p] = s2;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Packed-FP32 ISM / MSE partials: two particles per f32x2 lane pair. Same math, same partial
// layout as k_ism_partials; chunks of 2*NT particles, thread t of phase 1 owns particles
// (t, t+NT), phase 2 item (h, g) sweeps the staged particle pairs k = g, g+G, ...
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ f2 bc2(float a) { return mk2(a, a); }

__device__ __forceinline__ f2 rcp2(f2 a) {
  float lo, hi;
  un2(a, lo, hi);
  return mk2(fast_rcp(lo), fast_rcp(hi));
}

template <int MODE>
__device__ __forceinline__ void ism_load_particle(
    int64_t p, int64_t n, const float4* __restrict__ xv, const float4* __restrict__ sw,
    const float* __restrict__ x, const float* __restrict__ v, int64_t ldv,
    const float* __restrict__ w, float x_scale, float L, const float* __restrict__ Z, int64_t ldz,
    const int32_t* __restrict__ idx, int dv, float (&u)[4], float& wp, float (&q)[3]) {
  u[0] = u[1] = u[2] = u[3] = 0.f;
  q[0] = q[1] = q[2] = 0.f;
  wp = 0.f;
  if (p >= n) return;
  const int64_t r = idx ? (int64_t)idx[p] : p;
  if (xv) {
    const float4 A = xv[p];
    u[0] = A.x < 0.f ? A.x + L : A.x;
    u[1] = A.y; u[2] = A.z; u[3] = A.w;
    wp = sw[p].w;
  } else {
    u[0] = x[r];
    u[1] = v[r];
    u[2] = v[ldv + r];
    u[3] = dv > 2 ? v[2 * ldv + r] : 0.f;
    wp = w[r];
  }
  u[0] *= x_scale;
  if (MODE >= 2) {
    q[0] = Z[r];
    q[1] = Z[ldz + r];
    q[2] = dv > 2 ? Z[2 * ldz + r] : 0.f;
  }
}

template <int MODE, int NT>
__global__ void __launch_bounds__(NT) k_ism_partials_x2(
    const float* __restrict__ params, int H, int dv, const float4* __restrict__ xv,
    const float4* __restrict__ sw, const float* __restrict__ x, const float* __restrict__ v,
    int64_t ldv, const float* __restrict__ w, int64_t n, float x_scale, float L,
    const float* __restrict__ Z, int64_t ldz, const int32_t* __restrict__ idx, float inv_wsum,
    double* __restrict__ partials) {
  constexpr int CP = 2 * NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* Wp = (float4*)smem_raw;        // [H]
  float4* Bp = Wp + H;                   // [H]
  float4* U2 = Bp + H;                   // [NT][2]: (x_a, x_b, v0_a, v0_b), (v1_a, v1_b, v2_a, v2_b)
  float4* G2 = U2 + 2 * NT;          // [NT][2]: (g0_a, g0_b, g1_a, g1_b), (g2_a, g2_b, w_a, w_b)
  float4* Z2 = G2 + 2 * NT;          // [NT][2]: probes (MODE 2)
  float* coef = (float*)(Z2 + 2 * NT);
  double* acc64 = (double*)(((uintptr_t)(coef + H) + 15) & ~(uintptr_t)15);  // [items][10]
  __shared__ float b2[3];
  __shared__ double red[8 * 4];

  load_packed(params, H, dv, Wp, Bp, b2);
  __syncthreads();
  if (MODE == 0 || MODE == 1) {
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      const float4 a = Wp[h], b = Bp[h];
      if (MODE == 0) {
        coef[h] = b.y * a.y + b.z * a.z + b.w * a.w;
      } else {
        const float z0 = Z[0], z1 = Z[1], z2 = dv > 2 ? Z[2] : 0.f;
        coef[h] = (b.y * z0 + b.z * z1 + b.w * z2) * (a.y * z0 + a.z * z1 + a.w * z2);
      }
    }
  }
  const int G = max(1, NT / H);
  const int items = H * G;
  for (int it = threadIdx.x; it < items; it += blockDim.x)
    for (int k = 0; k < kIsmAcc; ++k) acc64[it * kIsmAcc + k] = 0.0;
  double lacc[4] = {0.0, 0.0, 0.0, 0.0};
  __syncthreads();
  const f2 one2 = bc2(1.f);

  const int64_t nchunks = (n + CP - 1) / CP;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    // ---- phase 1: particles (t, t+NT) as one packed pair ------------------------------
    float ua[4], ub[4], qa[3], qb[3], wa, wb;
    const int64_t pa = ch * CP + threadIdx.x, pb = pa + NT;
    ism_load_particle<MODE>(pa, n, xv, sw, x, v, ldv, w, x_scale, L, Z, ldz, idx, dv, ua, wa, qa);
    ism_load_particle<MODE>(pb, n, xv, sw, x, v, ldv, w, x_scale, L, Z, ldz, idx, dv, ub, wb, qb);
    if (MODE == 3) {
      wa *= inv_wsum;
      wb *= inv_wsum;
    }
    // stage the inputs first so the scalar copies die before the h loop (keeps the packed
    // pairs resident in register pairs instead of being rebuilt every iteration)
    U2[2 * threadIdx.x] = make_float4(ua[0], ub[0], ua[1], ub[1]);
    U2[2 * threadIdx.x + 1] = make_float4(ua[2], ub[2], ua[3], ub[3]);
    if (MODE == 2) {
      Z2[2 * threadIdx.x] = make_float4(qa[0], qb[0], qa[1], qb[1]);
      Z2[2 * threadIdx.x + 1] = make_float4(qa[2], qb[2], 0.f, 0.f);
    }
    const f2 X = mk2(ua[0], ub[0]), V0 = mk2(ua[1], ub[1]), V1 = mk2(ua[2], ub[2]),
             V2 = mk2(ua[3], ub[3]);
    const f2 Q0 = mk2(qa[0], qb[0]), Q1 = mk2(qa[1], qb[1]), Q2 = mk2(qa[2], qb[2]);
    f2 S0 = bc2(b2[0]), S1 = bc2(b2[1]), S2 = bc2(b2[2]), DIV = bc2(0.f);
#pragma unroll 4
    for (int h = 0; h < H; ++h) {
      const float4 a = Wp[h];
      const float4 b = Bp[h];
      const f2 z = fma2(V2, bc2(a.w), fma2(V1, bc2(a.z), fma2(V0, bc2(a.y), fma2(X, bc2(a.x), bc2(b.x)))));
      const f2 inv = rcp2(add2(abs2(z), one2));
      const f2 act = mul2(z, inv);
      S0 = fma2(act, bc2(b.y), S0);
      S1 = fma2(act, bc2(b.z), S1);
      S2 = fma2(act, bc2(b.w), S2);
      const f2 sp = mul2(inv, inv);
      if (MODE == 0 || MODE == 1) {
        DIV = fma2(sp, bc2(coef[h]), DIV);
      } else if (MODE == 2) {
        const f2 t = fma2(Q2, bc2(a.w), fma2(Q1, bc2(a.z), mul2(Q0, bc2(a.y))));
        const f2 r = fma2(Q2, bc2(b.w), fma2(Q1, bc2(b.z), mul2(Q0, bc2(b.y))));
        DIV = fma2(mul2(r, t), sp, DIV);
      }
    }
    float s[2][3], dvv[2];
    un2(S0, s[0][0], s[1][0]);
    un2(S1, s[0][1], s[1][1]);
    un2(S2, s[0][2], s[1][2]);
    un2(DIV, dvv[0], dvv[1]);
    float g[2][3];
    const float wv[2] = {wa, wb};
    float qq[2][3];
    un2(Q0, qq[0][0], qq[1][0]);
    un2(Q1, qq[0][1], qq[1][1]);
    un2(Q2, qq[0][2], qq[1][2]);
    const bool val[2] = {pa < n, pb < n};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float lp;
      if (MODE == 3) {
        const float e0 = s[e][0] - qq[e][0], e1 = s[e][1] - qq[e][1], e2 = s[e][2] - qq[e][2];
        lp = wv[e] * (e0 * e0 + e1 * e1 + e2 * e2);
        g[e][0] = 2.f * wv[e] * e0; g[e][1] = 2.f * wv[e] * e1; g[e][2] = 2.f * wv[e] * e2;
      } else {
        lp = wv[e] * (s[e][0] * s[e][0] + s[e][1] * s[e][1] + s[e][2] * s[e][2] + 2.f * dvv[e]);
        g[e][0] = 2.f * wv[e] * s[e][0]; g[e][1] = 2.f * wv[e] * s[e][1];
        g[e][2] = 2.f * wv[e] * s[e][2];
      }
      if (dv < 3) g[e][2] = 0.f;
      if (val[e]) {
        lacc[0] += (double)lp;
        lacc[1] += (double)g[e][0];
        lacc[2] += (double)g[e][1];
        lacc[3] += (double)g[e][2];
      } else {
        g[e][0] = g[e][1] = g[e][2] = 0.f;
      }
    }
    G2[2 * threadIdx.x] = make_float4(g[0][0], g[1][0], g[0][1], g[1][1]);
    G2[2 * threadIdx.x + 1] = make_float4(g[0][2], g[1][2], val[0] ? wa : 0.f, val[1] ? wb : 0.f);
    __syncthreads();
    // ---- phase 2: one (hidden unit, pair group) per thread, packed outer products ------
    const int64_t rem = n - ch * CP;
    const int npairs = (int)(rem < (int64_t)NT ? rem : (int64_t)NT);
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int h = it % H, gq = it / H;
      const float4 a = Wp[h], b = Bp[h];
      const float cc4 = (MODE == 0 || MODE == 1) ? 4.f * coef[h] : 0.f;
      f2 gw0 = bc2(0.f), gw1 = gw0, gw2 = gw0, gw3 = gw0, gb = gw0;
      f2 gv0 = gw0, gv1 = gw0, gv2 = gw0, phi = gw0;
#pragma unroll 2
      for (int k = gq; k < npairs; k += G) {
        const float4 A0 = U2[2 * k], A1 = U2[2 * k + 1];
        const float4 B0 = G2[2 * k], B1 = G2[2 * k + 1];
        const f2 X = mk2(A0.x, A0.y), V0 = mk2(A0.z, A0.w), V1 = mk2(A1.x, A1.y), V2 = mk2(A1.z, A1.w);
        const f2 g0 = mk2(B0.x, B0.y), g1 = mk2(B0.z, B0.w), g2 = mk2(B1.x, B1.y), W = mk2(B1.z, B1.w);
        const f2 z = fma2(V2, bc2(a.w), fma2(V1, bc2(a.z), fma2(V0, bc2(a.y), fma2(X, bc2(a.x), bc2(b.x)))));
        const f2 inv = rcp2(add2(abs2(z), one2));
        const f2 act = mul2(z, inv);
        const f2 sp = mul2(inv, inv);
        f2 d = mul2(fma2(g2, bc2(b.w), fma2(g1, bc2(b.z), mul2(g0, bc2(b.y)))), sp);
        if (MODE != 3) {
          // spp = -2 sign(z) sp inv (0 at z == 0); the factor -2 sign(z) is folded into
          // the sign bit (LOP3) and the weight (4 w c_h), keeping the FMA pipe for the math
          float ze, zo, me, mo;
          un2(z, ze, zo);
          un2(mul2(sp, inv), me, mo);
          const f2 spp = mk2(ze == 0.f ? 0.f : copysignf(me, -ze), zo == 0.f ? 0.f : copysignf(mo, -zo));
          f2 cw;  // 4 w c_h per particle
          if (MODE == 2) {
            const float4 Z0 = Z2[2 * k], Z1 = Z2[2 * k + 1];
            const f2 q0 = mk2(Z0.x, Z0.y), q1 = mk2(Z0.z, Z0.w), q2 = mk2(Z1.x, Z1.y);
            const f2 t = fma2(q2, bc2(a.w), fma2(q1, bc2(a.z), mul2(q0, bc2(a.y))));
            const f2 r = fma2(q2, bc2(b.w), fma2(q1, bc2(b.z), mul2(q0, bc2(b.y))));
            const f2 W2x = add2(W, W);
            const f2 k2 = mul2(W2x, sp);
            const f2 k2t = mul2(k2, t), k2r = mul2(k2, r);
            gv0 = fma2(k2t, q0, gv0);
            gv1 = fma2(k2t, q1, gv1);
            gv2 = fma2(k2t, q2, gv2);
            gw1 = fma2(k2r, q0, gw1);
            gw2 = fma2(k2r, q1, gw2);
            gw3 = fma2(k2r, q2, gw3);
            cw = mul2(add2(W2x, W2x), mul2(r, t));
          } else {
            cw = mul2(W, bc2(cc4));
            phi = fma2(W, sp, phi);
          }
          d = fma2(cw, spp, d);
        }
        gb = add2(gb, d);
        gw0 = fma2(d, X, gw0);
        gw1 = fma2(d, V0, gw1);
        gw2 = fma2(d, V1, gw2);
        gw3 = fma2(d, V2, gw3);
        gv0 = fma2(g0, act, gv0);
        gv1 = fma2(g1, act, gv1);
        gv2 = fma2(g2, act, gv2);
      }
      double* A = acc64 + it * kIsmAcc;
      const f2 accs[9] = {gw0, gw1, gw2, gw3, gb, gv0, gv1, gv2, phi};
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        float lo, hi;
        un2(accs[k], lo, hi);
        A[k] += (double)lo + (double)hi;
      }
    }
    __syncthreads();
  }
  block_sum<4>(lacc, red);
  const int64_t P = n_params(H, dv);
  const int64_t width = 1 + P + H;
  double* out = partials + (size_t)blockIdx.x * width;
  if (threadIdx.x == 0) {
    out[0] = lacc[0];
    for (int i = 0; i < dv; ++i) out[1 + P - dv + i] = lacc[1 + i];
  }
  const int64_t oW1 = 1, ob1 = oW1 + (int64_t)H * (1 + dv), oW2 = ob1 + H, oPhi = 1 + P;
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    double sacc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int gq = 0; gq < G; ++gq)
      for (int k = 0; k < 9; ++k) sacc[k] += acc64[(gq * H + h) * kIsmAcc + k];
    for (int k = 0; k < 1 + dv; ++k) out[oW1 + h * (1 + dv) + k] = sacc[k];
    out[ob1 + h] = sacc[4];
    for (int i = 0; i < dv; ++i) out[oW2 + i * H + h] = sacc[5 + i];
    out[oPhi + h] = sacc[8];
  }
}

// ------------------------------------------------------------------------------------------
// finalize: ordered reduction of block partials, divergence terms, AdamW with recovery
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_sbtm_finalize(
    const double* __restrict__ partials, int nblocks, int H, int dv, int div_mode,
    const float* __restrict__ z_shared, double* __restrict__ params, double* __restrict__ m,
    double* __restrict__ v2, double* __restrict__ opt, double beta1, double beta2, double eps,
    double wd, int reset_lr, int apply_step, float* __restrict__ params32,
    double* __restrict__ grads_out, double* __restrict__ loss_out, int32_t* flags) {
  extern __shared__ double g[];  // [1 + P + H], then candidate params [P]
  const int64_t P = n_params(H, dv);
  const int64_t width = 1 + P + H;
  double* cand = g + width;
  for (int64_t k = threadIdx.x; k < width; k += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partials[(size_t)b * width + k];
    g[k] = s;
  }
  __syncthreads();
  double* grad = g + 1;
  const double* Phi = g + 1 + P;
  const int64_t oW1 = 0, ob1 = (int64_t)H * (1 + dv), oW2 = ob1 + H;
  // coefficient-dependence of the divergence term (ref: score.py:317-318, 328-329)
  if (div_mode == 0 || div_mode == 1) {
    for (int64_t k = threadIdx.x; k < (int64_t)dv * H; k += blockDim.x) {
      const int i = (int)(k / H), h = (int)(k % H);
      if (div_mode == 0) {
        grad[oW2 + i * H + h] += 2.0 * Phi[h] * params[oW1 + h * (1 + dv) + 1 + i];
        grad[oW1 + h * (1 + dv) + 1 + i] += 2.0 * Phi[h] * params[oW2 + i * H + h];
      } else {
        double t = 0.0, r = 0.0;
        for (int q = 0; q < dv; ++q) {
          t += params[oW1 + h * (1 + dv) + 1 + q] * (double)z_shared[q];
          r += params[oW2 + q * H + h] * (double)z_shared[q];
        }
        grad[oW2 + i * H + h] += 2.0 * (double)z_shared[i] * t * Phi[h];
        grad[oW1 + h * (1 + dv) + 1 + i] += 2.0 * r * Phi[h] * (double)z_shared[i];
      }
    }
  }
  __syncthreads();
  adamw_with_recovery(g[0], grad, P, div_mode == 3, params, m, v2, opt, beta1, beta2, eps, wd,
                      reset_lr, apply_step, params32, grads_out, loss_out, cand, flags);
}

// Deterministic column sums of the [rows][width] block partials into one row, one warp per
// column (lane-strided rows, fixed shuffle tree), so the single-CTA finalize reads one row.
__global__ void k_ism_reduce_cols(const double* __restrict__ part, int rows, int64_t width,
                                  double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t col = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (col >= width) return;
  double s = 0.0;
  for (int r = lane; r < rows; r += 32) s += part[(size_t)r * width + col];
  s = warp_sum(s);
  if (lane == 0) out[col] = s;
}

// threads per block of the packed ISM kernel: 128 for small n (more blocks to hide latency)
static int ism_nt(int64_t n) { return n < (1 << 18) ? 128 : kIsmNT; }

static int ism_blocks(int64_t n) {
  const int nt = ism_nt(n);
  int64_t chunks = (n + 2 * nt - 1) / (2 * nt);  // packed kernel: 2*NT particles per chunk
  return (int)std::max<int64_t>(1, std::min<int64_t>(chunks, kIsmBlocksMax));
}

static size_t ism_smem(int H, int nt) {
  int G = std::max(1, nt / H);
  size_t b = sizeof(float4) * (2 * (size_t)H + 6 * (size_t)nt) + sizeof(float) * H + 16;
  b += sizeof(double) * (size_t)H * G * kIsmAcc;
  return b;
}

}  // namespace spic

using namespace spic;

extern "C" int64_t spic_mlp_num_params(int32_t H, int32_t dv) { return n_params(H, dv); }

extern "C" int spic_mlp_forward(const float* params32, int32_t H, int32_t dv, const float* xv,
                                const float* x, const float* v, int64_t ldv, int64_t n,
                                float x_scale, float* sw, float* s, int64_t lds, void* stream) {
  if (n < 0 || H < 1 || H > 4096 || (dv != 2 && dv != 3)) return SPIC_ERR_ARG;
  if (n == 0) return SPIC_OK;
  size_t smem = sizeof(float4) * 2 * (size_t)H;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_mlp_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 4);
  k_mlp_forward<<<blocks, 256, smem, (cudaStream_t)stream>>>(
      params32, H, dv, (const float4*)xv, x, v, ldv, n, x_scale, 1.0f / x_scale, (float4*)sw, s, lds); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" size_t spic_ism_scratch_bytes(int64_t n, int32_t H, int32_t dv) {
  // [blocks][width] partials + one reduced row
  return sizeof(double) * (size_t)(ism_blocks(n) + 1) * (size_t)(1 + n_params(H, dv) + H) + 64;
}

// mode: 0 exact, 1 shared Hutchinson (Z = z_shared float[dv] on device), 2 per-particle
// probes Z[dv][ldz], 3 MSE to target Z[dv][ldz]. idx (nullable) maps kernel particle p to the
// source row of the plane inputs and of Z. Block count is encoded in the scratch header.
extern "C" int spic_ism_partials_ex(const float* params32, int32_t H, int32_t dv, int32_t mode,
                                    const float* xv, const float* sw, const float* x,
                                    const float* v, int64_t ldv, const float* w, int64_t n,
                                    float x_scale, const float* Z, int64_t ldz,
                                    const int32_t* idx, double inv_wsum, void* scratch,
                                    size_t scratch_bytes, void* stream) {
  if (n < 1 || H < 1 || H > 2048 || (dv != 2 && dv != 3) || mode < 0 || mode > 3)
    return SPIC_ERR_ARG;
  if (mode >= 1 && !Z) return SPIC_ERR_ARG;
  if (scratch_bytes < spic_ism_scratch_bytes(n, H, dv)) return SPIC_ERR_SCRATCH;
  const int blocks = ism_blocks(n);
  const int nt = ism_nt(n);
  size_t smem = ism_smem(H, nt);
  cudaStream_t st = (cudaStream_t)stream;
  const float L = 1.0f / x_scale;
#define SPIC_ISM_LAUNCH_NT(MD, NT_)                                                           \
  do {                                                                                         \
    if (smem > 48 * 1024)                                                                      \
      cudaFuncSetAttribute(k_ism_partials_x2<MD, NT_>,                                         \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
    k_ism_partials_x2<MD, NT_><<<blocks, NT_, smem, st>>>(                                     \
        params32, H, dv, (const float4*)xv, (const float4*)sw, x, v, ldv, w, n, x_scale, L, Z, \
        ldz, idx, (float)inv_wsum, (double*)scratch);                                          \
    spic::count_launch();                                                                      \
  } while (0)
#define SPIC_ISM_LAUNCH(MD)                                                                    \
  do {                                                                                         \
    if (nt == 128) SPIC_ISM_LAUNCH_NT(MD, 128); else SPIC_ISM_LAUNCH_NT(MD, kIsmNT);           \
  } while (0)
  switch (mode) {
    case 0: SPIC_ISM_LAUNCH(0); break;
    case 1: SPIC_ISM_LAUNCH(1); break;
    case 2: SPIC_ISM_LAUNCH(2); break;
    default: SPIC_ISM_LAUNCH(3); break;
  }
#undef SPIC_ISM_LAUNCH
#undef SPIC_ISM_LAUNCH_NT
  SPIC_CHECK_LAUNCH();
  const int64_t width = 1 + n_params(H, dv) + H;
  double* part = (double*)scratch;
  k_ism_reduce_cols<<<(unsigned)((width + 7) / 8), 256, 0, st>>>(
      part, blocks, width, part + (size_t)blocks * width); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

extern "C" int spic_sbtm_finalize_ex(const void* scratch, int64_t n, int32_t H, int32_t dv,
                                     int32_t div_mode, const float* z_shared, double* params64,
                                     double* m, double* v2, double* opt_state, double beta1,
                                     double beta2, double eps, double weight_decay,
                                     int32_t reset_lr, int32_t apply_step, float* params32,
                                     double* grads_out, double* loss_out, int32_t* flags,
                                     void* stream) {
  if (n < 1 || H < 1 || (dv != 2 && dv != 3) || div_mode < 0 || div_mode > 3) return SPIC_ERR_ARG;
  const int64_t P = n_params(H, dv);
  size_t smem = sizeof(double) * (size_t)(1 + P + H + P);
  if (smem > 200 * 1024) return SPIC_ERR_UNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_sbtm_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_sbtm_finalize<<<1, 1024, smem, (cudaStream_t)stream>>>(
      (const double*)scratch + (size_t)ism_blocks(n) * (size_t)(1 + n_params(H, dv) + H), 1, H, dv,
      div_mode, z_shared, params64, m, v2, opt_state,
      beta1, beta2, eps, weight_decay, reset_lr, apply_step, params32, grads_out, loss_out, flags); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

namespace spic {
// Plain AdamW step on a flat float64 parameter vector (ref: score.py:371-386), used by the
// operator-level AdamW.step; the training loop uses k_sbtm_finalize instead.
__global__ void __launch_bounds__(1024) k_adamw_step(double* __restrict__ params,
                                                     const double* __restrict__ grads,
                                                     double* __restrict__ m, double* __restrict__ v2,
                                                     int64_t P, double* __restrict__ opt,
                                                     double beta1, double beta2, double eps,
                                                     double wd, float* __restrict__ params32) {
  const double t = opt[0] + 1.0, lr = opt[2];
  const double bc1 = 1.0 - pow(beta1, t), bc2 = 1.0 - pow(beta2, t);
  for (int64_t k = threadIdx.x; k < P; k += blockDim.x) {
    double p = params[k];
    if (wd != 0.0) p -= lr * wd * p;
    const double g = grads[k];
    const double mk = beta1 * m[k] + (1.0 - beta1) * g;
    const double vk = beta2 * v2[k] + (1.0 - beta2) * g * g;
    m[k] = mk;
    v2[k] = vk;
    p -= lr * (mk / bc1) / (sqrt(vk / bc2) + eps);
    params[k] = p;
    if (params32) params32[k] = (float)p;
  }
  __syncthreads();
  if (threadIdx.x == 0) opt[0] = t;
}
}  // namespace spic

extern "C" int spic_adamw_step(double* params64, const double* grads64, double* m, double* v2,
                               int64_t P, double* opt_state, double beta1, double beta2,
                               double eps, double weight_decay, float* params32, void* stream) {
  if (P < 0) return SPIC_ERR_ARG;
  k_adamw_step<<<1, 1024, 0, (cudaStream_t)stream>>>(params64, grads64, m, v2, P, opt_state, beta1,
                                                     beta2, eps, weight_decay, params32); spic::count_launch();
  SPIC_CHECK_LAUNCH();
  return SPIC_OK;
}

// Byte offset (in the ISM scratch) of the reduced [loss, grads, Phi] row that
// spic_sbtm_finalize_ex reads: a domain-decomposed run allreduces this row in place.
extern "C" int64_t spic_ism_row_offset(int64_t n, int32_t H, int32_t dv) {
  return (int64_t)sizeof(double) * ism_blocks(n) * (1 + n_params(H, dv) + H);
}
