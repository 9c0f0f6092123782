/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (never linked into the product path).
 *
 * Float64 CPU restatement of the scorepic per-timestep hot path
 * (reference: /root/reference/pkg/src/scorepic, "ref:" below). Each function
 * restates the published algorithm of the cited reference function in plain C;
 * no reference source is copied. It is used (a) by tests/ as the parity
 * checker of the CUDA path, (b) by bench.py as the CPU baseline / reference
 * arm ("port"), parallelised over cells / particle chunks with OpenMP when
 * compiled with -fopenmp (arithmetic per pair is unchanged; chunked reductions
 * are summed in a fixed order so results do not depend on the thread count).
 *
 * Pinned against golden vectors produced by the reference itself:
 * tests/golden/make_golden.py -> tests/golden/ fixtures, checked in
 * tests/test_oracle_golden.py.
 *
 * Layouts follow the reference: x[n], v[n*dv] row-major (particle-major),
 * w[n], scores[n*dv] row-major, all float64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define EPS_Z2 1e-24 /* ref: kernels.py:7 EPS_Z = 1e-12, squared in collision.py:100 */

/* ---------------------------------------------------------------------------------------
 * Grid.cell_of (ref: pic.py:27-30): min(floor(x/eta) mod M, M-1), Python floor-mod.
 * ------------------------------------------------------------------------------------- */
static inline int64_t cell_of(double x, double eta, int64_t M) {
  int64_t idx = (int64_t)floor(x / eta);
  int64_t r = idx % M;
  if (r < 0) r += M;
  return r < M - 1 ? r : M - 1;
}

void oracle_cell_of(const double* x, int64_t n, double eta, int64_t M, int64_t* cell) {
  for (int64_t i = 0; i < n; ++i) cell[i] = cell_of(x[i], eta, M);
}

/* build_cell_index (ref: collision.py:39-46): stable argsort by cell id, plus the
 * bin boundaries. A counting sort is stable by construction. starts has M+1 entries. */
void oracle_build_cell_index(const double* x, int64_t n, double eta, int64_t M,
                             int64_t* perm, int64_t* starts) {
  int64_t* cell = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* cursor = (int64_t*)calloc((size_t)M + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    cell[i] = cell_of(x[i], eta, M);
    cursor[cell[i] + 1]++;
  }
  for (int64_t c = 0; c < M; ++c) cursor[c + 1] += cursor[c];
  memcpy(starts, cursor, sizeof(int64_t) * (size_t)(M + 1));
  for (int64_t i = 0; i < n; ++i) perm[cursor[cell[i]]++] = i;
  free(cursor);
  free(cell);
}

/* Periodic stencil {c-1, c, c+1} deduplicated for tiny M (ref: collision.py:29-36). */
static int stencil_cells(int64_t c, int64_t M, int64_t out[3]) {
  int k = 0;
  for (int d = -1; d <= 1; ++d) {
    int64_t cd = ((c + d) % M + M) % M;
    int dup = 0;
    for (int q = 0; q < k; ++q) dup |= (out[q] == cd);
    if (!dup) out[k++] = cd;
  }
  return k;
}

/* ---------------------------------------------------------------------------------------
 * Landau collision force (ref: collision.py:49-110). For every target i in cell c and
 * every neighbour j of the stencil: min-image dx, skip |dx| >= eta, psi = (1-|dx|/eta)/eta,
 * z = v_i - v_j, u = s_i - s_j, skip |z|^2 <= 1e-24, coef = |z|^(gamma+2),
 * U_i += w_j psi coef (u - (z.u/|z|^2) z).
 * ------------------------------------------------------------------------------------- */
static void collision_targets(const double* xt, const double* vt, const double* st, int64_t nt,
                              const double* xn, const double* vn, const double* sn,
                              const double* wn, int64_t nn, int dv, double eta, double L,
                              double half_pow, double* out) {
  /* gathered, contiguous target / neighbour blocks like the reference's per-cell call
   * (ref: collision.py:107-108); out is (nt, dv) */
  for (int64_t a = 0; a < nt; ++a) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t b = 0; b < nn; ++b) {
      double dx = xt[a] - xn[b];
      if (dx > 0.5 * L)
        dx -= L;
      else if (dx < -0.5 * L)
        dx += L;
      double adx = fabs(dx);
      if (adx >= eta) continue;
      double psi = (1.0 - adx / eta) / eta;
      double z2 = 0.0, zu = 0.0;
      for (int k = 0; k < dv; ++k) {
        double zk = vt[a * dv + k] - vn[b * dv + k];
        double uk = st[a * dv + k] - sn[b * dv + k];
        z2 += zk * zk;
        zu += zk * uk;
      }
      if (z2 <= EPS_Z2) continue;
      double coef;
      if (half_pow == 0.0)
        coef = 1.0;
      else if (half_pow == -0.5)
        coef = 1.0 / sqrt(z2);
      else
        coef = pow(z2, half_pow);
      double cw = wn[b] * psi * coef;
      double proj = cw * zu / z2;
      for (int k = 0; k < dv; ++k)
        acc[k] += cw * (st[a * dv + k] - sn[b * dv + k]) - proj * (vt[a * dv + k] - vn[b * dv + k]);
    }
    for (int k = 0; k < dv; ++k) out[a * dv + k] = acc[k];
  }
}

/* gather rows idx[0..m) of (x, v, s, w) into contiguous blocks */
static void gather_rows(const double* x, const double* v, const double* s, const double* w,
                        int dv, const int64_t* idx, int64_t m, double* gx, double* gv, double* gs,
                        double* gw) {
  for (int64_t a = 0; a < m; ++a) {
    int64_t i = idx[a];
    gx[a] = x[i];
    if (gw) gw[a] = w[i];
    for (int k = 0; k < dv; ++k) {
      gv[a * dv + k] = v[i * dv + k];
      if (gs) gs[a * dv + k] = s[i * dv + k];
    }
  }
}

/* Returns 0, or -1 when a score is non-finite (ref: collision.py:95-96). cell_subset:
 * when stride > 1 only cells c with c % stride == 0 are evaluated (bounded CPU-baseline
 * samples); other rows of U are left untouched. */
int oracle_collision_force_sampled(const double* x, const double* v, const double* w,
                                   const double* s, int64_t n, int dv, int64_t M, double eta,
                                   double gamma, int64_t cell_stride, double* U) {
  for (int64_t i = 0; i < n * dv; ++i)
    if (!isfinite(s[i])) return -1;
  double L = (double)M * eta;
  double half_pow = (gamma + 2.0) / 2.0;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* starts = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M + 1));
  oracle_build_cell_index(x, n, eta, M, perm, starts);
  if (cell_stride < 1) cell_stride = 1;
#pragma omp parallel
  {
    size_t cap = (size_t)(n > 0 ? n : 1);
    int64_t* nbr = (int64_t*)malloc(sizeof(int64_t) * cap);
    double* buf = (double*)malloc(sizeof(double) * cap * (size_t)(3 + 5 * dv));
    double *xn = buf, *wn = xn + cap, *vn = wn + cap, *sn = vn + cap * dv;
    double *xt = sn + cap * dv, *vt = xt + cap, *stt = vt + cap * dv, *out = stt + cap * dv;
#pragma omp for schedule(dynamic, 1)
    for (int64_t c = 0; c < M; ++c) {
      if (c % cell_stride) continue;
      int64_t nt = starts[c + 1] - starts[c];
      if (nt == 0) continue;
      int64_t cells[3];
      int k = stencil_cells(c, M, cells);
      int64_t nn = 0;
      for (int q = 0; q < k; ++q)
        for (int64_t t = starts[cells[q]]; t < starts[cells[q] + 1]; ++t) nbr[nn++] = perm[t];
      const int64_t* tgt = perm + starts[c];
      gather_rows(x, v, s, w, dv, nbr, nn, xn, vn, sn, wn);
      gather_rows(x, v, s, w, dv, tgt, nt, xt, vt, stt, NULL);
      collision_targets(xt, vt, stt, nt, xn, vn, sn, wn, nn, dv, eta, L, half_pow, out);
      for (int64_t a = 0; a < nt; ++a)
        for (int kk = 0; kk < dv; ++kk) U[tgt[a] * dv + kk] = out[a * dv + kk];
    }
    free(buf);
    free(nbr);
  }
  free(perm);
  free(starts);
  return 0;
}

int oracle_collision_force(const double* x, const double* v, const double* w, const double* s,
                           int64_t n, int dv, int64_t M, double eta, double gamma, double* U) {
  memset(U, 0, sizeof(double) * (size_t)(n * dv));
  return oracle_collision_force_sampled(x, v, w, s, n, dv, M, eta, gamma, 1, U);
}

/* Ordered live pairs (|min-image dx| < eta over the stencil), the pair-rate unit. */
int64_t oracle_count_live_pairs(const double* x, int64_t n, int64_t M, double eta) {
  double L = (double)M * eta;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* starts = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M + 1));
  oracle_build_cell_index(x, n, eta, M, perm, starts);
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total)
  for (int64_t c = 0; c < M; ++c) {
    int64_t cells[3];
    int k = stencil_cells(c, M, cells);
    for (int64_t a = starts[c]; a < starts[c + 1]; ++a) {
      double xi = x[perm[a]];
      for (int q = 0; q < k; ++q)
        for (int64_t t = starts[cells[q]]; t < starts[cells[q] + 1]; ++t) {
          double dx = xi - x[perm[t]];
          if (dx > 0.5 * L)
            dx -= L;
          else if (dx < -0.5 * L)
            dx += L;
          total += fabs(dx) < eta;
        }
    }
  }
  free(perm);
  free(starts);
  return total;
}

/* ---------------------------------------------------------------------------------------
 * Blob KDE score (ref: score.py:453-523). Per cell: bandwidth h (fixed, or Silverman over
 * the stencil velocities, ref: score.py:493-500), then for each target
 * den = sum_j w_j psi exp(-|v_i-v_j|^2/(2h^2)), mu = sum_j (same) v_j,
 * s_i = (mu/den - v_i)/h^2. Returns -1 and *bad_index (lowest cell, then first target in
 * bin order) when den <= 0 or the score is non-finite (ref: score.py:518-521).
 * ------------------------------------------------------------------------------------- */
static double silverman(const double* v, int dv, const int64_t* idx, int64_t m) {
  double sigma = 0.0;
  if (m > 1) {
    for (int k = 0; k < dv; ++k) {
      double mean = 0.0;
      for (int64_t a = 0; a < m; ++a) mean += v[idx[a] * dv + k];
      mean /= (double)m;
      double ss = 0.0;
      for (int64_t a = 0; a < m; ++a) {
        double d = v[idx[a] * dv + k] - mean;
        ss += d * d;
      }
      sigma += sqrt(ss / (double)(m - 1));
    }
    sigma /= (double)dv;
  }
  double h = sigma * pow(4.0 / ((double)(dv + 2) * (double)m), 1.0 / (double)(dv + 4));
  return (h > 0.0 && isfinite(h)) ? h : 1.0;
}

double oracle_silverman_bandwidth(const double* v, int64_t m, int dv) {
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  for (int64_t a = 0; a < m; ++a) idx[a] = a;
  double h = silverman(v, dv, idx, m);
  free(idx);
  return h;
}

int oracle_blob_score_sampled(const double* x, const double* v, const double* w, int64_t n,
                              int dv, int64_t M, double eta, double bandwidth,
                              int64_t cell_stride, double* s, double* den_out,
                              int64_t* bad_index) {
  double L = (double)M * eta;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* starts = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M + 1));
  oracle_build_cell_index(x, n, eta, M, perm, starts);
  int64_t* bad_cell_first = (int64_t*)malloc(sizeof(int64_t) * (size_t)M);
  if (cell_stride < 1) cell_stride = 1;
#pragma omp parallel
  {
    int64_t* nbr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(dynamic, 1)
    for (int64_t c = 0; c < M; ++c) {
      bad_cell_first[c] = -1;
      if (c % cell_stride) continue;
      int64_t nt = starts[c + 1] - starts[c];
      if (nt == 0) continue;
      int64_t cells[3];
      int k = stencil_cells(c, M, cells);
      int64_t nn = 0;
      for (int q = 0; q < k; ++q)
        for (int64_t t = starts[cells[q]]; t < starts[cells[q] + 1]; ++t) nbr[nn++] = perm[t];
      double h = bandwidth > 0.0 ? bandwidth : silverman(v, dv, nbr, nn);
      double inv2h2 = 0.5 / (h * h);
      for (int64_t a = 0; a < nt; ++a) {
        int64_t i = perm[starts[c] + a];
        double den = 0.0, mu[3] = {0.0, 0.0, 0.0};
        for (int64_t b = 0; b < nn; ++b) {
          int64_t j = nbr[b];
          double dx = x[i] - x[j];
          if (dx > 0.5 * L)
            dx -= L;
          else if (dx < -0.5 * L)
            dx += L;
          double adx = fabs(dx);
          if (adx >= eta) continue;
          double psi = (1.0 - adx / eta) / eta;
          double q2 = 0.0;
          for (int kk = 0; kk < dv; ++kk) {
            double d = v[i * dv + kk] - v[j * dv + kk];
            q2 += d * d;
          }
          double kw = w[j] * psi * exp(-q2 * inv2h2);
          den += kw;
          for (int kk = 0; kk < dv; ++kk) mu[kk] += kw * v[j * dv + kk];
        }
        if (den_out) den_out[i] = den;
        int bad = !(den > 0.0);
        for (int kk = 0; kk < dv; ++kk) {
          double val = den > 0.0 ? (mu[kk] / den - v[i * dv + kk]) / (h * h) : 0.0;
          s[i * dv + kk] = val;
          if (!isfinite(val)) bad = 1;
        }
        if (bad && bad_cell_first[c] < 0) bad_cell_first[c] = i;
      }
    }
    free(nbr);
  }
  int rc = 0;
  for (int64_t c = 0; c < M; ++c)
    if (bad_cell_first[c] >= 0) {
      if (bad_index) *bad_index = bad_cell_first[c];
      rc = -1;
      break;
    }
  free(bad_cell_first);
  free(perm);
  free(starts);
  return rc;
}

int oracle_blob_score(const double* x, const double* v, const double* w, int64_t n, int dv,
                      int64_t M, double eta, double bandwidth, double* s, double* den_out,
                      int64_t* bad_index) {
  memset(s, 0, sizeof(double) * (size_t)(n * dv));
  return oracle_blob_score_sampled(x, v, w, n, dv, M, eta, bandwidth, 1, s, den_out, bad_index);
}

/* ---------------------------------------------------------------------------------------
 * Score MLP s(u) = W2 softsign(W1 u + b1) + b2, u = [x; v] (ref: score.py:38-86).
 * W1 is H x (1+dv) row-major, W2 is dv x H row-major.
 * ------------------------------------------------------------------------------------- */
void oracle_mlp_forward(const double* X, const double* V, int64_t n, int dv, int64_t H,
                        const double* W1, const double* b1, const double* W2,
                        const double* b2, double* S) {
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < n; ++p) {
    double s[3];
    for (int i = 0; i < dv; ++i) s[i] = b2[i];
    for (int64_t h = 0; h < H; ++h) {
      double z = b1[h] + W1[h * (1 + dv)] * X[p];
      for (int k = 0; k < dv; ++k) z += W1[h * (1 + dv) + 1 + k] * V[p * dv + k];
      double a = z / (1.0 + fabs(z));
      for (int i = 0; i < dv; ++i) s[i] += W2[i * H + h] * a;
    }
    for (int i = 0; i < dv; ++i) S[p * dv + i] = s[i];
  }
}

/* ISM loss + gradients (ref: score.py:128-251, driver score.py:303-338).
 * mode 0: shared coefficient vector coef[H] (exact: coef_h = sum_i W2[i,h] W1[h,1+i];
 *         shared Hutchinson: coef = r*t); Phi[H] = sum_p w_p sigma'(z_ph) is returned.
 * mode 1: per-particle Rademacher probes Zr[n*dv] (Phi unused).
 * grads layout (one flat buffer): gW1[H*(1+dv)], gb1[H], gW2[dv*H], gb2[dv].
 * Chunks of CH particles are reduced into per-chunk partials and then summed in chunk
 * order, so the result is independent of the OpenMP thread count. */
#define ISM_CHUNK 4096
static void ism_chunk(const double* X, const double* V, const double* w, int64_t p0,
                      int64_t p1, int dv, int64_t H, const double* W1, const double* b1,
                      const double* W2, const double* b2, const double* coef,
                      const double* Zr, double* out /* 1 + P + H */) {
  int64_t d_in = 1 + dv;
  int64_t P = H * d_in + H + dv * H + dv;
  double* gW1 = out + 1;
  double* gb1 = gW1 + H * d_in;
  double* gW2 = gb1 + H;
  double* gb2 = gW2 + dv * H;
  double* Phi = out + 1 + P;
  double* z = (double*)malloc(sizeof(double) * (size_t)H * 5);
  double* a = z + H;
  double* sp = a + H;
  double* t = sp + H;
  double* r = t + H;
  for (int64_t p = p0; p < p1; ++p) {
    double xp = X[p], wp = w[p];
    for (int64_t h = 0; h < H; ++h) {
      double acc = b1[h] + W1[h * d_in] * xp;
      double th = 0.0, rh = 0.0;
      for (int k = 0; k < dv; ++k) {
        acc += W1[h * d_in + 1 + k] * V[p * dv + k];
        if (Zr) {
          th += W1[h * d_in + 1 + k] * Zr[p * dv + k];
          rh += W2[k * H + h] * Zr[p * dv + k];
        }
      }
      z[h] = acc;
      double inv = 1.0 / (1.0 + fabs(acc));
      a[h] = acc * inv;
      sp[h] = inv * inv;
      t[h] = th;
      r[h] = rh;
    }
    double s2 = 0.0, gs[3];
    for (int i = 0; i < dv; ++i) {
      double acc = b2[i];
      for (int64_t h = 0; h < H; ++h) acc += W2[i * H + h] * a[h];
      s2 += acc * acc;
      gs[i] = 2.0 * wp * acc;
    }
    double div = 0.0;
    for (int64_t h = 0; h < H; ++h) div += (Zr ? r[h] * t[h] : coef[h]) * sp[h];
    out[0] += wp * (s2 + 2.0 * div);
    for (int i = 0; i < dv; ++i) gb2[i] += gs[i];
    for (int64_t h = 0; h < H; ++h) {
      double da = 0.0;
      for (int i = 0; i < dv; ++i) {
        da += gs[i] * W2[i * H + h];
        gW2[i * H + h] += gs[i] * a[h];
        if (Zr) gW2[i * H + h] += 2.0 * wp * sp[h] * t[h] * Zr[p * dv + i];
      }
      double inv = 1.0 / (1.0 + fabs(z[h]));
      double sgn = (z[h] > 0.0) - (z[h] < 0.0);
      double spp = -2.0 * sgn * inv * inv * inv;
      double ch = Zr ? r[h] * t[h] : coef[h];
      double d = da * sp[h] + 2.0 * wp * ch * spp;
      if (!Zr) Phi[h] += wp * sp[h];
      gb1[h] += d;
      gW1[h * d_in] += d * xp;
      for (int k = 0; k < dv; ++k) {
        gW1[h * d_in + 1 + k] += d * V[p * dv + k];
        if (Zr) gW1[h * d_in + 1 + k] += 2.0 * wp * sp[h] * r[h] * Zr[p * dv + k];
      }
    }
  }
  free(z);
}

double oracle_ism_kernel(const double* X, const double* V, const double* w, int64_t n, int dv,
                         int64_t H, const double* W1, const double* b1, const double* W2,
                         const double* b2, const double* coef, const double* Zr,
                         double* grads, double* Phi) {
  int64_t d_in = 1 + dv;
  int64_t P = H * d_in + H + dv * H + dv;
  int64_t width = 1 + P + H;
  int64_t nchunks = (n + ISM_CHUNK - 1) / ISM_CHUNK;
  double* part = (double*)calloc((size_t)(nchunks > 0 ? nchunks : 1) * (size_t)width, sizeof(double));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < nchunks; ++c) {
    int64_t p0 = c * ISM_CHUNK, p1 = p0 + ISM_CHUNK < n ? p0 + ISM_CHUNK : n;
    ism_chunk(X, V, w, p0, p1, dv, H, W1, b1, W2, b2, coef, Zr, part + c * width);
  }
  double loss = 0.0;
  memset(grads, 0, sizeof(double) * (size_t)P);
  if (Phi) memset(Phi, 0, sizeof(double) * (size_t)H);
  for (int64_t c = 0; c < nchunks; ++c) {
    const double* q = part + c * width;
    loss += q[0];
    for (int64_t k = 0; k < P; ++k) grads[k] += q[1 + k];
    if (Phi)
      for (int64_t h = 0; h < H; ++h) Phi[h] += q[1 + P + h];
  }
  free(part);
  return loss;
}

/* Weighted score MSE to a target and its gradients (pretraining, ref: score.py:254-300). */
double oracle_mse_kernel(const double* X, const double* V, const double* w, int64_t n, int dv,
                         int64_t H, const double* W1, const double* b1, const double* W2,
                         const double* b2, const double* target, double inv_wsum,
                         double* grads) {
  int64_t d_in = 1 + dv;
  int64_t P = H * d_in + H + dv * H + dv;
  double* gW1 = grads;
  double* gb1 = gW1 + H * d_in;
  double* gW2 = gb1 + H;
  double* gb2 = gW2 + dv * H;
  memset(grads, 0, sizeof(double) * (size_t)P);
  double* z = (double*)malloc(sizeof(double) * (size_t)H * 3);
  double* a = z + H;
  double* sp = a + H;
  double loss = 0.0;
  for (int64_t p = 0; p < n; ++p) {
    double xp = X[p], wp = w[p] * inv_wsum;
    for (int64_t h = 0; h < H; ++h) {
      double acc = b1[h] + W1[h * d_in] * xp;
      for (int k = 0; k < dv; ++k) acc += W1[h * d_in + 1 + k] * V[p * dv + k];
      z[h] = acc;
      double inv = 1.0 / (1.0 + fabs(acc));
      a[h] = acc * inv;
      sp[h] = inv * inv;
    }
    double err2 = 0.0, gs[3];
    for (int i = 0; i < dv; ++i) {
      double acc = b2[i];
      for (int64_t h = 0; h < H; ++h) acc += W2[i * H + h] * a[h];
      double e = acc - target[p * dv + i];
      err2 += e * e;
      gs[i] = 2.0 * wp * e;
    }
    loss += wp * err2;
    for (int i = 0; i < dv; ++i) gb2[i] += gs[i];
    for (int64_t h = 0; h < H; ++h) {
      double da = 0.0;
      for (int i = 0; i < dv; ++i) {
        da += gs[i] * W2[i * H + h];
        gW2[i * H + h] += gs[i] * a[h];
      }
      double d = da * sp[h];
      gb1[h] += d;
      gW1[h * d_in] += d * xp;
      for (int k = 0; k < dv; ++k) gW1[h * d_in + 1 + k] += d * V[p * dv + k];
    }
  }
  free(z);
  return loss;
}

/* ---------------------------------------------------------------------------------------
 * PIC: hat weights (ref: pic.py:33-40), deposit (pic.py:43-58), interpolate + Lorentz +
 * advance + wrap (pic.py:61-93, state.py:14-27), field steps (pic.py:96-115).
 * ------------------------------------------------------------------------------------- */
static inline void hat(double x, double eta, int64_t M, int64_t* i0, int64_t* i1, double* f0,
                       double* f1) {
  double g = x / eta - 0.5;
  double fl = floor(g);
  double f = g - fl;
  int64_t k = (int64_t)fl % M;
  if (k < 0) k += M;
  *i0 = k;
  *i1 = (k + 1) % M;
  *f0 = 1.0 - f;
  *f1 = f;
}

/* rho[M], J[dv*M] (J row-major (dv, M)). Sums in particle order, like bincount. */
void oracle_deposit(const double* x, const double* v, const double* w, int64_t n, int dv,
                    int64_t M, double eta, double* rho, double* J) {
  /* ref sums the i0 and i1 bincounts separately and adds them (pic.py:52-57) */
  double* r0 = (double*)calloc((size_t)M * 2 * (1 + dv), sizeof(double));
  double* r1 = r0 + M * (1 + dv);
  for (int64_t p = 0; p < n; ++p) {
    int64_t i0, i1;
    double f0, f1;
    hat(x[p], eta, M, &i0, &i1, &f0, &f1);
    double w0 = w[p] * f0, w1 = w[p] * f1;
    r0[i0] += w0;
    r1[i1] += w1;
    for (int k = 0; k < dv; ++k) {
      r0[(1 + k) * M + i0] += w0 * v[p * dv + k];
      r1[(1 + k) * M + i1] += w1 * v[p * dv + k];
    }
  }
  for (int64_t j = 0; j < M; ++j) {
    rho[j] = (r0[j] + r1[j]) / eta;
    for (int k = 0; k < dv; ++k) J[k * M + j] = (r0[(1 + k) * M + j] + r1[(1 + k) * M + j]) / eta;
  }
  free(r0);
}

/* Returns -1 on a non-finite position (ref: state.py:23-24). */
int oracle_push(double* x, double* v, int64_t n, int dv, const double* E1, const double* E2,
                const double* B3, int64_t M, double eta, double dt) {
  double L = (double)M * eta;
  int bad = 0;
  for (int64_t p = 0; p < n; ++p) {
    int64_t i0, i1;
    double f0, f1;
    hat(x[p], eta, M, &i0, &i1, &f0, &f1);
    double e1 = f0 * E1[i0] + f1 * E1[i1];
    double e2 = f0 * E2[i0] + f1 * E2[i1];
    double b3 = f0 * B3[i0] + f1 * B3[i1];
    double v1 = v[p * dv], v2 = v[p * dv + 1];
    /* ref: pic.py:77-88, dvx = E_p + (v2 B3, -v1 B3, 0); v += dt * dvx */
    double a1 = e1 + v2 * b3;
    double a2 = e2 - v1 * b3;
    v[p * dv] = v1 + dt * a1;
    v[p * dv + 1] = v2 + dt * a2;
    if (dv == 3) v[p * dv + 2] = v[p * dv + 2] + dt * 0.0;
    double xn = x[p] + dt * v[p * dv];
    if (!isfinite(xn)) {
      bad = 1;
      continue;
    }
    double m = fmod(xn, L);
    if (m < 0) m += L; /* numpy mod: result carries the sign of L */
    if (m >= L) m = 0.0;
    x[p] = m;
  }
  return bad ? -1 : 0;
}

void oracle_maxwell_step(double* E1, double* E2, double* B3, const double* J, int64_t M,
                         double eta, double dt) {
  double two_eta = 2.0 * eta;
  double* tmp = (double*)malloc(sizeof(double) * (size_t)M);
  for (int64_t j = 0; j < M; ++j) E1[j] -= dt * J[j];
  for (int64_t j = 0; j < M; ++j)
    tmp[j] = (B3[(j + 1) % M] - B3[(j - 1 + M) % M]) / two_eta;
  for (int64_t j = 0; j < M; ++j) E2[j] -= dt * (tmp[j] + J[M + j]);
  for (int64_t j = 0; j < M; ++j)
    tmp[j] = (E2[(j + 1) % M] - E2[(j - 1 + M) % M]) / two_eta;
  for (int64_t j = 0; j < M; ++j) B3[j] -= dt * tmp[j];
  free(tmp);
}

void oracle_vpl_field_step(double* E1, const double* J, int64_t M, double dt) {
  for (int64_t j = 0; j < M; ++j) E1[j] -= dt * J[j];
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}
