/*
 * scorepic_b200.h — C ABI of the B200-native (sm_100a) scorepic hot path.
 *
 * Every pointer is a DEVICE pointer unless stated otherwise; every op takes the caller's
 * cudaStream_t as `void* stream`, never allocates (scratch is passed in, sized by the
 * matching *_scratch_bytes query), never synchronizes, and returns 0 or a negative
 * SPIC_ERR_* status. Data-dependent error conditions (non-finite state, isolated blob
 * particles, training divergence) are reported through a device int32 flag array
 * `flags[SPIC_NFLAGS]` that the host reads once per step.
 *
 * Particle layout on device ("pid order" = the reference's particle index order):
 *   x  float[n]                       positions
 *   v  float[dv][ldv]                 velocity planes (SoA), plane k at v + k*ldv
 *   w  float[n]                       weights
 * Cell-sorted working copies ("sorted order", produced by spic_bin):
 *   xv float4[n] = (x', v0, v1, v2)   x' = x, or x - L for the % M quirk particle
 *   sw float4[n] = (s0, s1, s2, w)    scores written by the estimator, weight by spic_bin
 *   perm int32[n]                     sorted position -> pid
 * For dv == 2 the unused lanes are zero.
 *
 * Each entry point names the reference function(s) it replaces
 * (/root/reference/pkg/src/scorepic/<file>:<line>).
 */
#ifndef SCOREPIC_B200_H
#define SCOREPIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SPIC_OK = 0,
  SPIC_ERR_ARG = -1,          /* invalid argument (size, dv, M, H out of range) */
  SPIC_ERR_SCRATCH = -2,      /* scratch buffer too small */
  SPIC_ERR_UNSUPPORTED = -3,  /* valid in the reference, not supported by this build */
  SPIC_ERR_CUDA = -1000       /* -1000 - cudaError_t */
};

/* device flag indices (int32 each; nonzero = condition seen) */
enum {
  SPIC_FLAG_NONFINITE_X = 0,   /* ValueError("non-finite position"), state.py:23-24 */
  SPIC_FLAG_NONFINITE_V = 1,   /* ValueError("non-finite particle state"), state.py:47-49 */
  SPIC_FLAG_BAD_SCORE = 2,     /* ValueError("invalid score input"), collision.py:95-96 */
  SPIC_FLAG_ISOLATED = 3,      /* ValueError("isolated particle ..."), score.py:518-521 */
  SPIC_FLAG_TRAIN_FATAL = 4,   /* RuntimeError("training divergence"), score.py:584-585 */
  SPIC_FLAG_LR_HALVINGS = 5,   /* count of restore-and-halve events, score.py:579-583 */
  SPIC_FLAG_NON_NEUTRAL = 6,   /* ValueError("non-neutral plasma"), pic.py:126-127 */
  SPIC_FLAG_NONFINITE_FIELD = 7, /* ValueError("non-finite field state"), state.py:75-78 */
  SPIC_NFLAGS = 8
};

/* ---- version / build ------------------------------------------------------------------ */
int spic_version(void);
/* number of SMs the launch heuristics assume (148 on B200) */
int spic_num_sms(void);
/* total kernel launches issued by this library so far (host counter) */
long long spic_launch_count(void);
/* FP32 FMA throughput probe (roofline denominator): *flop (host) = FLOPs of the launch. */
int spic_fp32_probe(int32_t iters, int32_t blocks, float* out, double* flop, void* stream);

/* ---- binning (replaces Grid.cell_of pic.py:27-30, build_cell_index collision.py:39-46) -- */
/* cell[i] = min(floor(x_i/eta) mod M, M-1), float64 arithmetic on the float32 input. */
int spic_cell_of(const float* x, int64_t n, double eta, int32_t M, int32_t* cell, void* stream);

size_t spic_bin_scratch_bytes(int64_t n, int32_t M, int32_t S);
/* Stable sort by key = (cell, sub) where sub = floor(frac(x/eta)*S): a single-pass counting
 * sort below 2^21 records, an LSD radix sort (two <= 8-bit digit passes) above; both give the
 * same permutation.
 * S == 1 gives exactly np.argsort(cell_of(x), kind="stable") (the reference CellIndex).
 * Outputs: perm[n] (sorted position -> pid), cell_start[M+1], sub_start[M*S+1] (nullable).
 * Optional fused gather (all nullable): xv[n], sw[n] (w lane only) in sorted order. */
int spic_bin(const float* x, const float* v, int64_t ldv, const float* w, int64_t n, int32_t dv,
             double eta, int32_t M, int32_t S, int32_t* perm, int32_t* cell_start,
             int32_t* sub_start, float* xv, float* sw, void* scratch, size_t scratch_bytes,
             void* stream);
/* Gather pid-order scores s[dv][lds] into the sorted records sw (lanes 0..dv-1). */
int spic_gather_scores(const float* s, int64_t lds, const int32_t* perm, int64_t n, int32_t dv,
                       float* sw, int32_t* flags, void* stream);

/* ---- Landau collision (replaces _collision_cell collision.py:49-89, collision_force
 *      collision.py:92-110, collision_push collision.py:113-116) --------------------------- */
size_t spic_landau_scratch_bytes(int64_t n, int32_t M, int32_t dv, int32_t nsplit);
/* Targets per tile of the antisymmetric pair kernel for an M-cell grid (threads x targets per
 * thread of the configuration in use). A tile owns the pairs with its forward window, so the
 * number of pairs one launch evaluates depends on it (bench.py's evaluated-pair count; no
 * reference counterpart: _collision_cell, collision.py:49-89, loops over whole cells). */
int spic_landau_tile_targets(int32_t M);
/* U (sorted order, float[dv][n]) for all targets against their 3-cell stencil.
 * gamma must be -3 (dv=3) or -2 (dv=2) or any value (generic pow path).
 * uniform_w > 0: all weights equal uniform_w (sw.w ignored). nsplit: j-window split
 * factor (0 = automatic).
 * dv = 3, gamma = -3, uniform_w > 0 run the antisymmetric unordered-pair kernel (each pair
 * evaluated once for both targets; deterministic slot fold); its slot storage is part of
 * the scratch (sized for a near-uniform ensemble, <= 16 GiB); an ensemble needing more
 * runs the ordered enumeration inside the same launches. Results identical to 1e-6 rel. */
int spic_landau(const float* xv, const float* sw, int64_t n, int32_t dv, const int32_t* cell_start,
                const int32_t* sub_start, int32_t M, int32_t S, double eta, double gamma,
                float uniform_w, int32_t nsplit, float* U_sorted, void* scratch,
                size_t scratch_bytes, void* stream);
/* Same, with targets restricted to the cells [c_lo, c_hi) (a domain rank's owned cells;
 * halo cells only act as neighbours). U_sorted entries of other cells are not written.
 * Scratch: spic_landau_range_scratch_bytes (per-cell sizes estimated over the range). */
size_t spic_landau_range_scratch_bytes(int64_t n, int32_t M, int32_t dv, int32_t nsplit,
                                       int32_t c_lo, int32_t c_hi);
int spic_landau_range(const float* xv, const float* sw, int64_t n, int32_t dv,
                      const int32_t* cell_start, const int32_t* sub_start, int32_t M, int32_t S,
                      double eta, double gamma, float uniform_w, int32_t nsplit, int32_t c_lo,
                      int32_t c_hi, float* U_sorted, void* scratch, size_t scratch_bytes,
                      void* stream);
/* Sum nsplit partial U planes [nsplit][dv][n] into U_sorted in a fixed order. */
int spic_landau_fold(const float* U_part, int32_t nsplit, int32_t dv, int64_t n, float* U_sorted,
                     void* stream);
/* Epilogue: U_pid[:, perm[k]] = U_sorted[:, k] (nullable), v[:, perm[k]] -= nu_dt*U (if
 * nu_dt != 0), and diagnostics partial sums; red_out (float64, nullable) receives
 * [H_dot = sum w s.U, E_K = 1/2 sum w |v|^2 (post-push), P_0..P_{dv-1}]. */
int spic_collision_epilogue(const float* U_sorted, const float* sw, const int32_t* perm,
                            int64_t n, int32_t dv, float nu_dt, float* v, int64_t ldv,
                            float* U_pid, int64_t ldu, double* red_out, int32_t* flags,
                            void* scratch, size_t scratch_bytes, void* stream);
/* Same over the sorted positions [k0, k1) only (a domain rank's owned targets). */
int spic_collision_epilogue_range(const float* U_sorted, const float* sw, const int32_t* perm,
                                  int64_t n, int32_t dv, int64_t k0, int64_t k1, float nu_dt,
                                  float* v, int64_t ldv, float* U_pid, int64_t ldu,
                                  double* red_out, int32_t* flags, void* scratch,
                                  size_t scratch_bytes, void* stream);
/* number of ordered live pairs |min-image dx| < eta over the stencil (the pair-rate unit) */
int spic_count_live_pairs(const float* xv, int64_t n, const int32_t* cell_start, int32_t M,
                          double eta, unsigned long long* count, void* stream);

/* ---- blob KDE score (replaces _blob_cell score.py:453-490, silverman_bandwidth
 *      score.py:493-500, blob_score score.py:503-523) -------------------------------------- */
size_t spic_blob_scratch_bytes(int64_t n, int32_t M, int32_t dv);
/* Writes s into sw lanes 0..dv-1 (sorted order). bandwidth <= 0: Silverman per cell over
 * the stencil. dv = 3 with uniform_w > 0 sums over unordered pairs (symmetric weights;
 * a second exponential only across two cells' Silverman bandwidths). On den <= 0 / non-finite: SPIC_FLAG_ISOLATED and *bad_pid = pid of the first
 * offending particle in (cell, pid) order (bad_pid must be preset to INT64_MAX). */
int spic_blob(const float* xv, float* sw, const int32_t* perm, int64_t n, int32_t dv,
              const int32_t* cell_start, const int32_t* sub_start, int32_t M, int32_t S, double eta,
              double bandwidth, float uniform_w, float* h_cell, long long* bad_pid, int32_t* flags,
              void* scratch, size_t scratch_bytes, void* stream);

/* ---- SBTM score network (replaces mlp_forward score.py:80-86, _ism_kernel_shared
 *      score.py:128-187, _ism_kernel_perparticle score.py:190-251, ism_loss_and_grad
 *      score.py:303-338, AdamW.step score.py:371-386, sbtm_update score.py:547-588,
 *      _mse_kernel score.py:254-300) ---------------------------------------------------------
 * Parameter vector layout (float64 master and float32 working copy), P = 8H+... :
 *   W1[H][1+dv] row-major, b1[H], W2[dv][H] row-major, b2[dv]. */
int64_t spic_mlp_num_params(int32_t H, int32_t dv);
/* s = W2 softsign(W1 [x*x_scale; v] + b1) + b2. Input either sorted records (xv != NULL;
 * x' < 0 is mapped back by +L = 1/x_scale) or pid-order planes (x, v, ldv). Output either
 * into sw lanes (sw != NULL) or planes s[dv][lds]. */
int spic_mlp_forward(const float* params32, int32_t H, int32_t dv, const float* xv,
                     const float* x, const float* v, int64_t ldv, int64_t n, float x_scale,
                     float* sw, float* s, int64_t lds, void* stream);
size_t spic_ism_scratch_bytes(int64_t n, int32_t H, int32_t dv);
/* Per-block float64 partial sums of [loss, gW1, gb1, gW2, gb2, Phi] into scratch.
 * mode 0: exact divergence (coefficients sum_i W2[i,h] W1[h,1+i] formed in-kernel);
 * mode 1: shared Hutchinson probe Z = z[dv] (float32, device);
 * mode 2: per-particle Rademacher probes Z[dv][ldz];
 * mode 3: weighted MSE to target Z[dv][ldz] with weights w*inv_wsum (pretraining).
 * Input: sorted records xv/sw (xv != NULL; x' < 0 mapped back by +L) or planes x, v, w.
 * idx (nullable) maps kernel particle p to the source row of the planes and of Z. */
int spic_ism_partials_ex(const float* params32, int32_t H, int32_t dv, int32_t mode,
                         const float* xv, const float* sw, const float* x, const float* v,
                         int64_t ldv, const float* w, int64_t n, float x_scale, const float* Z,
                         int64_t ldz, const int32_t* idx, double inv_wsum, void* scratch,
                         size_t scratch_bytes, void* stream);
/* Single-CTA finalize of one ISM/MSE step: fixed-order reduction of the partials, the
 * coefficient-dependence terms of the divergence (div_mode 0 exact, 1 shared Hutchinson with
 * z_shared float32[dv]; 2 per-particle and 3 MSE have none), then (apply_step != 0) AdamW on
 * the float64 master parameters with the reference's restore-and-halve recovery.
 * opt_state (float64[4]) = {t, lr_current, base_lr, 0}; reset_lr restarts lr_current from
 * base_lr. Writes params64/m/v2 (in place), params32, grads_out[P] and loss_out (nullable). */
int spic_sbtm_finalize_ex(const void* scratch, int64_t n, int32_t H, int32_t dv,
                          int32_t div_mode, const float* z_shared, double* params64, double* m,
                          double* v2, double* opt_state, double beta1, double beta2, double eps,
                          double weight_decay, int32_t reset_lr, int32_t apply_step,
                          float* params32, double* grads_out, double* loss_out, int32_t* flags,
                          void* stream);

/* Byte offset of the reduced row [loss, grads (P), Phi (H)] (float64) inside the ISM scratch;
 * a domain-decomposed run allreduces this row between partials and finalize. */
int64_t spic_ism_row_offset(int64_t n, int32_t H, int32_t dv);
/* Plain AdamW step (ref: score.py:371-386) on a flat float64 vector with precomputed
 * gradients; opt_state = {t, unused, lr, 0}; t is incremented on device. */
int spic_adamw_step(double* params64, const double* grads64, double* m, double* v2, int64_t P,
                    double* opt_state, double beta1, double beta2, double eps,
                    double weight_decay, float* params32, void* stream);

/* ---- M1 extension: the BASELINE "2 x 128 SiLU" score network (no reference counterpart;
 *      the reference's softsign net is score.py:38-71). Hidden GEMMs on tcgen05 tensor cores
 *      in split-BF16 with float32 TMEM accumulation; H must be 128, dv = 3.
 * Params (float32 working copy / float64 master): W1[H][4], b1[H], W2[H][H], b2[H], W3[3][H],
 * b3[3]; u = [x * x_scale, v]. Inputs are cell-sorted records xv/sw (x' < 0 mapped back by
 * +L = 1/x_scale; weight in sw.w). ---------------------------------------------------------- */
int64_t spic_silu_num_params(int32_t H);
size_t spic_silu_scratch_bytes(int64_t n);
/* s into sw_out lanes 0..2 (lane 3 = the input weight); sw_out may alias sw. */
int spic_silu_forward(const float* params32, int32_t H, const float* xv, const float* sw,
                      int64_t n, float x_scale, float* sw_out, void* stream);
/* Per-CTA float64 partials of [loss, grads] of sum_p w_p (|s_p|^2 + 2 div_p) with the exact
 * divergence, reduced in fixed order into the row at spic_silu_row_offset(n). */
int spic_silu_ism_partials(const float* params32, int32_t H, const float* xv, const float* sw,
                           int64_t n, float x_scale, void* scratch, size_t scratch_bytes,
                           void* stream);
/* Weighted MSE (pretraining, ref: score.py:254-300 / 402-445 with this network): partials of
 * sum_p w_p inv_wsum |s_p - Z_p|^2 from pid-order planes x (scaled by x_scale), v[3][ldv],
 * w, targets Z[3][ldz]; idx (nullable) maps kernel particle p to the source row. */
int spic_silu_mse_partials(const float* params32, int32_t H, const float* x, const float* v,
                           int64_t ldv, const float* w, int64_t n, float x_scale,
                           const float* Z, int64_t ldz, const int32_t* idx, double inv_wsum,
                           void* scratch, size_t scratch_bytes, void* stream);
int64_t spic_silu_row_offset(int64_t n);
/* AdamW with restore-and-halve recovery on the reduced row (same contract as
 * spic_sbtm_finalize_ex; mse != 0 selects its div_mode 3 semantics). */
int spic_silu_finalize(void* scratch, int64_t n, int32_t H, int32_t mse, double* params64,
                       double* m, double* v2, double* opt_state, double beta1, double beta2,
                       double eps, double weight_decay, int32_t reset_lr, int32_t apply_step,
                       float* params32, double* grads_out, double* loss_out, int32_t* flags,
                       void* stream);
/* Tensor-core self-test: float32 [128][128] W, X, Y -> D1 = W X^T, D2 = W^T Y^T, D3 = Y^T X
 * through the same split-BF16 tcgen05 GEMM views the SiLU kernel uses. */
int spic_umma_selftest(const float* W, const float* X, const float* Y, float* D1, float* D2,
                       float* D3, void* stream);

/* ---- PIC (replaces interpolate_fields pic.py:61-74, lorentz_push pic.py:77-88,
 *      advance_positions pic.py:91-93 + wrap_position state.py:14-27, deposit
 *      pic.py:43-58, maxwell_step pic.py:96-110, vpl_field_step pic.py:113-115,
 *      poisson_solve pic.py:118-134, compute_diagnostics diagnostics.py:20-35) ---------------
 * Fields are float64 [M] arrays on device (E1, E2, B3); J is float64 [dv][M]. */
/* interpolate + Lorentz (v += dt(E + v x B)) + x += dt v1 + periodic wrap, in place. */
int spic_push(float* x, float* v, int64_t ldv, int64_t n, int32_t dv, const double* E1,
              const double* E2, const double* B3, int32_t M, double eta, float dt,
              int32_t* flags, void* stream);
/* Unfused forms of the push for the operator API: interpolate_fields (pic.py:61-74) ->
 * E_p float[dv][lde] = (E1, E2, 0), B_p float[3][ldb] = (0, 0, B3); lorentz_push
 * (pic.py:77-88): v += dt (E_p + v x B_p) with B = (0, 0, B3). */
int spic_interpolate(const float* x, int64_t n, int32_t dv, const double* E1, const double* E2,
                     const double* B3, int32_t M, double eta, float* Ep, int64_t lde, float* Bp,
                     int64_t ldb, void* stream);
int spic_lorentz(float* v, int64_t ldv, int64_t n, int32_t dv, const float* Ep, int64_t lde,
                 const float* Bp, int64_t ldb, float dt, int32_t* flags, void* stream);
size_t spic_deposit_scratch_bytes(int32_t M, int32_t dv);
/* rho[M], J[dv][M] from sorted records; then (field_mode 1 = VPL: E1 -= dt J1;
 * 2 = VML maxwell_step; 0 = none). diag_out (nullable) receives [E_E, E_B, E_l2]. */
int spic_deposit_field(const float* xv, const float* sw, int64_t n, int32_t dv,
                       const int32_t* cell_start, int32_t M, double eta, float uniform_w,
                       double* rho, double* J, int32_t field_mode, double dt, double* E1,
                       double* E2, double* B3, double* diag_out, int32_t* flags, void* scratch,
                       size_t scratch_bytes, void* stream);
/* Standalone field updates (for the operator API). */
int spic_field_step(double* E1, double* E2, double* B3, const double* J, int32_t M, double eta,
                    double dt, int32_t field_mode, double* diag_out, int32_t* flags,
                    void* stream);
/* E1 = spectral solve of -phi'' = rho - rho_ion, E1 = -phi' (single-CTA float64 DFT). */
int spic_poisson(const double* rho, double rho_ion, int32_t M, double eta, double* E1,
                 int32_t* flags, void* stream);
size_t spic_moments_scratch_bytes(int64_t n);
/* out (float64): [E_K, P_0..P_{dv-1}, sum w] over pid-order planes; also flags non-finite v. */
int spic_moments(const float* v, int64_t ldv, const float* w, int64_t n, int32_t dv,
                 float uniform_w, double* out, int32_t* flags, void* scratch,
                 size_t scratch_bytes, void* stream);

/* ---- cell-range domain decomposition (the reference is single-
 *      process: these replace the per-rank bookkeeping of its run loop, run.py:81-118, when
 *      particles are partitioned by cell over ranks) ------------------------------------------
 * Message = float4 pairs: pair 0 = header int32 {rows, rows in the receiver's owned cells,
 * rows dropped for capacity, 0}; pair r+1 = (x, v0, v1, v2), (w, gid as int32 bits, 0, 0).
 * send_cells / recv_cells are HOST int32[4]: two cell ranges [a0, a1) and [b0, b1) (empty when
 * a1 <= a0) giving the cyclic cell range to send and its part owned by the receiver. Rows are
 * read from pid-order planes through perm (sorted position -> pid) over cell_start. */
int spic_dist_pack(const float* x, const float* v, int64_t ldv, int32_t dv, const float* w,
                   float uniform_w, const int32_t* gid, const int32_t* perm,
                   const int32_t* cell_start, int32_t M, const int32_t* send_cells,
                   const int32_t* recv_cells, int64_t cap, float* msg, void* stream);
/* rows [0, rows) of a message -> planes at [at, at + rows) (w nullable). */
int spic_dist_unpack(const float* msg, int64_t rows, int64_t at, float* x, float* v, int64_t ldv,
                     int32_t dv, float* w, int32_t* gid, void* stream);
size_t spic_dist_epilogue_scratch_bytes(void);
/* Collision epilogue over the owned sorted positions [cell_start[lo], cell_start[hi]) (read
 * on device): v_new = v[perm[k]] - nu_dt U[:, k]; the rank's next particle state is written
 * compacted in sorted order (out_x/out_v/out_w/out_gid at k - cell_start[lo]); red_out
 * (float64[6]) = [H_dot, E_K, P_0, P_1, P_2, sum w] over those particles. */
int spic_dist_epilogue(const float* U_sorted, int64_t ldu, const float* sw, const int32_t* perm,
                       const int32_t* cell_start, int32_t lo, int32_t hi, int32_t dv, float nu_dt,
                       const float* x, const float* v, int64_t ldv, const float* w,
                       const int32_t* gid, float* out_x, float* out_v, int64_t ldo,
                       float* out_w, int32_t* out_gid, double* red_out, int32_t* flags,
                       void* scratch, size_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif
