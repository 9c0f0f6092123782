// adamw.cuh — the tail of every score-net training step: AdamW on the float64 master
// parameters with the reference's restore-and-halve recovery (ref: score.py:371-386,
// score.py:568-587). Called by all threads of a single-CTA finalize kernel; `grad` and `cand`
// (candidate parameters, P doubles) may live in shared or global memory.
#pragma once
#include "common.cuh"

namespace spic {

// mse: pretraining semantics (a non-finite loss raises at once; the step is always applied)
__device__ __forceinline__ void adamw_with_recovery(
    double loss, const double* grad, int64_t P, bool mse, double* __restrict__ params,
    double* __restrict__ m, double* __restrict__ v2, double* __restrict__ opt, double beta1,
    double beta2, double eps, double wd, int reset_lr, int apply_step, float* __restrict__ params32,
    double* __restrict__ grads_out, double* __restrict__ loss_out, double* cand, int32_t* flags) {
  if (threadIdx.x == 0 && loss_out) *loss_out = loss;
  if (grads_out)
    for (int64_t k = threadIdx.x; k < P; k += blockDim.x) grads_out[k] = grad[k];
  if (!apply_step) return;
  // a fatal divergence earlier in this update raised in the reference: no further steps
  if (flags && flags[SPIC_FLAG_TRAIN_FATAL]) return;
  double lr = reset_lr ? opt[2] : opt[1];
  if (!isfinite(loss)) {
    // ism_loss_and_grad raises before the optimizer step; sbtm_update restores (a no-op),
    // halves lr and retries the same (non-finite) loss until lr < 1e-12 -> RuntimeError.
    // The MSE path (pretraining) raises straight away (ref: score.py:348-349).
    if (threadIdx.x == 0) {
      int halvings = 0;
      if (!mse)
        do {
          lr *= 0.5;
          ++halvings;
        } while (!(lr < 1e-12));
      atomicAdd(flags + SPIC_FLAG_LR_HALVINGS, halvings);
      atomicOr(flags + SPIC_FLAG_TRAIN_FATAL, 1);
      opt[1] = lr;
    }
    return;
  }
  double t = opt[0];
  for (;;) {
    t += 1.0;
    const double bc1 = 1.0 - pow(beta1, t), bc2 = 1.0 - pow(beta2, t);
    int ok = 1;
    for (int64_t k = threadIdx.x; k < P; k += blockDim.x) {
      double p = params[k];
      if (wd != 0.0) p -= lr * wd * p;
      const double gk = grad[k];
      const double mk = beta1 * m[k] + (1.0 - beta1) * gk;
      const double vk = beta2 * v2[k] + (1.0 - beta2) * gk * gk;
      m[k] = mk;
      v2[k] = vk;
      p -= lr * (mk / bc1) / (sqrt(vk / bc2) + eps);
      cand[k] = p;
      ok &= isfinite(p) ? 1 : 0;
    }
    ok = __syncthreads_and(ok);
    if (ok || mse) {
      for (int64_t k = threadIdx.x; k < P; k += blockDim.x) {
        params[k] = cand[k];
        params32[k] = (float)cand[k];
      }
      break;
    }
    // restore (params untouched), halve, retry with the same gradient (ref: score.py:578-585)
    lr *= 0.5;
    if (threadIdx.x == 0) atomicAdd(flags + SPIC_FLAG_LR_HALVINGS, 1);
    if (lr < 1e-12) {
      if (threadIdx.x == 0) atomicOr(flags + SPIC_FLAG_TRAIN_FATAL, 1);
      break;
    }
  }
  if (threadIdx.x == 0) {
    opt[0] = t;
    opt[1] = lr;
  }
}

// Multi-CTA form of adamw_with_recovery for large parameter vectors (the SiLU net's 17.5 k):
// every CTA runs the first AdamW attempt on its slice (m, v updated in place as in the
// single-CTA loop, candidates kept), all CTAs meet at a spin barrier (atomic ticket; the
// launch is a few dozen CTAs, all co-resident), and each commits its own slice if every
// slice is finite; otherwise CTA 0 continues the restore-and-halve loop alone (rare).
// `sync` = [ticket, ok flags per CTA], ticket zeroed by the caller before the launch. Same
// arithmetic per parameter as the single-CTA kernel: identical results.
__device__ __forceinline__ void adamw_with_recovery_mc(
    double loss, const double* grad, int64_t P, bool mse, double* __restrict__ params,
    double* __restrict__ m, double* __restrict__ v2, double* __restrict__ opt, double beta1,
    double beta2, double eps, double wd, int reset_lr, int apply_step, float* __restrict__ params32,
    double* __restrict__ grads_out, double* __restrict__ loss_out, double* cand, int32_t* flags,
    int32_t* sync) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  if (gtid == 0 && loss_out) *loss_out = loss;
  if (grads_out)
    for (int64_t k = gtid; k < P; k += gstride) grads_out[k] = grad[k];
  if (!apply_step) return;
  if (flags && flags[SPIC_FLAG_TRAIN_FATAL]) return;  // every CTA reads it before the barrier
  if (!isfinite(loss)) {  // see adamw_with_recovery; one thread records it
    if (gtid == 0) {
      double lr = reset_lr ? opt[2] : opt[1];
      int halvings = 0;
      if (!mse)
        do {
          lr *= 0.5;
          ++halvings;
        } while (!(lr < 1e-12));
      atomicAdd(flags + SPIC_FLAG_LR_HALVINGS, halvings);
      atomicOr(flags + SPIC_FLAG_TRAIN_FATAL, 1);
      opt[1] = lr;
    }
    return;
  }
  double lr = reset_lr ? opt[2] : opt[1];
  double t = opt[0] + 1.0;
  __shared__ int s_all;
  {
    const double bc1 = 1.0 - pow(beta1, t), bc2 = 1.0 - pow(beta2, t);
    int ok = 1;
    for (int64_t k = gtid; k < P; k += gstride) {
      double p = params[k];
      if (wd != 0.0) p -= lr * wd * p;
      const double gk = grad[k];
      const double mk = beta1 * m[k] + (1.0 - beta1) * gk;
      const double vk = beta2 * v2[k] + (1.0 - beta2) * gk * gk;
      m[k] = mk;
      v2[k] = vk;
      p -= lr * (mk / bc1) / (sqrt(vk / bc2) + eps);
      cand[k] = p;
      ok &= isfinite(p) ? 1 : 0;
    }
    ok = __syncthreads_and(ok);
    if (threadIdx.x == 0) {
      sync[1 + blockIdx.x] = ok;
      __threadfence();
      atomicAdd(sync, 1);
      while (((volatile int32_t*)sync)[0] < (int)gridDim.x) {
      }
      __threadfence();
      int all = 1;
      for (int b = 0; b < (int)gridDim.x; ++b) all &= ((volatile int32_t*)sync)[1 + b];
      s_all = all;
    }
    __syncthreads();
    if (s_all || mse) {
      for (int64_t k = gtid; k < P; k += gstride) {  // own slice: own candidates
        params[k] = cand[k];
        params32[k] = (float)cand[k];
      }
      if (gtid == 0) {
        opt[0] = t;
        opt[1] = lr;
      }
      return;
    }
  }
  if (blockIdx.x != 0) return;
  // CTA 0 alone: restore (params untouched), halve, retry with the same gradient
  for (;;) {
    lr *= 0.5;
    if (threadIdx.x == 0) atomicAdd(flags + SPIC_FLAG_LR_HALVINGS, 1);
    if (lr < 1e-12) {
      if (threadIdx.x == 0) atomicOr(flags + SPIC_FLAG_TRAIN_FATAL, 1);
      break;
    }
    t += 1.0;
    const double bc1 = 1.0 - pow(beta1, t), bc2 = 1.0 - pow(beta2, t);
    int ok = 1;
    for (int64_t k = threadIdx.x; k < P; k += blockDim.x) {
      double p = params[k];
      if (wd != 0.0) p -= lr * wd * p;
      const double gk = grad[k];
      const double mk = beta1 * ((volatile double*)m)[k] + (1.0 - beta1) * gk;
      const double vk = beta2 * ((volatile double*)v2)[k] + (1.0 - beta2) * gk * gk;
      m[k] = mk;
      v2[k] = vk;
      p -= lr * (mk / bc1) / (sqrt(vk / bc2) + eps);
      cand[k] = p;
      ok &= isfinite(p) ? 1 : 0;
    }
    ok = __syncthreads_and(ok);
    if (ok) {
      for (int64_t k = threadIdx.x; k < P; k += blockDim.x) {
        params[k] = cand[k];
        params32[k] = (float)cand[k];
      }
      break;
    }
  }
  if (threadIdx.x == 0) {
    opt[0] = t;
    opt[1] = lr;
  }
}

}  // namespace spic
