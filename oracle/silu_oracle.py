"""TEST INFRASTRUCTURE ONLY — float64 oracle for the BASELINE "2x128 SiLU" score network (M1).

The reference ships only the one-hidden-layer softsign net (ref: score.py:38-71); BASELINE
configs 0/2 name a deeper network, "score MLP (x,v) in R^4 -> 2x128 SiLU -> R^3", which this
package adds as an extension. There is no reference
implementation to pin against, so this restatement is pinned instead against torch float64
autograd (double backward through the exact Jacobian trace) in
``tests/test_silu_oracle.py``, and by central finite differences.

Network (u = [x/L, v0, v1, v2], parameters in this flat order):
    a1 = W1 u + b1,  h1 = silu(a1)          W1 [H][4], b1 [H]
    a2 = W2 h1 + b2, h2 = silu(a2)          W2 [H][H], b2 [H]
    s  = W3 h2 + b3                         W3 [3][H], b3 [3]
ISM loss (exact divergence, ref: score.py:303-338 with this network):
    loss = sum_p w_p (|s_p|^2 + 2 div_p),  div = sum_k d s_k / d v_k
with the tangents t1_k = silu'(a1) * W1[:, 1+k], c2_k = W2 t1_k, t2_k = silu'(a2) * c2_k,
div = sum_k W3[k] . t2_k. Gradients are the analytic reverse-mode sweep the CUDA kernel
implements (paper_2603_25832_b200/csrc/silu.cu).

Only tests/, __graft_entry__.smoke() and bench.py may import this module.
"""

from __future__ import annotations

import numpy as np


def n_params(H: int) -> int:
    return 4 * H + H + H * H + H + 3 * H + 3


def split(params: np.ndarray, H: int):
    p = np.asarray(params, dtype=np.float64)
    o = 0
    W1 = p[o:o + 4 * H].reshape(H, 4); o += 4 * H
    b1 = p[o:o + H]; o += H
    W2 = p[o:o + H * H].reshape(H, H); o += H * H
    b2 = p[o:o + H]; o += H
    W3 = p[o:o + 3 * H].reshape(3, H); o += 3 * H
    b3 = p[o:o + 3]; o += 3
    assert o == p.size
    return W1, b1, W2, b2, W3, b3


def glorot(H: int, rng: np.random.Generator) -> np.ndarray:
    """Glorot-uniform W1, W2, W3 drawn in that order, zero biases (the package's init)."""
    def uni(fan_out, fan_in):
        lim = np.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-lim, lim, size=(fan_out, fan_in))
    W1, W2, W3 = uni(H, 4), uni(H, H), uni(3, H)
    return np.concatenate([W1.ravel(), np.zeros(H), W2.ravel(), np.zeros(H), W3.ravel(),
                           np.zeros(3)])


def _sig(a):
    return 1.0 / (1.0 + np.exp(-a))


def _silu_terms(a):
    s = _sig(a)
    return a * s, s * (1.0 + a * (1.0 - s)), s * (1.0 - s) * (2.0 + a * (1.0 - 2.0 * s))


def inputs(x, v, L: float) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    return np.concatenate([(x / L)[:, None], v], axis=1)


def forward(params, u, H: int, with_div: bool = True):
    """s [n][3] and the divergence div [n] (None unless with_div)."""
    W1, b1, W2, b2, W3, b3 = split(params, H)
    a1 = u @ W1.T + b1
    h1, d1, _ = _silu_terms(a1)
    a2 = h1 @ W2.T + b2
    h2, d2, _ = _silu_terms(a2)
    s = h2 @ W3.T + b3
    if not with_div:
        return s, None
    div = np.zeros(u.shape[0])
    for k in range(3):
        c2 = (d1 * W1[:, 1 + k]) @ W2.T
        div += (d2 * c2) @ W3[k]
    return s, div


def ism_loss_and_grad(params, u, w, H: int):
    """(loss, grads[P]) of sum_p w_p (|s_p|^2 + 2 div_p), float64."""
    W1, b1, W2, b2, W3, b3 = split(params, H)
    w = np.asarray(w, dtype=np.float64)
    a1 = u @ W1.T + b1
    h1, d1, e1 = _silu_terms(a1)
    a2 = h1 @ W2.T + b2
    h2, d2, e2 = _silu_terms(a2)
    s = h2 @ W3.T + b3
    t1 = [d1 * W1[:, 1 + k] for k in range(3)]
    c2 = [t @ W2.T for t in t1]
    t2 = [d2 * c for c in c2]
    div = sum(t2[k] @ W3[k] for k in range(3))
    loss = float(np.sum(w * (np.sum(s * s, axis=1) + 2.0 * div)))

    tw = 2.0 * w[:, None]                        # d loss / d div_p = 2 w_p
    gs = tw * s                                  # d loss / d s
    gW3 = gs.T @ h2 + np.stack([(tw * t2[k]).sum(axis=0) for k in range(3)])
    gb3 = gs.sum(axis=0)
    dh2 = gs @ W3
    q = sum(c2[k] * W3[k] for k in range(3))
    da2 = d2 * dh2 + tw * e2 * q
    dc2 = [tw * d2 * W3[k] for k in range(3)]
    gb2 = da2.sum(axis=0)
    gW2 = da2.T @ h1 + sum(dc2[k].T @ t1[k] for k in range(3))
    dh1 = da2 @ W2
    dt1 = [dc @ W2 for dc in dc2]
    da1 = d1 * dh1 + e1 * sum(W1[:, 1 + k] * dt1[k] for k in range(3))
    gb1 = da1.sum(axis=0)
    gW1 = da1.T @ u
    for k in range(3):
        gW1[:, 1 + k] += (d1 * dt1[k]).sum(axis=0)
    grads = np.concatenate([gW1.ravel(), gb1, gW2.ravel(), gb2, gW3.ravel(), gb3])
    return loss, grads


def mse_loss_and_grad(params, u, w, target, H: int):
    """(loss, grads[P]) of sum_p (w_p / sum w) |s_p - target_p|^2 (pretraining, ref:
    score.py:254-300 / 340-350 restated for this network), float64."""
    W1, b1, W2, b2, W3, b3 = split(params, H)
    wi = np.asarray(w, dtype=np.float64) / float(np.sum(w))
    a1 = u @ W1.T + b1
    h1, d1, _ = _silu_terms(a1)
    a2 = h1 @ W2.T + b2
    h2, d2, _ = _silu_terms(a2)
    r = h2 @ W3.T + b3 - np.asarray(target, dtype=np.float64)
    loss = float(np.sum(wi * np.sum(r * r, axis=1)))
    gs = 2.0 * wi[:, None] * r
    gW3, gb3 = gs.T @ h2, gs.sum(axis=0)
    da2 = d2 * (gs @ W3)
    gW2, gb2 = da2.T @ h1, da2.sum(axis=0)
    da1 = d1 * (da2 @ W2)
    gW1, gb1 = da1.T @ u, da1.sum(axis=0)
    return loss, np.concatenate([gW1.ravel(), gb1, gW2.ravel(), gb2, gW3.ravel(), gb3])


def adamw_step(params, grads, m, v2, t: int, lr: float, betas=(0.9, 0.999), eps=1e-8,
               weight_decay=0.0):
    """One AdamW step (ref: score.py:371-386) on flat float64 arrays; returns new arrays."""
    b1, b2 = betas
    p = params.copy()
    if weight_decay != 0.0:
        p -= lr * weight_decay * p
    m = b1 * m + (1.0 - b1) * grads
    v2 = b2 * v2 + (1.0 - b2) * grads * grads
    p -= lr * (m / (1.0 - b1 ** t)) / (np.sqrt(v2 / (1.0 - b2 ** t)) + eps)
    return p, m, v2
