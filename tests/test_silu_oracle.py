"""Pins the float64 SiLU-net oracle (oracle/silu_oracle.py) against torch float64 autograd
(forward, exact Jacobian trace via autograd, and the ISM gradient via double backward) and
central finite differences. CPU only."""

import numpy as np
import pytest
import torch

from oracle import silu_oracle as so


def _case(n=37, H=16, seed=3):
    rng = np.random.default_rng(seed)
    params = so.glorot(H, rng)
    params[4 * H:5 * H] = rng.normal(0, 0.3, H)                 # nonzero b1
    params[5 * H + H * H:6 * H + H * H] = rng.normal(0, 0.3, H)  # nonzero b2
    params[-3:] = rng.normal(0, 0.3, 3)
    x = rng.uniform(0, 6.0, n)
    v = rng.normal(0, 1.0, (n, 3))
    w = rng.uniform(0.5, 1.5, n) / n
    return params, so.inputs(x, v, 6.0), w, H


def _torch_loss(params_t, u_t, w_t, H):
    o = 0
    W1 = params_t[o:o + 4 * H].reshape(H, 4); o += 4 * H
    b1 = params_t[o:o + H]; o += H
    W2 = params_t[o:o + H * H].reshape(H, H); o += H * H
    b2 = params_t[o:o + H]; o += H
    W3 = params_t[o:o + 3 * H].reshape(3, H); o += 3 * H
    b3 = params_t[o:o + 3]
    u = u_t.clone().requires_grad_(True)
    silu = torch.nn.functional.silu
    s = silu(silu(u @ W1.T + b1) @ W2.T + b2) @ W3.T + b3
    div = 0.0
    for k in range(3):
        gk = torch.autograd.grad(s[:, k].sum(), u, create_graph=True)[0]
        div = div + gk[:, 1 + k]
    return (w_t * ((s * s).sum(1) + 2.0 * div)).sum(), s, div


def test_forward_and_divergence_match_autograd():
    params, u, w, H = _case()
    s, div = so.forward(params, u, H)
    pt = torch.tensor(params, dtype=torch.float64)
    _, s_t, div_t = _torch_loss(pt, torch.tensor(u), torch.tensor(w), H)
    np.testing.assert_allclose(s, s_t.detach().numpy(), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(div, div_t.detach().numpy(), rtol=1e-11, atol=1e-13)


def test_ism_grad_matches_double_backward():
    params, u, w, H = _case()
    loss, g = so.ism_loss_and_grad(params, u, w, H)
    pt = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    lt, _, _ = _torch_loss(pt, torch.tensor(u), torch.tensor(w), H)
    (gt,) = torch.autograd.grad(lt, pt)
    assert loss == pytest.approx(float(lt.detach()), rel=1e-12)
    np.testing.assert_allclose(g, gt.numpy(), rtol=1e-10, atol=1e-12)


def test_ism_grad_finite_differences():
    params, u, w, H = _case(n=9, H=6)
    _, g = so.ism_loss_and_grad(params, u, w, H)
    rng = np.random.default_rng(0)
    for k in rng.choice(params.size, 12, replace=False):
        e = np.zeros_like(params)
        e[k] = 1e-6
        lp, _ = so.ism_loss_and_grad(params + e, u, w, H)
        lm, _ = so.ism_loss_and_grad(params - e, u, w, H)
        assert g[k] == pytest.approx((lp - lm) / 2e-6, rel=1e-5, abs=1e-8)


def test_param_layout():
    assert so.n_params(128) == 128 * 128 + 9 * 128 + 3 == 17539
    rng = np.random.default_rng(0)
    p = so.glorot(8, rng)
    W1, b1, W2, b2, W3, b3 = so.split(p, 8)
    assert W1.shape == (8, 4) and W2.shape == (8, 8) and W3.shape == (3, 8)
    assert not b1.any() and not b2.any() and not b3.any()
    assert np.abs(W2).max() <= np.sqrt(6.0 / 16)


def test_mse_grad_matches_autograd():
    params, u, w, H = _case()
    target = np.random.default_rng(4).normal(size=(u.shape[0], 3))
    loss, g = so.mse_loss_and_grad(params, u, w, target, H)
    pt = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    o = 0
    W1 = pt[o:o + 4 * H].reshape(H, 4); o += 4 * H
    b1 = pt[o:o + H]; o += H
    W2 = pt[o:o + H * H].reshape(H, H); o += H * H
    b2 = pt[o:o + H]; o += H
    W3 = pt[o:o + 3 * H].reshape(3, H); o += 3 * H
    b3 = pt[o:o + 3]
    silu = torch.nn.functional.silu
    s = silu(silu(torch.tensor(u) @ W1.T + b1) @ W2.T + b2) @ W3.T + b3
    wt = torch.tensor(w) / float(np.sum(w))
    lt = (wt * ((s - torch.tensor(target)) ** 2).sum(1)).sum()
    (gt,) = torch.autograd.grad(lt, pt)
    assert loss == pytest.approx(float(lt.detach()), rel=1e-12)
    np.testing.assert_allclose(g, gt.numpy(), rtol=1e-10, atol=1e-13)
