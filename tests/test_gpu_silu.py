"""GPU parity of the SiLU score network (extension M1, tcgen05 split-BF16 hidden GEMMs)
against the float64 oracle (oracle/silu_oracle.py, itself pinned to torch autograd).

Tolerances (stated; there is no reference implementation of this network): the split-BF16
products are accurate to ~2^-16 relative with float32 accumulation, so
  * raw GEMM self-test: max |err| <= 3e-5 * max |ref|;
  * scores: relative L2 <= 1e-4 and per particle |err| <= 1e-4 * max |ref|;
  * ISM loss <= 1e-4 relative, gradients <= 1e-4 relative L2 per parameter tensor;
  * network outputs after K AdamW steps: relative L2 <= 1e-4.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import silu_oracle as so  # noqa: E402

H = 128


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_25832_b200 import _lib

    _lib.load()
    return _lib


def relL2(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _params(seed=0, bias=0.3):
    rng = np.random.default_rng(seed)
    p = so.glorot(H, rng)
    p[4 * H:5 * H] = rng.normal(0, bias, H)
    p[5 * H + H * H:6 * H + H * H] = rng.normal(0, bias, H)
    p[-3:] = rng.normal(0, bias, 3)
    return p.astype(np.float32).astype(np.float64)  # the kernels read the float32 copy


def _ensemble(n, L, seed=1):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, L, n).astype(np.float32).astype(np.float64)
    v = rng.normal(0, 1.0, (n, 3)).astype(np.float32).astype(np.float64)
    w = np.full(n, L / n, dtype=np.float32).astype(np.float64)
    return x, v, w


def _net(params):
    from paper_2603_25832_b200.silu_net import SiluScoreNet

    net = SiluScoreNet()
    net.set_flat(params)
    return net


def test_umma_selftest_all_operand_views(lib):
    rng = np.random.default_rng(0)
    W, X, Y = (torch.tensor(rng.normal(size=(H, H)), dtype=torch.float32, device="cuda")
               for _ in range(3))
    D = [torch.empty(H, H, dtype=torch.float32, device="cuda") for _ in range(3)]
    lib.call("spic_umma_selftest", *(lib.ptr(t) for t in (W, X, Y, *D)), lib.stream_handle())
    torch.cuda.synchronize()
    Wd, Xd, Yd = W.double(), X.double(), Y.double()
    refs = [Wd @ Xd.T, Wd.T @ Yd.T, Yd.T @ Xd]
    for name, got, ref in zip(("W X^T", "W^T Y^T", "Y^T X"), D, refs):
        err = float((got.double() - ref).abs().max() / ref.abs().max())
        assert err <= 3e-5, (name, err)


@pytest.mark.parametrize("n", [1, 31, 1000, 148 * 32 * 2 + 7])
def test_silu_forward_matches_oracle(lib, n):
    from paper_2603_25832_b200.silu_net import silu_forward

    L = 4 * math.pi
    params = _params()
    x, v, _ = _ensemble(n, L)
    s = silu_forward(_net(params), x, v, L).cpu().numpy()
    ref, _ = so.forward(params, so.inputs(x, v, L), H)
    assert relL2(s, ref) <= 1e-4
    assert np.max(np.abs(s - ref)) <= 1e-4 * np.max(np.abs(ref))


@pytest.mark.parametrize("n", [5, 4099, 148 * 32 * 3 + 11, 250007])
def test_silu_ism_loss_and_grad_matches_oracle(lib, n):
    """250 007 particles = ~35 chunks per CTA: float32 TMEM accumulation of dW2 and M over a
    long chunk sequence still meets the tolerance."""
    from paper_2603_25832_b200.silu_net import silu_ism_loss_and_grad

    L = 4 * math.pi
    params = _params(seed=n)
    x, v, w = _ensemble(n, L, seed=n + 1)
    net = _net(params)
    loss, g = silu_ism_loss_and_grad(net, x, v, w, L)
    g = g.cpu().numpy()
    ref_loss, ref_g = so.ism_loss_and_grad(params, so.inputs(x, v, L), w, H)
    assert abs(loss - ref_loss) <= 1e-4 * abs(ref_loss)
    for (a, b, _), name in zip(net._slices(), ("W1", "b1", "W2", "b2", "W3", "b3")):
        assert relL2(g[a:b], ref_g[a:b]) <= 1e-4, (name, relL2(g[a:b], ref_g[a:b]))


def test_silu_ism_is_bit_reproducible_over_many_launches(lib):
    """The ISM kernel synchronises its phases with warpgroup barriers, mbarriers and hand-off
    barriers only (no CTA-wide barrier inside a chunk). 40 launches on the same 2^19 + 77
    particles (~74 chunks per CTA, flushes of the TMEM accumulators included) must give the
    same loss and gradient bits every time — any race between a warpgroup's partials, the
    chunk records or the operand tiles would show up as a difference."""
    from paper_2603_25832_b200.silu_net import silu_ism_loss_and_grad

    L = 4 * math.pi
    n = (1 << 19) + 77
    params = _params(seed=11)
    x, v, w = _ensemble(n, L, seed=12)
    net = _net(params)
    loss0, g0 = silu_ism_loss_and_grad(net, x, v, w, L)
    g0 = g0.clone()
    for _ in range(39):
        loss, g = silu_ism_loss_and_grad(net, x, v, w, L)
        assert loss == loss0
        assert torch.equal(g, g0)


def test_silu_sorted_records_quirk_and_weights(lib):
    """Record inputs: x' = x - L (the %M quirk record) maps back to x; per-particle weights."""
    from paper_2603_25832_b200 import _lib
    from paper_2603_25832_b200.silu_net import _silu_finalize, _silu_partials, records
    from paper_2603_25832_b200.score import AdamW

    n, L = 700, 10 * math.pi
    params = _params(seed=5)
    x, v, _ = _ensemble(n, L, seed=6)
    w = np.random.default_rng(7).uniform(0.2, 2.0, n).astype(np.float32).astype(np.float64)
    net = _net(params)
    xv, sw = records(x, v, w, L, torch.device("cuda"))
    xv[::7, 0] -= L  # quirk records
    buf = _silu_partials(net, xv, sw, n, L)
    g = torch.empty(net.n_params, dtype=torch.float64, device="cuda")
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    _silu_finalize(net, buf, n, AdamW(device="cuda"), grads_out=g, loss_out=loss)
    ref_loss, ref_g = so.ism_loss_and_grad(params, so.inputs(x, v, L), w, H)
    assert abs(float(loss.item()) - ref_loss) <= 1e-4 * abs(ref_loss)
    assert relL2(g.cpu().numpy(), ref_g) <= 1e-4
    out = sw.clone()
    _lib.call("spic_silu_forward", _lib.ptr(net.params32), H, _lib.ptr(xv), _lib.ptr(sw), n,
              float(1 / L), _lib.ptr(out), _lib.stream_handle())
    s_ref, _ = so.forward(params, so.inputs(x, v, L), H)
    assert relL2(out[:, :3].cpu().numpy(), s_ref) <= 1e-4
    np.testing.assert_array_equal(out[:, 3].cpu().numpy(), sw[:, 3].cpu().numpy())


def test_silu_trainer_k_steps_matches_oracle_adamw(lib):
    from paper_2603_25832_b200.score import AdamW
    from paper_2603_25832_b200.silu_net import SiluTrainer, silu_forward
    from paper_2603_25832_b200.state import ParticleEnsemble

    n, L, K, lr = 3000, 4 * math.pi, 4, 1e-3
    params = _params(seed=9)
    x, v, w = _ensemble(n, L, seed=10)
    net = _net(params)
    p = ParticleEnsemble.from_arrays(x, v, w)
    tr = SiluTrainer(net, AdamW(lr=lr, weight_decay=0.0, device="cuda"), K, L)
    tr.run(n, particles=p)
    u = so.inputs(x, v, L)
    P = params.copy()
    m = np.zeros_like(P)
    v2 = np.zeros_like(P)
    losses = []
    for t in range(1, K + 1):
        loss, g = so.ism_loss_and_grad(P, u, w, H)
        losses.append(loss)
        P, m, v2 = so.adamw_step(P, g, m, v2, t, lr)
    np.testing.assert_allclose(tr.losses[:K].cpu().numpy(), losses, rtol=1e-4)
    s_dev = silu_forward(net, x, v, L).cpu().numpy()
    s_ref, _ = so.forward(P, u, H)
    assert relL2(s_dev, s_ref) <= 1e-4


def test_engine_step_with_silu_estimator_and_graph(lib):
    """Config-0-shaped engine steps with the SiLU estimator: collisions conserve momentum,
    the captured CUDA graph reproduces the eager step bit for bit."""
    from paper_2603_25832_b200.engine import Simulation
    from paper_2603_25832_b200.pic import Grid, deposit, poisson_solve
    from paper_2603_25832_b200.silu_net import SiluEstimator, SiluScoreNet
    from paper_2603_25832_b200.state import FieldState, ParticleEnsemble

    n, M, L = 20000, 32, 4 * math.pi
    x, v, w = _ensemble(n, L, seed=12)
    grid = Grid(M, L / M)

    def make():
        p = ParticleEnsemble.from_arrays(x, v, w)
        rho, _ = deposit(p, grid)
        rho_ion = float(rho.sum()) * grid.eta / L
        f = FieldState.zeros(M, 3, rho_ion)
        f.E1.copy_(poisson_solve(rho, rho_ion, grid))
        r = np.random.default_rng(3)
        net = SiluScoreNet.init_glorot(r)
        est = SiluEstimator(net, L, 3, r, lr=1e-3, weight_decay=0.0)
        return Simulation(p, f, grid, dt=0.05, nu=0.1, mode="VPL", gamma=-3.0, estimator=est,
                          max_rows=8), p

    a, pa = make()
    b, pb = make()
    for k in range(1, 4):
        a.step(k)
    b.step(1)
    b.capture(2)
    b.replay(2)
    b.replay(3)
    torch.cuda.synchronize()
    assert torch.equal(pa.x, pb.x) and torch.equal(pa.vp, pb.vp)
    d = a.diag.cpu().numpy()
    assert np.all(np.isfinite(d[1:4]))
    a.check()


def test_silu_mse_partials_match_oracle(lib):
    """Pretraining loss (weighted MSE to a target, idx-mapped minibatch) vs the oracle."""
    from paper_2603_25832_b200.score import AdamW, _planes
    from paper_2603_25832_b200.silu_net import _silu_finalize, _silu_mse_partials

    n, L = 2500, 4 * math.pi
    params = _params(seed=21)
    x, v, _ = _ensemble(n, L, seed=22)
    rng = np.random.default_rng(23)
    w = rng.uniform(0.5, 1.5, n).astype(np.float32).astype(np.float64)
    target = rng.normal(size=(n, 3)).astype(np.float32).astype(np.float64)
    idx = rng.permutation(n)[:1000]
    net = _net(params)
    dev = torch.device("cuda")
    xn = torch.tensor(x / L, dtype=torch.float32, device=dev)
    vp = _planes(v, dev)
    wd = torch.tensor(w, dtype=torch.float32, device=dev)
    T = _planes(target, dev)
    idx_d = torch.tensor(idx, dtype=torch.int32, device=dev)
    inv = 1.0 / float(w[idx].sum())
    buf = _silu_mse_partials(net, 1000, x=xn, vp=vp, w=wd, Z=T, ldz=n, idx=idx_d, inv_wsum=inv,
                             ldv=n)
    g = torch.empty(net.n_params, dtype=torch.float64, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    _silu_finalize(net, buf, 1000, AdamW(device=dev), grads_out=g, loss_out=loss, mse=True)
    u = so.inputs(x[idx], v[idx], L)
    ref_loss, ref_g = so.mse_loss_and_grad(params, u, w[idx], target[idx], H)
    assert abs(float(loss.item()) - ref_loss) <= 1e-4 * abs(ref_loss)
    g = g.cpu().numpy()
    for (a, b, _), name in zip(net._slices(), ("W1", "b1", "W2", "b2", "W3", "b3")):
        assert relL2(g[a:b], ref_g[a:b]) <= 1e-4, (name, relL2(g[a:b], ref_g[a:b]))


def test_run_end_to_end_with_silu_net(lib, tmp_path):
    """run() with DeviceOptions(score_net="silu"): pretraining on the analytic score, SBTM
    steps with the SiLU net, diagnostics finite and momentum conserved by the collisions."""
    from paper_2603_25832_b200.config import DeviceOptions, build_config
    from paper_2603_25832_b200.run import run

    cfg = build_config(overrides=dict(preset="landau_damping", n=8192, M=16, dt=0.05,
                                      t_final=0.2, K=2, divergence="exact", hidden=128,
                                      pretrain_budget=300, pretrain_batch=2048, seed=3))
    recs = run(cfg, str(tmp_path), options=DeviceOptions(score_net="silu"))
    assert len(recs) == 5
    E = np.array([r.E_total for r in recs])
    assert np.all(np.isfinite(E))
    assert abs(E[-1] - E[0]) <= 1e-2 * abs(E[0])
    assert (tmp_path / "diagnostics.csv").exists()


def test_silu_forward_large_n_repeatable(lib):
    """n = 2^22 (~590 chunks per CTA through the double-buffered forward pipeline): three
    launches are bit-identical and a sample matches the float64 oracle. Guards the per-chunk
    hand-off between the compute warpgroups and the MMA-issuing warp."""
    from paper_2603_25832_b200.silu_net import silu_forward

    n, L = 1 << 22, 2 * math.pi / 1.25
    params = _params(seed=3)
    x, v, _ = _ensemble(n, L, seed=4)
    net = _net(params)
    outs = [silu_forward(net, x, v, L).cpu().numpy() for _ in range(3)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    idx = np.random.default_rng(5).choice(n, 4096, replace=False)
    ref, _ = so.forward(params, so.inputs(x[idx], v[idx], L), H)
    assert relL2(outs[0][idx], ref) <= 1e-4


@pytest.mark.parametrize("lr", [1e-3, 1e300])
def test_silu_multicta_finalize_equals_single_cta(lib, lr):
    """The multi-CTA AdamW finalize (default) against the single-CTA kernel
    (SPIC_SILU_FINALIZE=1): identical parameters, moments, optimizer state and flags, also when
    the first candidate is non-finite (lr = 1e300: restore and halve until finite)."""
    import os

    from paper_2603_25832_b200.score import AdamW
    from paper_2603_25832_b200.silu_net import _silu_finalize, _silu_partials, records
    from paper_2603_25832_b200.state import new_flags

    L = 4 * math.pi
    params = _params(seed=7)
    x, v, w = _ensemble(20000, L, seed=8)
    out = []
    for env in ({}, {"SPIC_SILU_FINALIZE": "1"}):
        old = {k: os.environ.get(k) for k in ("SPIC_SILU_FINALIZE",)}
        os.environ.update(env)
        try:
            net = _net(params)
            xv, sw = records(x, v, w, L, "cuda")
            opt = AdamW(lr=lr, device="cuda")
            flags = new_flags("cuda")
            for _ in range(2):
                buf = _silu_partials(net, xv, sw, xv.shape[0], L)
                _silu_finalize(net, buf, xv.shape[0], opt, reset_lr=False, apply_step=True,
                               flags=flags)
            torch.cuda.synchronize()
            out.append([t.cpu().numpy().copy() for t in (net.params64, net.params32, opt.m, opt.v,
                                                          opt.state, flags)])
        finally:
            for k, val in old.items():
                if val is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = val
    for a, b in zip(*out):
        assert np.array_equal(a, b)
    if lr > 1.0:
        assert out[0][5][lib.FLAG_LR_HALVINGS] > 0
