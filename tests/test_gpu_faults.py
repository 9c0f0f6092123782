"""GPU parity of the fault paths and of the analysis mode, against the reference's own outputs
(tests/golden/faults.npz, tests/golden/score_test.npz, made by tests/golden/make_golden.py)
and, for the SiLU network the reference does not have, against the float64 oracle driven
through the reference's sbtm_update semantics.

  * restore-and-halve recovery (ref: score.py:568-587, test_score.py:231-237): the warning
    list, the learning-rate floor, t and the restored parameters exactly; the recovered
    parameters to 1e-9 relative (the weight-decay overflow term dominates them and is exact in
    float64), Adam moments 1e-5 (softsign) / 1e-4 (SiLU) relative L2 (float32 gradients);
  * score_test (ref: run.py:134-185), blob estimator: x equal to the float32 rounding of the
    reference's x, v likewise, s_est and U relative L2 <= 1e-4 and per particle
    <= 1e-4 * max|ref|, the reported MSE 1e-4 relative.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import silu_oracle as so  # noqa: E402


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


def _softsign_net(g, prefix):
    from paper_2603_25832_b200.score import MlpScoreNet

    net = MlpScoreNet(3, g[prefix + "W1"].shape[0], device="cuda")
    net.set_params([g[prefix + k] for k in ("W1", "b1", "W2", "b2")])
    return net


def _fault_particles(g):
    from paper_2603_25832_b200.state import ParticleEnsemble

    return ParticleEnsemble.from_arrays(g["fault_x"], g["fault_v"], g["fault_w"])


def test_softsign_fatal_divergence_matches_reference(lib, golden):
    """Non-finite loss (W2[0,0] = inf): 30 halvings to the 1e-12 floor, RuntimeError, nothing
    stepped, lr restored on the host afterwards."""
    from paper_2603_25832_b200.score import AdamW, sbtm_update

    g = golden("faults.npz")
    net = _softsign_net(g, "faultA_init_")
    opt = AdamW(lr=1e-3, weight_decay=0.0, device="cuda")
    warn = []
    with pytest.raises(RuntimeError, match="training divergence"):
        sbtm_update(net, opt, _fault_particles(g), 2, L=4 * math.pi,
                    rng=np.random.default_rng(1), divergence="exact", warnings=warn)
    assert warn == [str(s) for s in g["faultA_warnings"]]
    assert opt.lr == float(g["faultA_lr_after"])
    assert opt.t == int(g["faultA_t"])
    for a, k in zip(net.numpy_params(), ("W1", "b1", "W2", "b2")):
        assert np.array_equal(a, g["faultA_final_" + k])


def test_softsign_overflow_recovery_matches_reference(lib, golden):
    """lr = wd = 1e155: the decoupled weight decay overflows, the step is restored and lr
    halved six times; m, v and t advance on every attempt (ref: score.py:371-386)."""
    from paper_2603_25832_b200.score import AdamW, sbtm_update

    g = golden("faults.npz")
    net = _softsign_net(g, "faultB_init_")
    opt = AdamW(lr=1e155, weight_decay=1e155, device="cuda")
    warn = []
    losses = sbtm_update(net, opt, _fault_particles(g), 1, L=4 * math.pi,
                         rng=np.random.default_rng(1), divergence="exact", warnings=warn)
    np.testing.assert_allclose(losses, g["faultB_losses"], rtol=1e-5)
    assert warn == [str(s) for s in g["faultB_warnings"]]
    assert opt.lr == float(g["faultB_lr_after"])
    assert opt.t == int(g["faultB_t"])
    for a, k in zip(net.numpy_params(), ("W1", "b1", "W2", "b2")):
        assert relL2(a, g["faultB_final_" + k]) <= 1e-9
    sl = net._slices()
    m, v = opt.m.cpu().numpy(), opt.v.cpu().numpy()
    for k, (a, b, _) in enumerate(sl):
        assert relL2(m[a:b], g[f"faultB_m{k}"].ravel()) <= 1e-5
        assert relL2(v[a:b], g[f"faultB_v{k}"].ravel()) <= 1e-5


# ------------------------------------------------------------------------------ SiLU network
def _silu_setup(seed, n=3000, L=4 * math.pi):
    from paper_2603_25832_b200.silu_net import SiluScoreNet
    from paper_2603_25832_b200.state import ParticleEnsemble

    rng = np.random.default_rng(seed)
    params = so.glorot(128, rng)
    params[4 * 128:5 * 128] = rng.normal(0, 0.3, 128)
    params = params.astype(np.float32).astype(np.float64)
    x = rng.uniform(0, L, n).astype(np.float32).astype(np.float64)
    v = rng.normal(0, 1.0, (n, 3)).astype(np.float32).astype(np.float64)
    w = np.full(n, L / n, dtype=np.float32).astype(np.float64)
    net = SiluScoreNet(device="cuda")
    net.set_flat(params)
    return net, params, ParticleEnsemble.from_arrays(x, v, w), (x, v, w, L)


def _oracle_update(params, x, v, w, L, K, lr, wd, betas=(0.9, 0.999), eps=1e-8):
    """The reference's sbtm_update loop (score.py:556-587) over the float64 SiLU oracle."""
    u = so.inputs(x, v, L)
    P, m, v2, t = params.copy(), np.zeros_like(params), np.zeros_like(params), 0
    b1, b2 = betas
    warn, losses = [], []
    for _ in range(K):
        while True:
            loss, g = so.ism_loss_and_grad(P, u, w, 128)
            ok = np.isfinite(loss)
            if ok:
                t += 1
                p = P.copy()
                if wd:
                    p -= lr * wd * p
                m = b1 * m + (1.0 - b1) * g
                v2 = b2 * v2 + (1.0 - b2) * g * g
                p -= lr * (m / (1.0 - b1 ** t)) / (np.sqrt(v2 / (1.0 - b2 ** t)) + eps)
                ok = bool(np.all(np.isfinite(p)))
            if ok:
                P = p
                losses.append(loss)
                break
            lr *= 0.5
            warn.append(f"training divergence: learning rate halved to {lr:g}")
            if lr < 1e-12:
                return P, m, v2, t, warn, losses, True
    return P, m, v2, t, warn, losses, False


def test_silu_overflow_recovery_matches_oracle(lib):
    from paper_2603_25832_b200.silu_net import SiluEstimator

    net, params, p, (x, v, w, L) = _silu_setup(11)
    est = SiluEstimator(net, L, 1, np.random.default_rng(0), lr=1e155, weight_decay=1e155)
    est.update(p)
    P, m, v2, t, warn, losses, fatal = _oracle_update(params, x, v, w, L, 1, 1e155, 1e155)
    assert not fatal and len(warn) > 0
    assert est.warnings == warn
    assert est.optimizer.t == t
    assert relL2(net.params64.cpu().numpy(), P) <= 1e-9
    assert relL2(est.optimizer.m.cpu().numpy(), m) <= 1e-4
    assert relL2(est.optimizer.v.cpu().numpy(), v2) <= 1e-4


def test_silu_fatal_divergence_matches_oracle(lib):
    """W2[0][0] = inf: every hidden unit of layer 2 sees inf * h1, the loss is non-finite, the
    update halves to the floor and raises; the parameters and t are untouched, and no later
    step of the update runs (the reference raises out of the loop)."""
    from paper_2603_25832_b200.silu_net import SiluEstimator

    net, params, p, (x, v, w, L) = _silu_setup(12)
    params[5 * 128] = np.inf
    net.set_flat(params)
    est = SiluEstimator(net, L, 3, np.random.default_rng(0), lr=1e-3, weight_decay=0.0)
    with pytest.raises(RuntimeError, match="training divergence"):
        est.update(p)
    P, m, v2, t, warn, losses, fatal = _oracle_update(params, x, v, w, L, 3, 1e-3, 0.0)
    assert fatal and len(warn) == 30
    assert est.warnings == warn
    assert est.optimizer.t == t == 0
    assert np.array_equal(net.params64.cpu().numpy(), params)


def test_score_test_blob_csv_matches_reference(lib, golden, tmp_path):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.run import score_test

    g = golden("score_test.npz")
    cfg = build_config(overrides=dict(preset="two_stream", n=4096, M=16, seed=3,
                                      estimator="blob"))
    rep = score_test(cfg, str(tmp_path), compute_force=True, estimators=("blob",))
    path = rep["blob"]["csv"]
    with open(path, encoding="utf-8") as fh:
        header = fh.readline().strip().split(",")
    data = np.loadtxt(path, delimiter=",", skiprows=1)
    assert header == [str(c) for c in g["columns"]]
    ref = g["data"]
    col = {c: i for i, c in enumerate(header)}

    def block(d, name):
        return d[:, [col[f"{name}{k}"] for k in (1, 2, 3)]]

    assert np.array_equal(data[:, 0], ref[:, 0].astype(np.float32).astype(np.float64))
    assert np.array_equal(block(data, "v"), block(ref, "v").astype(np.float32).astype(np.float64))
    for name in ("s_est", "U"):
        a, b = block(data, name), block(ref, name)
        assert relL2(a, b) <= 1e-4, (name, relL2(a, b))
        assert np.max(np.abs(a - b)) <= 1e-4 * np.max(np.abs(b)), name
    assert relL2(block(data, "s_true"), block(ref, "s_true")) <= 1e-5
    assert abs(rep["blob"]["mse"] - float(g["mse"])) <= 1e-4 * abs(float(g["mse"]))
