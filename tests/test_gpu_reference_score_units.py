"""The reference's score-estimator unit tests (ref: pkg/tests/test_score.py) restated against
this package's device API: softsign MLP forward, ISM loss, AdamW, pretraining, sbtm_update,
the blob KDE and the parameter layout. The network and optimizer state are float64 on the
device, the kernels read float32 parameters and particles, so per-value bounds are float32
rounding where the reference asserts 1e-12-1e-15; structural properties (identities, signs,
trends, thresholds) keep the reference's bounds.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_25832_b200 import _lib

    _lib.load()
    return _lib


def npy(t):
    return t.double().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t, float)


def random_net(dv, hidden, seed, scale=1.0):
    from paper_2603_25832_b200.score import MlpScoreNet
    from paper_2603_25832_b200.state import seeded_rng

    rng = seeded_rng(seed)
    net = MlpScoreNet.init_glorot(dv, hidden, rng)
    W1, W2 = net.numpy_params()[0] * scale, net.numpy_params()[2] * scale
    net.set_params([W1, rng.normal(size=hidden) * 0.1 * scale, W2,
                    rng.normal(size=dv) * 0.1 * scale])
    return net


def ens(x, v, w):
    from paper_2603_25832_b200.state import ParticleEnsemble

    return ParticleEnsemble.from_arrays(np.asarray(x, float), np.asarray(v, float),
                                        np.asarray(w, float))


# ------------------------------------------------------------------------------ forward
def test_mlp_forward_zero_constant_and_per_sample_loop(lib):
    from paper_2603_25832_b200.score import MlpScoreNet, mlp_forward
    from paper_2603_25832_b200.state import seeded_rng

    assert np.allclose(npy(mlp_forward(MlpScoreNet(3, 8), np.zeros(5), np.zeros((5, 3)))), 0.0)
    net = MlpScoreNet(2, 8)
    net.b2 = [1.5, -0.25]
    rng = seeded_rng(0)
    out = npy(mlp_forward(net, rng.random(7), rng.normal(size=(7, 2))))
    np.testing.assert_allclose(out, np.tile([1.5, -0.25], (7, 1)), rtol=1e-7)
    net = random_net(3, 16, seed=1)
    W1, b1, W2, b2 = (a.astype(np.float32).astype(np.float64) for a in net.numpy_params())
    rng = seeded_rng(2)
    x = rng.random(10).astype(np.float32).astype(np.float64)
    v = rng.normal(size=(10, 3)).astype(np.float32).astype(np.float64)
    got = npy(mlp_forward(net, x, v))
    for p in range(10):  # per-sample loop, no matrix algebra
        u = [x[p], *v[p]]
        hid = []
        for h in range(16):
            zz = b1[h] + sum(W1[h, m] * u[m] for m in range(4))
            hid.append(zz / (1.0 + abs(zz)))
        for i in range(3):
            ref = b2[i] + sum(W2[i, h] * hid[h] for h in range(16))
            assert got[p, i] == pytest.approx(ref, abs=2e-6)


# ---------------------------------------------------------------------------------- ISM
def test_ism_zero_network_loss_value_and_divergence_error(lib):
    from paper_2603_25832_b200.score import MlpScoreNet, ism_loss_and_grad
    from paper_2603_25832_b200.state import seeded_rng

    loss, grads = ism_loss_and_grad(MlpScoreNet(3, 8), np.zeros(4), np.ones((4, 3)),
                                    np.full(4, 0.25), divergence="exact")
    assert loss == 0.0 and all(np.allclose(npy(g), 0.0) for g in grads)
    # loss against the float64 oracle, exact and shared-probe Hutchinson
    net = random_net(3, 16, seed=11)
    rng = seeded_rng(12)
    x = rng.random(32).astype(np.float32).astype(np.float64)
    v = rng.normal(size=(32, 3)).astype(np.float32).astype(np.float64)
    w = np.full(32, 0.1)
    onet = O.Net(*[a.astype(np.float32).astype(np.float64) for a in net.numpy_params()])
    z = np.array([1.0, -1.0, 1.0])
    for mode, probe in (("exact", None), ("hutchinson", z)):
        loss, _ = ism_loss_and_grad(net, x, v, w, divergence=mode, z=probe)
        ref, _ = O.ism_loss_and_grad(onet, x, v, np.float32(0.1) * np.ones(32), divergence=mode,
                                     z=probe)
        assert loss == pytest.approx(ref, rel=1e-5)
    # a near-linear net emulating s(v) = -v: loss = sum w (|v|^2 - 2 dv) ~ -dv sum w
    dv, n, eps = 3, 20000, 1e-4
    net = MlpScoreNet(dv, dv)
    W1 = np.zeros((dv, 1 + dv))
    W1[:, 1:] = eps * np.eye(dv)
    net.W1 = W1
    net.W2 = -(1.0 / eps) * np.eye(dv)
    rng = seeded_rng(17)
    v = rng.normal(size=(n, dv))
    w = np.full(n, 1.0 / n)
    loss, _ = ism_loss_and_grad(net, rng.random(n), v, w, divergence="exact")
    ref = float(np.sum(w * (np.einsum("ij,ij->i", v, v) - 2.0 * dv)))
    assert loss == pytest.approx(ref, abs=5e-3) and loss == pytest.approx(-dv, abs=0.1)
    net = random_net(2, 8, seed=18)
    W2 = net.numpy_params()[2]
    W2[0, 0] = np.inf
    net.W2 = W2
    with pytest.raises(RuntimeError, match="training divergence"):
        ism_loss_and_grad(net, np.zeros(4), np.ones((4, 2)), np.full(4, 0.25), divergence="exact")


# ------------------------------------------------------------------------------- AdamW
def test_adamw_cases(lib):
    from paper_2603_25832_b200.score import AdamW, MlpScoreNet
    from paper_2603_25832_b200.state import seeded_rng

    proto = MlpScoreNet(2, 2)  # W1 (2 x 3), b1 (2), W2 (2 x 2), b2 (2): 14 parameters
    P = proto.n_params

    def net_with(vals):
        net = MlpScoreNet(2, 2)
        net.params64.copy_(torch.as_tensor(vals, dtype=torch.float64))
        net.refresh32()
        return net

    def split(flat):
        return [np.asarray(flat[a:b]).reshape(shape) for a, b, shape in proto._slices()]

    start = np.linspace(-2.0, 3.0, P)
    net = net_with(start)
    AdamW(lr=1e-3, weight_decay=0.0).step(net, split(np.zeros(P)))
    np.testing.assert_array_equal(npy(net.params64), start)
    g = np.resize([0.5, -0.5, 2.0, -2.0], P)
    net = net_with(np.zeros(P))
    AdamW(lr=1e-3, weight_decay=0.0).step(net, split(g))
    np.testing.assert_allclose(npy(net.params64), -1e-3 * np.sign(g), rtol=1e-6)
    rng = seeded_rng(19)
    grads = [rng.normal(size=P) for _ in range(10)]
    out = []
    for _ in range(2):
        net = net_with(np.ones(P))
        opt = AdamW(lr=1e-3, weight_decay=1e-2)
        for gg in grads:
            opt.step(net, split(gg))
        out.append(npy(net.params64))
    np.testing.assert_array_equal(out[0], out[1])
    net = net_with(np.ones(P))
    AdamW(lr=0.1, weight_decay=0.5).step(net, split(np.zeros(P)))
    np.testing.assert_allclose(npy(net.params64), 0.95, rtol=1e-15)


# --------------------------------------------------------------------- pretrain / SBTM
def test_pretrain_cases(lib):
    from paper_2603_25832_b200.score import MlpScoreNet, pretrain
    from paper_2603_25832_b200.state import seeded_rng

    def particles(n, dv, seed, L=4 * math.pi):
        rng = seeded_rng(seed)
        return ens(rng.uniform(0, L, n), rng.normal(size=(n, dv)), np.full(n, L / n)), rng

    p, rng = particles(512, 2, 20)
    net = MlpScoreNet.init_glorot(2, 16, rng)
    net.W2 = net.numpy_params()[2] * 0.01
    res = pretrain(net, p, lambda x, v: torch.zeros_like(v), L=4 * math.pi, rng=rng,
                   budget=2000, batch=256, tol=1e-6)
    assert res.converged and res.final_mse < 1e-6
    p, rng = particles(10000, 3, 21)
    net = MlpScoreNet.init_glorot(3, 256, rng)
    res = pretrain(net, p, lambda x, v: -v, L=4 * math.pi, rng=rng, budget=3000, batch=2048,
                   lr=1e-3)
    mean_s2 = float(np.mean(np.sum(npy(p.v) ** 2, axis=1)))
    assert res.final_mse / mean_s2 < 1e-2
    p, rng = particles(256, 2, 22)
    net = MlpScoreNet.init_glorot(2, 8, rng)
    res = pretrain(net, p, lambda x, v: -v, L=4 * math.pi, rng=rng, budget=3, batch=64)
    assert not res.converged and res.steps == 3


def test_sbtm_update_identity_and_loss_trend(lib):
    from paper_2603_25832_b200.score import AdamW, MlpScoreNet, sbtm_update
    from paper_2603_25832_b200.state import seeded_rng

    rng = seeded_rng(23)
    net = MlpScoreNet.init_glorot(2, 8, rng)
    before = npy(net.params64).copy()
    p = ens(rng.uniform(0, 1, 64), rng.normal(size=(64, 2)), np.full(64, 1.0 / 64))
    assert sbtm_update(net, AdamW(), p, 0, L=1.0, rng=rng) == []
    np.testing.assert_array_equal(npy(net.params64), before)
    rng = seeded_rng(24)
    net = MlpScoreNet.init_glorot(2, 32, rng)
    p = ens(rng.uniform(0, 2, 2000), rng.normal(size=(2000, 2)), np.full(2000, 2.0 / 2000))
    losses = sbtm_update(net, AdamW(lr=1e-3), p, 200, L=2.0, rng=rng)
    assert np.median(losses[-20:]) < np.median(losses[:20])


# -------------------------------------------------------------------------------- blob
def test_blob_cases(lib):
    from paper_2603_25832_b200.collision import build_cell_index
    from paper_2603_25832_b200.pic import Grid
    from paper_2603_25832_b200.score import BlobEstimator, blob_score, silverman_bandwidth
    from paper_2603_25832_b200.state import seeded_rng

    g = Grid(4, 1.0)
    p = ens([0.5], [[0.3, -0.7]], [1.0])
    np.testing.assert_allclose(npy(blob_score(p, build_cell_index(p, g), g, bandwidth=1.0)), 0.0,
                               atol=1e-7)
    a, h = 0.8, 0.6  # two co-located particles at +-a: -(2a/h^2) q/(1+q), q = exp(-2a^2/h^2)
    p = ens([0.5, 0.5], [[a, 0.0], [-a, 0.0]], [1.0, 1.0])
    s = npy(blob_score(p, build_cell_index(p, g), g, bandwidth=h))
    q = math.exp(-2.0 * a * a / (h * h))
    expected = -(2.0 * a / h ** 2) * q / (1.0 + q)
    assert s[0, 0] == pytest.approx(expected, rel=1e-5) and abs(s[0, 1]) <= 1e-7
    assert s[1, 0] == pytest.approx(-expected, rel=1e-5)
    rng = seeded_rng(25)  # Gaussian bulk MSE in one global cell
    n, L = 10000, 4.0
    g1 = Grid(1, L)
    p = ens(rng.uniform(0, L, n), rng.normal(size=(n, 3)), np.full(n, L / n))
    s = npy(blob_score(p, build_cell_index(p, g1), g1))
    v = npy(p.v)
    bulk = np.linalg.norm(v, axis=1) <= 2.0
    assert float(np.mean((s[bulk] + v[bulk]) ** 2)) < 0.05
    rng = seeded_rng(26)
    vv = rng.normal(size=(500, 3)) * 1.7
    sig = np.mean(np.std(vv, axis=0, ddof=1))
    assert silverman_bandwidth(vv) == pytest.approx(sig * (4.0 / (5 * 500)) ** (1.0 / 7), rel=1e-12)
    assert silverman_bandwidth(np.zeros((5, 2))) == 1.0
    rng = seeded_rng(27)
    g = Grid(8, 0.5)
    p = ens(rng.uniform(0, 4, 300), rng.normal(size=(300, 2)), np.full(300, 4.0 / 300))
    ci = build_cell_index(p, g)
    est = BlobEstimator(g)
    assert torch.equal(est.estimate(p, ci), blob_score(p, ci, g))
    est.update(p)


def test_network_parameter_count(lib):
    from paper_2603_25832_b200.score import MlpScoreNet

    for dv, hidden in ((2, 16), (3, 256), (3, 512)):
        assert MlpScoreNet(dv, hidden).n_params == (1 + dv) * hidden + hidden + hidden * dv + dv
