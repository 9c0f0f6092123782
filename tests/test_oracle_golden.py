"""Pin the float64 oracle (oracle/) against golden vectors produced by the reference itself
(tests/golden/make_golden.py). CPU only."""

import math

import numpy as np
import pytest

from oracle import oracle as O


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(1e-300, float(np.max(np.abs(b)))))


def test_binning_bit_exact(golden):
    g = golden("binning.npz")
    for k in range(int(g["ncases"])):
        x, M, eta = g[f"x_{k}"], int(g[f"M_{k}"]), float(g[f"eta_{k}"])
        assert np.array_equal(O.cell_of(x, eta, M), g[f"cell_{k}"])
        perm, starts = O.build_cell_index(x, eta, M)
        assert np.array_equal(perm, g[f"perm_{k}"]), k
        assert np.array_equal(starts, g[f"starts_{k}"]), k


def test_collision_matches_reference(golden):
    g = golden("collision.npz")
    for k in range(int(g["ncases"])):
        v = g[f"v_{k}"]
        U = O.collision_force(g[f"x_{k}"], v, g[f"w_{k}"], g[f"s_{k}"], float(g[f"eta_{k}"]),
                              int(g[f"M_{k}"]), -float(v.shape[1]))
        ref = g[f"U_{k}"]
        scale = max(1.0, float(np.max(np.abs(ref))))
        assert np.max(np.abs(U - ref)) <= 1e-12 * scale, k


def test_collision_nonfinite_score_rejected(golden):
    g = golden("collision.npz")
    s = g["s_0"].copy()
    s[3, 1] = np.nan
    with pytest.raises(ValueError, match="invalid score input"):
        O.collision_force(g["x_0"], g["v_0"], g["w_0"], s, float(g["eta_0"]), int(g["M_0"]), -3.0)


def test_blob_matches_reference(golden):
    g = golden("blob.npz")
    for k in range(int(g["ncases"])):
        bw = float(g[f"bw_{k}"])
        s = O.blob_score(g[f"x_{k}"], g[f"v_{k}"], g[f"w_{k}"], float(g[f"eta_{k}"]),
                         int(g[f"M_{k}"]), None if bw < 0 else bw)
        assert rel(s, g[f"s_{k}"]) <= 1e-11, k
    assert O.silverman_bandwidth(g["silver_v"]) == pytest.approx(float(g["silver_h"]), rel=1e-14)
    with pytest.raises(ValueError) as exc:
        O.blob_score(g["iso_x"], g["iso_v"], g["iso_w"], 1.0, 4, 0.05)
    assert str(exc.value) == str(g["iso_msg"])


def _net(g, prefix):
    return O.Net(g[prefix + "W1"].copy(), g[prefix + "b1"].copy(), g[prefix + "W2"].copy(),
                 g[prefix + "b2"].copy())


def test_mlp_and_ism_match_reference(golden):
    g = golden("mlp_ism.npz")
    for k in range(int(g["ncases"])):
        p = f"c{k}_"
        net = _net(g, p)
        x, v, w = g[p + "x"], g[p + "v"], g[p + "w"]
        assert rel(O.mlp_forward(net, x, v), g[p + "S"]) <= 1e-13
        for mode, probe in (("exact", None), ("shared", g[p + "zs"]), ("pp", g[p + "Zp"])):
            div = "exact" if mode == "exact" else "hutchinson"
            loss, grads = O.ism_loss_and_grad(net, x, v, w, divergence=div, z=probe)
            assert loss == pytest.approx(float(g[f"{p}{mode}_loss"]), rel=1e-11)
            for name, gr in zip(("gW1", "gb1", "gW2", "gb2"), grads):
                assert rel(gr, g[f"{p}{mode}_{name}"]) <= 1e-11, (k, mode, name)
        loss, grads = O.mse_loss_and_grad(net, x, v, w, -v)
        assert loss == pytest.approx(float(g[p + "mse_loss"]), rel=1e-12)
        for name, gr in zip(("gW1", "gb1", "gW2", "gb2"), grads):
            assert rel(gr, g[f"{p}mse_{name}"]) <= 1e-12


def test_adamw_and_sbtm_update_match_reference(golden):
    g = golden("adamw_sbtm.npz")
    for wd in (0.0, 1e-2):
        opt = O.AdamW(lr=1e-3, weight_decay=wd)
        p = [np.ones((3, 5))]
        for t, gr in enumerate(g["adam_grads"]):
            opt.step(p, [gr])
            assert np.array_equal(p[0], g[f"adam_wd{wd}_traj"][t])
    for tag, div in (("exact", "exact"), ("hutch", "hutchinson")):
        p = f"sbtm_{tag}_"
        net = _net(g, p + "init_")
        opt = O.AdamW(lr=1e-3, weight_decay=0.0)
        seed = int(g[p + "seed"])
        L = 4 * math.pi
        losses = O.sbtm_update(net, opt, g[p + "x"], g[p + "v"], g[p + "w"], 6, L=L,
                               rng=np.random.default_rng(seed + 1000), divergence=div)
        np.testing.assert_allclose(losses, g[p + "losses"], rtol=1e-10)
        S = O.mlp_forward(net, g[p + "x"] / L, g[p + "v"])
        assert rel(S, g[p + "S"]) <= 1e-8


def test_pic_matches_reference(golden):
    g = golden("pic.npz")
    for k in range(int(g["ncases"])):
        p = f"c{k}_"
        x, v, w = g[p + "x"], g[p + "v"], g[p + "w"]
        M, eta, dt = int(g[p + "M"]), float(g[p + "eta"]), float(g[p + "dt"])
        rho, J = O.deposit(x, v, w, eta, M)
        assert rel(rho, g[p + "rho"]) <= 1e-13 and rel(J, g[p + "J"]) <= 1e-13
        x1, v1 = O.push(x, v, g[p + "E1"], g[p + "E2"], g[p + "B3"], eta, M, dt)
        assert np.max(np.abs(x1 - g[p + "x1"])) <= 1e-12 * M * eta
        assert rel(v1, g[p + "v1"]) <= 1e-14
        E1, E2, B3 = O.maxwell_step(g[p + "E1"], g[p + "E2"], g[p + "B3"], g[p + "J"], eta, dt)
        for a, b in ((E1, "mE1"), (E2, "mE2"), (B3, "mB3")):
            assert rel(a, g[p + b]) <= 1e-14
        assert rel(O.vpl_field_step(g[p + "E1"], g[p + "J"], dt), g[p + "vE1"]) <= 1e-14
        d = O.diagnostics(g[p + "v1"], w, g[p + "mE1"], g[p + "mE2"], g[p + "mB3"], eta,
                          nu=0.1, U=g[p + "U"], s=g[p + "sc"])
        ref = g[p + "diag"]
        got = [d["E_K"], d["E_E"], d["E_B"], d["E_total"], d["H_dot"], d["E_l2"]]
        np.testing.assert_allclose(got, ref, rtol=1e-13)
        np.testing.assert_allclose(d["P"], g[p + "P"], rtol=1e-12, atol=1e-14)
    for j in range(int(g["npoisson"])):
        E1 = O.poisson_solve(g[f"poisson_rho_{j}"], float(g[f"poisson_ion_{j}"]),
                             float(g[f"poisson_eta_{j}"]))
        assert rel(E1, g[f"poisson_E1_{j}"]) <= 1e-13


def _oracle_run(x0, v0, *, L, M, dt, steps, mode, nu, estimator, alpha_B=0.0, k=1.0,
                bandwidth=None):
    eta = L / M
    n, dv = v0.shape
    w = np.full(n, L / n)
    rho, J = O.deposit(x0, v0, w, eta, M)
    rho_ion = float(rho.sum() * eta / L)
    E1, E2, B3 = np.zeros(M), np.zeros(M), np.zeros(M)
    if mode == "VML":
        B3 = alpha_B * np.sin(k * (np.arange(M) + 0.5) * eta)
    else:
        E1 = O.poisson_solve(rho, rho_ion, eta)
    state = dict(x=x0.copy(), v=v0.copy(), w=w, E1=E1, E2=E2, B3=B3)
    recs = [O.diagnostics(v0, w, E1, E2, B3, eta)]
    for _ in range(steps):
        recs.append(O.full_step(state, eta=eta, M=M, dt=dt, nu=nu, mode=mode, gamma=-dv,
                                net=None, opt=None, K=0, estimator=estimator,
                                bandwidth=bandwidth))
    return recs


@pytest.mark.parametrize("tag", ["vml", "blob"])
def test_oracle_full_steps_match_reference_run(golden, tag):
    g = golden("run.npz")
    if tag == "vml":
        kw = dict(L=10 * math.pi, M=16, dt=0.05, steps=5, mode="VML", nu=0.0, estimator="none",
                  alpha_B=1e-3, k=0.2)
    else:
        kw = dict(L=10 * math.pi, M=16, dt=0.05, steps=5, mode="VPL", nu=0.05, estimator="blob")
    recs = _oracle_run(g[f"{tag}_x0"], g[f"{tag}_v0"], **kw)
    ref = g[f"{tag}_diag"]
    got = np.array([[r["E_K"], r["E_E"], r["E_B"], r["E_total"], r["H_dot"], r["E_l2"]]
                    for r in recs])
    np.testing.assert_allclose(got, ref[:, [2, 3, 4, 5, 6, 7]], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(np.array([r["P"] for r in recs]), g[f"{tag}_P"], rtol=1e-9,
                               atol=1e-11)


def test_sbtm_recovery_paths_match_reference(golden):
    """sbtm_update's restore-and-halve recovery (ref: score.py:568-587; the construction of
    test_score.py:231-237): (A) a non-finite loss halves lr down to the 1e-12 floor and raises,
    parameters untouched, no optimizer step; (B) an AdamW step that overflows (lr * wd = inf)
    restores and halves until finite, m, v and t advancing on every attempt."""
    g = golden("faults.npz")
    x, v, w, L = g["fault_x"], g["fault_v"], g["fault_w"], 4 * math.pi
    net = _net(g, "faultA_init_")
    opt = O.AdamW(lr=1e-3, weight_decay=0.0)
    warn = []
    with pytest.raises(RuntimeError, match="training divergence"):
        O.sbtm_update(net, opt, x, v, w, 2, L=L, divergence="exact", warnings=warn)
    assert warn == list(g["faultA_warnings"])
    assert opt.lr == float(g["faultA_lr_after"]) and opt.t == int(g["faultA_t"])
    for a, b in zip(net.params(), _net(g, "faultA_final_").params()):
        assert np.array_equal(a, b)
    net = _net(g, "faultB_init_")
    opt = O.AdamW(lr=1e155, weight_decay=1e155)
    warn = []
    losses = O.sbtm_update(net, opt, x, v, w, 1, L=L, divergence="exact", warnings=warn)
    np.testing.assert_allclose(losses, g["faultB_losses"], rtol=1e-12)
    assert warn == list(g["faultB_warnings"])
    assert opt.lr == float(g["faultB_lr_after"]) and opt.t == int(g["faultB_t"])
    for a, b in zip(net.params(), _net(g, "faultB_final_").params()):
        assert rel(a, b) <= 1e-12
    for k in range(4):
        assert rel(opt.m[k], g[f"faultB_m{k}"]) <= 1e-10
        assert rel(opt.v[k], g[f"faultB_v{k}"]) <= 1e-10


def test_score_test_fixture_matches_oracle_blob(golden):
    """The reference's score_test blob CSV (ref: run.py:134-185): the oracle's blob scores and
    Landau U on the CSV's own x, v columns reproduce its s_est and U columns."""
    g = golden("score_test.npz")
    cols = [str(c) for c in g["columns"]]
    d = g["data"]
    col = {c: i for i, c in enumerate(cols)}
    x = d[:, col["x"]]
    v = d[:, [col["v1"], col["v2"], col["v3"]]]
    s = d[:, [col["s_est1"], col["s_est2"], col["s_est3"]]]
    U = d[:, [col["U1"], col["U2"], col["U3"]]]
    n, M, L = x.size, 16, 10 * math.pi
    eta = L / M
    w = np.full(n, L / n)
    assert rel(O.blob_score(x, v, w, eta, M), s) <= 1e-11
    assert rel(O.collision_force(x, v, w, s, eta, M, -3.0), U) <= 1e-11


def test_equilibrium_oracles_match_reference(golden):
    """The long-time equilibrium oracles the acceptance tests use (ref: equilibrium.py:24-55)."""
    g = golden("equilibrium.npz")
    for k in range(3):
        E0, rho, vol = g[f"vpl_in_{k}"]
        T, u = O.vpl_equilibrium(E0, g[f"vpl_P_{k}"], rho, vol)
        assert T == pytest.approx(float(g[f"vpl_T_{k}"]), rel=1e-14)
        np.testing.assert_allclose(u, g[f"vpl_u_{k}"], rtol=1e-14)
    for k in range(2):
        E0, vol = g[f"vml_in_{k}"]
        T, _ = O.vml_equilibrium(E0, g[f"vml_B_{k}"], 1.0, vol)
        assert T == pytest.approx(float(g[f"vml_T_{k}"]), rel=1e-14)
