"""Generate golden input/output vectors by running the REFERENCE itself.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/*.npz. All particle inputs are first rounded to float32 and then
upcast, so the same fixtures serve the float64 oracle (tight tolerances) and the float32
CUDA path (the tolerances stated in the GPU tests). Nothing here is imported at test time.
"""

import math
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from scorepic import collision, diagnostics, pic, run, score  # noqa: E402
from scorepic.config import build_config  # noqa: E402
from scorepic.equilibrium import analytic_initial_score  # noqa: E402
from scorepic.state import FieldState, ParticleEnsemble  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def ensemble(rng, n, dv, L, vscale=1.0):
    x = f32(rng.uniform(0, L, n))
    x = np.where(x >= L, 0.0, x)
    v = f32(rng.normal(size=(n, dv)) * vscale)
    w = np.full(n, L / n)
    return x, v, w


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def gen_binning():
    rng = np.random.default_rng(100)
    out = {}
    cases = []
    for n, M, L in [(1000, 13, 4 * math.pi), (5000, 64, 4 * math.pi), (777, 1, 3.0),
                    (500, 2, 5.0), (3000, 128, 10 * math.pi), (64, 8, 4.0)]:
        x = f32(rng.uniform(0, L, n))
        cases.append((x, M, L / M))
    # boundary floor convention (ref test_collision.py:30-36) and empty cells
    cases.append((np.array([0.5, 0.0, 0.49999997, 3.9999998]), 8, 0.5))
    # all particles in a single cell, other cells empty
    cases.append((np.full(100, f32(0.1)), 8, 0.5))
    # x just below L for an eta whose quotient rounds up to M (the % M quirk, pic.py:27-30)
    eta = 0.1
    M = 10
    xq = np.array([np.nextafter(M * eta, 0.0), 0.95, 0.05, 0.999999999999])
    cases.append((xq, M, eta))
    for k, (x, M, eta) in enumerate(cases):
        p = ParticleEnsemble(x=x, v=np.zeros((x.shape[0], 2)), w=np.ones(x.shape[0]))
        ci = collision.build_cell_index(p, pic.Grid(M, eta))
        out[f"x_{k}"] = x
        out[f"M_{k}"] = np.array(M)
        out[f"eta_{k}"] = np.array(eta)
        out[f"cell_{k}"] = pic.Grid(M, eta).cell_of(x)
        out[f"perm_{k}"] = np.concatenate(ci.bins).astype(np.int64)
        out[f"starts_{k}"] = np.concatenate(
            [[0], np.cumsum([b.size for b in ci.bins])]).astype(np.int64)
    out["ncases"] = np.array(len(cases))
    save("binning.npz", **out)


def gen_collision():
    rng = np.random.default_rng(101)
    out = {}
    cases = []
    for n, dv, M, L in [(300, 3, 8, 4 * math.pi), (200, 2, 5, 6.0), (150, 3, 1, 5.0),
                        (180, 3, 2, 5.0), (120, 2, 3, 4.0), (2000, 3, 16, 4 * math.pi)]:
        x, v, w = ensemble(rng, n, dv, L)
        s = f32(rng.normal(size=(n, dv)) * 2.0)
        cases.append((x, v, w, s, M, L / M))
    # config-1 shape: co-located particles, two-stream mixture velocities, exact score
    n = 512
    L = 2.0
    x = np.full(n, 1.0)
    v = f32(rng.normal(size=(n, 3)))
    v[:, 0] += np.where(rng.random(n) < 0.5, 1.5, -1.5)
    v = f32(v)
    s = f32(analytic_initial_score("two_stream", x, v, c=1.5))
    cases.append((x, v, np.full(n, L / n), s, 1, L))
    # two-particle hand example (ref test_collision.py:67-79)
    cases.append((np.array([0.5, 0.5]), np.array([[1.0, 0, 0], [0, 0, 0]]), np.ones(2),
                  np.array([[0, 1.0, 0], [0, 0, 0]]), 4, 1.0))
    for k, (x, v, w, s, M, eta) in enumerate(cases):
        p = ParticleEnsemble(x=x, v=v, w=w)
        grid = pic.Grid(M, eta)
        dv = v.shape[1]
        U = collision.collision_force(p, s, collision.build_cell_index(p, grid), grid,
                                      -float(dv))
        out.update({f"x_{k}": x, f"v_{k}": v, f"w_{k}": w, f"s_{k}": s, f"M_{k}": np.array(M),
                    f"eta_{k}": np.array(eta), f"U_{k}": U})
    out["ncases"] = np.array(len(cases))
    save("collision.npz", **out)


def gen_blob():
    rng = np.random.default_rng(102)
    out = {}
    cases = []
    for n, dv, M, L, bw in [(400, 3, 8, 4 * math.pi, None), (300, 2, 4, 4.0, None),
                            (500, 3, 1, 4.0, 0.4), (250, 3, 5, 5.0, 0.025),
                            (1500, 3, 16, 4 * math.pi, None)]:
        x, v, w = ensemble(rng, n, dv, L)
        cases.append((x, v, w, M, L / M, bw))
    a, h = 0.8, 0.6  # two-particle closed form (ref test_score.py:343-356)
    cases.append((np.array([0.5, 0.5]), np.array([[a, 0.0], [-a, 0.0]]), np.ones(2), 4, 1.0, h))
    for k, (x, v, w, M, eta, bw) in enumerate(cases):
        p = ParticleEnsemble(x=x, v=v, w=w)
        grid = pic.Grid(M, eta)
        s = score.blob_score(p, collision.build_cell_index(p, grid), grid, bw)
        out.update({f"x_{k}": x, f"v_{k}": v, f"w_{k}": w, f"M_{k}": np.array(M),
                    f"eta_{k}": np.array(eta), f"bw_{k}": np.array(-1.0 if bw is None else bw),
                    f"s_{k}": s})
    # isolated particle: tiny fixed bandwidth + far-apart velocities -> exp underflow
    x = np.array([0.2, 0.3, 2.5, 2.6])
    v = np.array([[0.0, 0.0, 0.0], [0.1, 0.0, 0.0], [0.0, 0.0, 0.0], [30.0, 0.0, 0.0]])
    iso_w = np.array([1.0, 1.0, 1.0, 0.0])  # zero self-weight -> den == 0 for particle 3
    p = ParticleEnsemble(x=x, v=v, w=iso_w)
    grid = pic.Grid(4, 1.0)
    try:
        score.blob_score(p, collision.build_cell_index(p, grid), grid, 0.05)
        msg = ""
    except ValueError as exc:
        msg = str(exc)
    out.update(iso_x=x, iso_v=v, iso_w=iso_w, iso_msg=np.array(msg))
    rs = np.random.default_rng(26)
    vv = rs.normal(size=(500, 3)) * 1.7
    out.update(silver_v=vv, silver_h=np.array(score.silverman_bandwidth(vv)))
    out["ncases"] = np.array(len(cases))
    save("blob.npz", **out)


def random_net(dv, H, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    net = score.MlpScoreNet.init_glorot(dv, H, rng)
    net.W1 *= scale
    net.W2 *= scale
    net.b1 = rng.normal(size=H) * 0.1 * scale
    net.b2 = rng.normal(size=dv) * 0.1 * scale
    return net


def net_arrays(prefix, net):
    return {f"{prefix}W1": net.W1.copy(), f"{prefix}b1": net.b1.copy(),
            f"{prefix}W2": net.W2.copy(), f"{prefix}b2": net.b2.copy()}


def gen_mlp_ism():
    rng = np.random.default_rng(103)
    out = {}
    k = 0
    for dv, H, n in [(3, 16, 64), (3, 128, 1000), (2, 24, 300), (3, 256, 500)]:
        net = random_net(dv, H, seed=200 + k)
        x = f32(rng.random(n))
        v = f32(rng.normal(size=(n, dv)))
        w = np.full(n, 4 * math.pi / n)
        zs = rng.integers(0, 2, size=dv).astype(np.float64) * 2.0 - 1.0
        Zp = rng.integers(0, 2, size=(n, dv)).astype(np.float64) * 2.0 - 1.0
        S = score.mlp_forward(net, x, v)
        out.update(net_arrays(f"c{k}_", net))
        out.update({f"c{k}_x": x, f"c{k}_v": v, f"c{k}_w": w, f"c{k}_S": S, f"c{k}_zs": zs,
                    f"c{k}_Zp": Zp})
        for mode, probe in (("exact", None), ("shared", zs), ("pp", Zp)):
            div = "exact" if mode == "exact" else "hutchinson"
            loss, grads = score.ism_loss_and_grad(net, x, v, w, divergence=div, z=probe)
            out[f"c{k}_{mode}_loss"] = np.array(loss)
            for name, g in zip(("gW1", "gb1", "gW2", "gb2"), grads):
                out[f"c{k}_{mode}_{name}"] = g
        target = -v
        loss, grads = score.mse_loss_and_grad(net, x, v, w, target)
        out[f"c{k}_mse_loss"] = np.array(loss)
        for name, g in zip(("gW1", "gb1", "gW2", "gb2"), grads):
            out[f"c{k}_mse_{name}"] = g
        k += 1
    out["ncases"] = np.array(k)
    save("mlp_ism.npz", **out)


def gen_adamw_sbtm():
    out = {}
    rng = np.random.default_rng(104)
    grads = [rng.normal(size=(3, 5)) for _ in range(6)]
    for wd in (0.0, 1e-2):
        opt = score.AdamW(lr=1e-3, weight_decay=wd)
        p = [np.ones((3, 5))]
        traj = []
        for g in grads:
            opt.step(p, [g])
            traj.append(p[0].copy())
        out[f"adam_wd{wd}_traj"] = np.array(traj)
    out["adam_grads"] = np.array(grads)
    # sbtm_update: K ISM steps on fixed particles (exact and shared-Hutchinson)
    for tag, div, seed in (("exact", "exact", 7), ("hutch", "hutchinson", 8)):
        prng = np.random.default_rng(300 + seed)
        n, dv, H, L = 2048, 3, 32, 4 * math.pi
        x = f32(prng.uniform(0, L, n))
        v = f32(prng.normal(size=(n, dv)))
        w = np.full(n, L / n)
        net = score.MlpScoreNet.init_glorot(dv, H, np.random.default_rng(seed))
        out.update(net_arrays(f"sbtm_{tag}_init_", net))
        opt = score.AdamW(lr=1e-3, weight_decay=0.0)
        p = ParticleEnsemble(x=x, v=v, w=w)
        losses = score.sbtm_update(net, opt, p, 6, L=L, rng=np.random.default_rng(seed + 1000),
                                   divergence=div, rademacher="shared")
        out.update(net_arrays(f"sbtm_{tag}_final_", net))
        out.update({f"sbtm_{tag}_x": x, f"sbtm_{tag}_v": v, f"sbtm_{tag}_w": w,
                    f"sbtm_{tag}_losses": np.array(losses), f"sbtm_{tag}_seed": np.array(seed),
                    f"sbtm_{tag}_S": score.mlp_forward(net, x / L, v)})
    save("adamw_sbtm.npz", **out)


def gen_pic():
    rng = np.random.default_rng(105)
    out = {}
    k = 0
    for n, dv, M, L in [(500, 3, 16, 4 * math.pi), (300, 2, 7, 5.0), (400, 3, 1, 3.0),
                        (1000, 3, 64, 2 * math.pi / 1.25)]:
        x, v, w = ensemble(rng, n, dv, L, vscale=2.0)
        grid = pic.Grid(M, L / M)
        p = ParticleEnsemble(x=x.copy(), v=v.copy(), w=w)
        rho, J = pic.deposit(p, grid)
        fields = FieldState.zeros(M, dv)
        fields.E1 = rng.normal(size=M) * 0.3
        fields.E2 = rng.normal(size=M) * 0.3
        fields.B3 = rng.normal(size=M) * 0.3
        E1, E2, B3 = fields.E1.copy(), fields.E2.copy(), fields.B3.copy()
        E_p, B_p = pic.interpolate_fields(p, fields, grid)
        dt = 0.05
        pic.lorentz_push(p, E_p, B_p, dt)
        pic.advance_positions(p, dt, grid.L)
        fm = FieldState(E1=E1.copy(), E2=E2.copy(), B3=B3.copy(), rho=rho, J=J, rho_ion=0.0)
        pic.maxwell_step(fm, J, dt, grid)
        fv = FieldState(E1=E1.copy(), E2=E2.copy(), B3=B3.copy(), rho=rho, J=J, rho_ion=0.0)
        pic.vpl_field_step(fv, J, dt)
        rng_s = np.random.default_rng(400 + k)
        U = rng_s.normal(size=(n, dv))
        sc = rng_s.normal(size=(n, dv))
        rec = diagnostics.compute_diagnostics(p, fm, grid.eta, step=1, t=dt, nu=0.1, U=U,
                                              scores=sc)
        out.update({f"c{k}_x": x, f"c{k}_v": v, f"c{k}_w": w, f"c{k}_M": np.array(M),
                    f"c{k}_eta": np.array(L / M), f"c{k}_dt": np.array(dt),
                    f"c{k}_rho": rho, f"c{k}_J": J, f"c{k}_E1": E1, f"c{k}_E2": E2,
                    f"c{k}_B3": B3, f"c{k}_x1": p.x, f"c{k}_v1": p.v,
                    f"c{k}_mE1": fm.E1, f"c{k}_mE2": fm.E2, f"c{k}_mB3": fm.B3,
                    f"c{k}_vE1": fv.E1, f"c{k}_U": U, f"c{k}_sc": sc,
                    f"c{k}_diag": np.array([rec.E_K, rec.E_E, rec.E_B, rec.E_total, rec.H_dot,
                                            rec.E_l2]), f"c{k}_P": rec.P})
        k += 1
    out["ncases"] = np.array(k)
    # Poisson (ref: pic.py:118-134)
    for j, (M, L, a, kk) in enumerate([(100, 4 * math.pi, 0.1, 0.5), (64, 10 * math.pi, 0.001, 0.2),
                                       (33, 2 * math.pi, 0.05, 3.0)]):
        grid = pic.Grid(M, L / M)
        rho = 1.0 + a * np.cos(kk * grid.centers) + 0.01 * np.random.default_rng(j).normal(size=M)
        rho_ion = float(rho.sum() * grid.eta / grid.L)
        out[f"poisson_rho_{j}"] = rho
        out[f"poisson_ion_{j}"] = np.array(rho_ion)
        out[f"poisson_eta_{j}"] = np.array(grid.eta)
        out[f"poisson_E1_{j}"] = pic.poisson_solve(rho, rho_ion, grid)
    out["npoisson"] = np.array(3)
    save("pic.npz", **out)


def gen_run():
    """Short end-to-end runs through run.run (the solver entry point)."""
    out = {}
    configs = {
        "sbtm": dict(preset="landau_damping", n=4096, M=16, dt=0.05, t_final=0.25, nu=0.1,
                     K=3, hidden=16, lr=1e-3, weight_decay=0.0, divergence="exact",
                     pretrain_budget=40, pretrain_batch=512, alpha=0.1, seed=3),
        "blob": dict(preset="two_stream", n=4096, M=16, dt=0.05, t_final=0.25, nu=0.05,
                     estimator="blob", bandwidth="silverman", alpha=0.01, seed=4),
        "vml": dict(preset="weibel", n=4096, M=16, dt=0.05, t_final=0.25, nu=0.0,
                    estimator="none", seed=5),
    }
    for tag, ov in configs.items():
        cfg = build_config(overrides=ov)
        with tempfile.TemporaryDirectory() as d:
            recs = run.run(cfg, d)
            P0 = diagnostics.read_snapshot(os.path.join(d, "snapshot_000000.bin"))[0]
        out[f"{tag}_diag"] = np.array([[r.step, r.t, r.E_K, r.E_E, r.E_B, r.E_total, r.H_dot,
                                        r.E_l2] for r in recs])
        out[f"{tag}_P"] = np.array([r.P for r in recs])
        out[f"{tag}_x0"] = P0.x
        out[f"{tag}_v0"] = P0.v
    save("run.npz", **out)


def gen_faults():
    """sbtm_update's restore-and-halve recovery (ref: score.py:568-587): (A) a non-finite loss
    (W2[0,0] = inf, the reference test_score.py:231-237 construction) halves the learning rate
    down to the 1e-12 floor and raises "training divergence"; (B) a finite loss whose AdamW step
    overflows (lr * weight_decay = inf) restores the parameters and halves until the step is
    finite, with m, v and t advancing on every attempt."""
    out = {}
    n, dv, H, L = 512, 3, 16, 4 * math.pi
    prng = np.random.default_rng(400)
    x = f32(prng.uniform(0, L, n))
    v = f32(prng.normal(size=(n, dv)))
    w = np.full(n, L / n)
    p = ParticleEnsemble(x=x, v=v, w=w)
    out.update(fault_x=x, fault_v=v, fault_w=w)
    # (A) fatal
    net = score.MlpScoreNet.init_glorot(dv, H, np.random.default_rng(41))
    net.W2[0, 0] = np.inf
    out.update(net_arrays("faultA_init_", net))
    opt = score.AdamW(lr=1e-3, weight_decay=0.0)
    warn = []
    try:
        score.sbtm_update(net, opt, p, 2, L=L, rng=np.random.default_rng(1),
                          divergence="exact", warnings=warn)
        raise AssertionError("expected training divergence")
    except RuntimeError as exc:
        assert "training divergence" in str(exc)
    out.update(net_arrays("faultA_final_", net))
    out["faultA_warnings"] = np.array(warn)
    out["faultA_lr_after"] = np.array(opt.lr)
    out["faultA_t"] = np.array(opt.t)
    # (B) recovery
    net = score.MlpScoreNet.init_glorot(dv, H, np.random.default_rng(42))
    out.update(net_arrays("faultB_init_", net))
    opt = score.AdamW(lr=1e155, weight_decay=1e155)
    warn = []
    losses = score.sbtm_update(net, opt, p, 1, L=L, rng=np.random.default_rng(1),
                               divergence="exact", warnings=warn)
    out.update(net_arrays("faultB_final_", net))
    out["faultB_losses"] = np.array(losses)
    out["faultB_warnings"] = np.array(warn)
    out["faultB_lr_after"] = np.array(opt.lr)
    out["faultB_t"] = np.array(opt.t)
    for k, (m_, v_) in enumerate(zip(opt.m, opt.v)):
        out[f"faultB_m{k}"] = m_
        out[f"faultB_v{k}"] = v_
    save("faults.npz", **out)


def gen_score_test():
    """run.score_test (ref: run.py:134-185) with the blob estimator (deterministic): the
    reference's CSV columns x, v*, s_est*, s_true*, U* and its reported MSE."""
    cfg = build_config(overrides=dict(preset="two_stream", n=4096, M=16, seed=3,
                                      estimator="blob"))
    with tempfile.TemporaryDirectory() as d:
        rep = run.score_test(cfg, d, compute_force=True, estimators=("blob",))
        path = os.path.join(d, "score_test_blob.csv")
        with open(path, encoding="utf-8") as fh:
            header = fh.readline().strip().split(",")
        data = np.loadtxt(path, delimiter=",", skiprows=1)
    save("score_test.npz", columns=np.array(header), data=data,
         mse=np.array(rep["blob"]["mse"]))


def gen_equilibrium():
    """Long-time equilibrium oracles (ref: equilibrium.py:24-55) on a few inputs."""
    from scorepic.equilibrium import vml_equilibrium, vpl_equilibrium

    out = {}
    cases = [(12.3, [0.1, -0.02], 1.0, 4 * math.pi), (7.5, [0.0, 0.0, 0.3], 1.0, 2 * math.pi),
             (0.9, [0.01, 0.02, 0.0], 0.5, 5.0)]
    for k, (E0, P0, rho, vol) in enumerate(cases):
        eq = vpl_equilibrium(E0, np.array(P0), rho, vol)
        out[f"vpl_in_{k}"] = np.array([E0, rho, vol])
        out[f"vpl_P_{k}"] = np.array(P0)
        out[f"vpl_T_{k}"] = np.array(eq.T_inf)
        out[f"vpl_u_{k}"] = eq.u_inf
    for k, (E0, B, vol) in enumerate([(3.0, [0.0, 0.0, 0.2], 2 * math.pi),
                                      (1.5, [0.1, 0.0, 0.05], 5.0)]):
        eq = vml_equilibrium(E0, np.array(B), 1.0, vol)
        out[f"vml_in_{k}"] = np.array([E0, vol])
        out[f"vml_B_{k}"] = np.array(B)
        out[f"vml_T_{k}"] = np.array(eq.T_inf)
    save("equilibrium.npz", **out)


if __name__ == "__main__":
    gen_binning()
    gen_collision()
    gen_blob()
    gen_mlp_ism()
    gen_adamw_sbtm()
    gen_pic()
    gen_run()
    gen_faults()
    gen_score_test()
    gen_equilibrium()
