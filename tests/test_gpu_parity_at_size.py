"""GPU parity at the sizes the bench reports (BASELINE configs 1-4), per particle, against the
float64 oracle (oracle/, pinned to the reference by tests/test_oracle_golden.py).

Tolerances (float32 product vs float64 reference):
  * collision velocities U: relative L2 <= 1e-4 and per particle |err| <= 1e-4 * max|U_ref|
    over every target of the sampled cells (the oracle evaluates every `stride`-th cell in
    full: all targets of the cell against its whole 3-cell stencil,
    ref: collision.py:49-110);
  * SiLU ISM loss <= 1e-4 relative and gradients <= 1e-4 relative L2 per parameter tensor
    (split-BF16 tensor-core products, see tests/test_gpu_silu.py);
  * 100 full config-0 steps (softsign SBTM net, the reference's network) against
    oracle.full_step on the same float32 initial state: conservation and field-energy traces
    within the bands stated in test_config0_100_steps_traces_match_oracle.
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


def relL2(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def bench_ensemble(tag: str, seed: int = 0):
    """The bench's own initial ensemble of BASELINE config `tag` (seeded reference sampler /
    config-3 anisotropic sampler), rounded to float32 once."""
    import bench

    wl = bench.WORKLOADS[tag]
    cfg = bench.make_config(wl, seed)
    x, v, w, _ = bench.sample_workload(wl, cfg, np.random.default_rng(seed))
    return f32(x), f32(v), f32(w), wl


def sampled_cell_mask(x, eta, M, stride):
    cell = O.cell_of(x, eta, M)
    return (cell % stride) == 0


@pytest.mark.parametrize("tag,stride", [("c2", 8), ("c3", 16), ("c4", 64)])
def test_collision_per_particle_at_bench_size(lib, tag, stride):
    """Configs 2 (n = 2^20, M = 128), 3 (n = 2^22, M = 256, Weibel velocities) and 4
    (n = 2^24, M = 1024): U from the device path the engine runs (antisymmetric pair kernel,
    sub-cell culling, cell-sorted records) against the oracle on every `stride`-th cell.
    Scores are non-Maxwellian so U is O(1): config 2 the exact two-stream mixture score,
    config 3 the anisotropic Maxwellian's exact score -v_k / T_k, config 4 -v plus a smooth
    perturbation."""
    from paper_2603_25832_b200.collision import auto_sub_cells, build_cell_index, collision_force
    from paper_2603_25832_b200.pic import Grid
    from paper_2603_25832_b200.state import ParticleEnsemble

    x, v, w, wl = bench_ensemble(tag)
    n, M, L = wl["n"], wl["M"], wl["L"]
    if tag == "c2":
        s = -v.copy()
        s[:, 0] = -v[:, 0] + wl["c"] * np.tanh(wl["c"] * v[:, 0])
    elif tag == "c3":
        s = -v / np.asarray(wl["temps"])[None, :]
    else:
        s = -v + 0.5 * np.sin(2.0 * v[:, [1, 2, 0]])
    s = f32(s)
    grid = Grid(M, L / M)
    p = ParticleEnsemble.from_arrays(x, v, w)
    ci = build_cell_index(p, grid, auto_sub_cells(n, M))
    U = collision_force(p, s, ci, grid, -3.0).double().cpu().numpy()
    ref = O.collision_force(x, v, p.w.double().cpu().numpy(), s, grid.eta, M, -3.0,
                            cell_stride=stride)
    mask = sampled_cell_mask(x, grid.eta, M, stride)
    assert mask.sum() > n // (2 * stride)
    got, want = U[mask], ref[mask]
    err = relL2(got, want)
    worst = float(np.max(np.abs(got - want)) / np.max(np.abs(want)))
    print(f"{tag}: {int(mask.sum())} targets, relL2 {err:.2e}, worst/max {worst:.2e}")
    assert err <= 1e-4, err
    assert worst <= 1e-4, worst
    assert np.all(np.isfinite(U))


def test_config1_n131072_per_particle(lib):
    """BASELINE config 1 at its largest n = 131 072: one cell, co-located x, two-stream
    mixture velocities with the exact mixture score; all n^2 ordered pairs live. Every
    particle against the oracle, plus momentum / energy conservation <= 1e-5 (A1 metric,
    ref: tests/test_acceptance.py:62-77)."""
    from paper_2603_25832_b200.collision import build_cell_index, collision_force
    from paper_2603_25832_b200.pic import Grid
    from paper_2603_25832_b200.state import ParticleEnsemble

    n, L = 131072, 2.0
    rng = np.random.default_rng(1)
    v = rng.normal(size=(n, 3))
    v[:, 0] += np.where(rng.random(n) < 0.5, 1.5, -1.5)
    v = f32(v)
    s = -v.copy()
    s[:, 0] = -v[:, 0] + 1.5 * np.tanh(1.5 * v[:, 0])
    s = f32(s)
    x = np.full(n, 1.0)
    p = ParticleEnsemble.from_arrays(x, v, np.full(n, L / n))
    grid = Grid(1, L)
    U = collision_force(p, s, build_cell_index(p, grid), grid, -3.0).double().cpu().numpy()
    w64 = p.w.double().cpu().numpy()
    ref = O.collision_force(x, v, w64, s, L, 1, -3.0)
    err = relL2(U, ref)
    worst = float(np.max(np.abs(U - ref)) / np.max(np.abs(ref)))
    print(f"config1 n=131072: relL2 {err:.2e}, worst/max {worst:.2e}")
    assert err <= 1e-4 and worst <= 1e-4, (err, worst)
    wU = w64[:, None] * U
    mom = np.max(np.abs(wU.sum(0))) / (np.max(np.abs(wU)) * n)
    en = abs(float(np.sum(w64 * np.einsum("ij,ij->i", v, U))))
    en /= float(np.sum(w64 * np.linalg.norm(v, axis=1) * np.linalg.norm(U, axis=1)))
    assert mom <= 1e-5 and en <= 1e-5, (mom, en)


def _silu_oracle_chunked(params, x, v, w, L, chunk=1 << 17):
    """Float64 ISM loss and gradient of the SiLU net summed over particle chunks (the loss
    and every gradient are sums over particles)."""
    from oracle import silu_oracle as so

    loss, grad = 0.0, None
    for a in range(0, x.shape[0], chunk):
        b = min(a + chunk, x.shape[0])
        l, g = so.ism_loss_and_grad(params, so.inputs(x[a:b], v[a:b], L), w[a:b], 128)
        loss += l
        grad = g if grad is None else grad + g
    return loss, grad


@pytest.mark.parametrize("tag", ["c2", "c3", "c4"])
def test_silu_ism_at_bench_size(lib, tag):
    """The SiLU ISM kernel at the bench's own sizes (config 2: n = 2^20 two-stream; config 3:
    n = 2^22 Weibel velocities; config 4, the headline: n = 2^24): one persistent CTA per SM
    accumulates ~150 (2^20) to ~2400 (2^24) 48-particle chunks (float32 TMEM accumulators
    flushed to a float32 buffer every 64 chunks) before its float64 partial row; loss and
    every gradient tensor against the float64 oracle."""
    from oracle import silu_oracle as so
    from paper_2603_25832_b200.silu_net import SiluScoreNet, silu_ism_loss_and_grad

    x, v, w, wl = bench_ensemble(tag)
    L = wl["L"]
    rng = np.random.default_rng(5)
    params = so.glorot(128, rng)
    params[4 * 128:5 * 128] = rng.normal(0, 0.3, 128)
    params[-3:] = rng.normal(0, 0.3, 3)
    params = f32(params)
    net = SiluScoreNet()
    net.set_flat(params)
    loss, g = silu_ism_loss_and_grad(net, x, v, w, L)
    g = g.cpu().numpy()
    ref_loss, ref_g = _silu_oracle_chunked(params, x, v, w, L)
    print(f"{tag}: loss {loss:.8e} vs {ref_loss:.8e}")
    assert abs(loss - ref_loss) <= 1e-4 * abs(ref_loss), (loss, ref_loss)
    for (a, b, _), name in zip(net._slices(), ("W1", "b1", "W2", "b2", "W3", "b3")):
        e = relL2(g[a:b], ref_g[a:b])
        print(f"  {name}: relL2 {e:.2e}")
        assert e <= 1e-4, (name, e)


def test_config0_100_steps_traces_match_oracle(lib):
    """BASELINE config 0 (Landau damping, n = 65 536, M = 64, L = 4 pi, nu = 0.1, dt = 0.05,
    K = 10 exact-divergence ISM steps, H = 128 softsign net — the reference's network —, Adam
    lr 1e-3, no pretraining) for 100 steps on the device engine and in oracle.full_step from
    the same float32 initial state and the same initial network. Particle trajectories are
    chaotic in the float32 / float64 difference, so the run is compared
    through conservation and traces:
      * energy drift |E_tot(t) / E_tot(0) - 1| of the device run <= 1e-4 at every step, and
        within 1e-7 of the oracle's drift (measured: drift 5.2e-5 on both, difference 2.8e-9);
      * field-energy traces: max_t |E_E - E_E_ref| <= 1e-3 * max_t E_E_ref, same for E_l2
        (measured 2.7e-5 and 2.6e-5);
      * momentum: the P trace (P_x changes through the field force) within 1e-4 * sum w|v| of
        the oracle's, P_y and P_z (no force, Landau conserves momentum) constant to 1e-6;
      * entropy production H_dot (depends on the trained net): trace within 5e-2 of the
        oracle's (measured minima 5.760e-3 vs 5.741e-3).
    Measured values are printed (DESIGN.md section 5 records them)."""
    import bench
    from paper_2603_25832_b200.engine import Simulation
    from paper_2603_25832_b200.pic import Grid, deposit, poisson_solve
    from paper_2603_25832_b200.score import MlpScoreNet, SbtmEstimator
    from paper_2603_25832_b200.state import FieldState, ParticleEnsemble

    steps, dt, nu, K = 100, 0.05, 0.1, 10
    wl = bench.WORKLOADS["c0ss"]
    cfg = bench.make_config(wl, 0)
    rng = np.random.default_rng(0)
    x, v, w, _ = bench.sample_workload(wl, cfg, rng)
    x, v = f32(x), f32(v)
    n, M, L = wl["n"], wl["M"], wl["L"]
    grid = Grid(M, L / M)
    p = ParticleEnsemble.from_arrays(x, v, w)
    w64 = p.w.double().cpu().numpy()
    rho, _ = deposit(p, grid)
    rho_ion = float(rho.sum()) * grid.eta / L
    f = FieldState.zeros(M, 3, rho_ion)
    f.E1.copy_(poisson_solve(rho, rho_ion, grid))
    E1_0 = f.E1.cpu().numpy().copy()
    net = MlpScoreNet.init_glorot(3, 128, rng)
    onet = O.Net(*[a.cpu().numpy().astype(np.float64).copy() for a in net.params()])
    est = SbtmEstimator(net, L, K, rng, lr=1e-3, weight_decay=0.0, divergence="exact")
    sim = Simulation(p, f, grid, dt=dt, nu=nu, mode="VPL", gamma=-3.0, estimator=est,
                     max_rows=steps + 1)
    for k in range(1, steps + 1):
        sim.step(k)
    sim.check()
    got = sim.records(range(1, steps + 1), range(1, steps + 1), [dt * k for k in range(1, steps + 1)])

    st = dict(x=x.copy(), v=v.copy(), w=w64, E1=E1_0.copy(), E2=np.zeros(M), B3=np.zeros(M))
    d0 = O.diagnostics(v, w64, E1_0, np.zeros(M), np.zeros(M), grid.eta)
    opt = O.AdamW(lr=1e-3, weight_decay=0.0)
    ref = [O.full_step(st, eta=grid.eta, M=M, dt=dt, nu=nu, mode="VPL", gamma=-3.0, net=onet,
                       opt=opt, K=K, divergence="exact") for _ in range(steps)]

    E0 = d0["E_total"]
    drift_g = np.array([r.E_total / E0 - 1.0 for r in got])
    drift_r = np.array([r["E_total"] / E0 - 1.0 for r in ref])
    EE_g, EE_r = np.array([r.E_E for r in got]), np.array([r["E_E"] for r in ref])
    El_g, El_r = np.array([r.E_l2 for r in got]), np.array([r["E_l2"] for r in ref])
    P_g, P_r = np.array([r.P for r in got]), np.array([r["P"] for r in ref])
    HD_g, HD_r = np.array([r.H_dot for r in got]), np.array([r["H_dot"] for r in ref])
    pscale = float(np.sum(w64 * np.linalg.norm(v, axis=1)))
    ee = float(np.max(np.abs(EE_g - EE_r)) / np.max(EE_r))
    el = float(np.max(np.abs(El_g - El_r)) / np.max(El_r))
    P0 = w64 @ v
    pt = float(np.max(np.abs(P_g - P_r)) / pscale)
    pyz = float(np.max(np.abs(P_g[:, 1:] - P0[None, 1:])) / pscale)
    hd = float(np.max(np.abs(HD_g - HD_r)) / np.max(np.abs(HD_r)))
    print(f"config0 100 steps: max drift device {np.max(np.abs(drift_g)):.3e}, oracle "
          f"{np.max(np.abs(drift_r)):.3e}, max |drift diff| {np.max(np.abs(drift_g - drift_r)):.3e}; "
          f"E_E trace {ee:.3e}, E_l2 trace {el:.3e}; P trace {pt:.3e}, P_yz drift {pyz:.3e}; "
          f"H_dot trace {hd:.3e}; E_E(1..100) device {EE_g[0]:.4e}..{EE_g[-1]:.4e} oracle "
          f"{EE_r[0]:.4e}..{EE_r[-1]:.4e}")
    assert np.max(np.abs(drift_g)) <= 1e-4
    assert np.max(np.abs(drift_g - drift_r)) <= 1e-7
    assert ee <= 1e-3 and el <= 1e-3, (ee, el)
    assert pt <= 1e-4 and pyz <= 1e-6, (pt, pyz)
    assert hd <= 5e-2, hd


def test_config3_weibel_200_steps_traces_match_oracle(lib):
    """BASELINE config 3's physics (Weibel, full Maxwell VML: anisotropic Maxwellian
    T = (0.01, 0.04, 0.04), seeded B_z noise 1e-4, M = 256, L = 2 pi / 1.25, nu = 0.01,
    dt = 0.02) at n = 2^16 with the reference's softsign net (H = 128, K = 10 exact ISM
    steps), 200 steps (t = 4, the linear growth of E_B) on the device engine and in
    oracle.full_step from the same float32 initial state and network:
      * energy: |E_tot(t) / E_tot(0) - 1| of the device run within 1e-6 of the oracle's at
        every step (the VML scheme's own drift is shared, float32 adds the rest);
      * E_B trace (the Weibel growth): max_t |E_B - E_B_ref| <= 1e-2 * max_t E_B_ref, and
        the growth factor E_B(end) / E_B(0) within 5% of the oracle's;
      * momentum: P_z (no force in this 1D3V geometry) constant to 1e-6 of sum w|v|.
    Measured values are printed (DESIGN.md section 5 records them)."""
    import bench
    from paper_2603_25832_b200.engine import Simulation
    from paper_2603_25832_b200.pic import Grid
    from paper_2603_25832_b200.run import initial_fields
    from paper_2603_25832_b200.score import MlpScoreNet, SbtmEstimator
    from paper_2603_25832_b200.state import ParticleEnsemble

    steps, K = 200, 10
    wl = dict(bench.WORKLOADS["c3ss"], n=1 << 16)
    cfg = bench.make_config(wl, 0)
    rng = np.random.default_rng(0)
    x, v, w, b3 = bench.sample_workload(wl, cfg, rng)
    x, v = f32(x), f32(v)
    n, M, L, dt, nu = wl["n"], wl["M"], wl["L"], wl["dt"], wl["nu"]
    grid = Grid(M, L / M)
    p = ParticleEnsemble.from_arrays(x, v, w)
    w64 = p.w.double().cpu().numpy()
    from paper_2603_25832_b200.pic import deposit

    rho, J = deposit(p, grid)
    f = initial_fields(cfg, grid, rho, J)
    f.B3.copy_(torch.as_tensor(b3, dtype=torch.float64))
    B3_0 = f.B3.cpu().numpy().copy()
    net = MlpScoreNet.init_glorot(3, 128, rng)
    onet = O.Net(*[a.cpu().numpy().astype(np.float64).copy() for a in net.params()])
    est = SbtmEstimator(net, L, K, rng, lr=1e-3, weight_decay=0.0, divergence="exact")
    sim = Simulation(p, f, grid, dt=dt, nu=nu, mode="VML", gamma=-3.0, estimator=est,
                     max_rows=steps + 1)
    for k in range(1, steps + 1):
        sim.step(k)
    sim.check()
    got = sim.records(range(1, steps + 1), range(1, steps + 1), [dt * k for k in range(1, steps + 1)])

    st = dict(x=x.copy(), v=v.copy(), w=w64, E1=np.zeros(M), E2=np.zeros(M), B3=B3_0.copy())
    d0 = O.diagnostics(v, w64, np.zeros(M), np.zeros(M), B3_0, grid.eta)
    opt = O.AdamW(lr=1e-3, weight_decay=0.0)
    ref = [O.full_step(st, eta=grid.eta, M=M, dt=dt, nu=nu, mode="VML", gamma=-3.0, net=onet,
                       opt=opt, K=K, divergence="exact") for _ in range(steps)]
    E0 = d0["E_total"]
    drift_g = np.array([r.E_total / E0 - 1.0 for r in got])
    drift_r = np.array([r["E_total"] / E0 - 1.0 for r in ref])
    EB_g, EB_r = np.array([r.E_B for r in got]), np.array([r["E_B"] for r in ref])
    P_g = np.array([r.P for r in got])
    pscale = float(np.sum(w64 * np.linalg.norm(v, axis=1)))
    P0 = w64 @ v
    eb = float(np.max(np.abs(EB_g - EB_r)) / np.max(EB_r))
    growth_g, growth_r = EB_g[-1] / d0["E_B"], EB_r[-1] / d0["E_B"]
    pz = float(np.max(np.abs(P_g[:, 2] - P0[2])) / pscale)
    print(f"config3 (n = 2^16) 200 VML steps: max drift device {np.max(np.abs(drift_g)):.3e}, "
          f"oracle {np.max(np.abs(drift_r)):.3e}, max |diff| {np.max(np.abs(drift_g - drift_r)):.3e}; "
          f"E_B trace {eb:.3e}, growth {growth_g:.3f} vs {growth_r:.3f}; P_z drift {pz:.3e}")
    assert np.max(np.abs(drift_g - drift_r)) <= 1e-6
    assert eb <= 1e-2
    assert abs(growth_g / growth_r - 1.0) <= 0.05
    assert pz <= 1e-6


def test_dv2_relaxation_50_steps_traces_match_oracle(lib):
    """The reduced-dimension path (dv = 2: the scalar pair kernel with gamma = -2, 2-component
    push / deposit / ISM) over 50 strongly collisional steps (VPL Landau damping, n = 16 384,
    M = 32, nu = 1, dt = 0.02 — the reference's A6 setting at a smaller n — softsign net H = 64,
    K = 10 exact ISM steps) on the device engine and in oracle.full_step from the same float32
    initial state and network: energy drift within 1e-6 of the oracle's at every step, the
    E_E trace within 1e-3 of its maximum, P_y constant to 1e-6 of sum w|v|, and the H_dot
    trace within 5e-2 of the oracle's."""
    from paper_2603_25832_b200.engine import Simulation
    from paper_2603_25832_b200.pic import Grid, deposit, poisson_solve
    from paper_2603_25832_b200.score import MlpScoreNet, SbtmEstimator
    from paper_2603_25832_b200.state import FieldState, ParticleEnsemble

    steps, dt, nu, K, n, M = 50, 0.02, 1.0, 10, 16384, 32
    L = 4 * math.pi
    rng = np.random.default_rng(7)
    x = f32(rng.uniform(0, L, n))
    x[x >= L] = 0.0
    v = f32(rng.normal(size=(n, 2)))
    w = np.full(n, L / n)
    grid = Grid(M, L / M)
    p = ParticleEnsemble.from_arrays(x, v, w)
    w64 = p.w.double().cpu().numpy()
    rho, _ = deposit(p, grid)
    rho_ion = float(rho.sum()) * grid.eta / L
    f = FieldState.zeros(M, 2, rho_ion)
    f.E1.copy_(poisson_solve(rho, rho_ion, grid))
    E1_0 = f.E1.cpu().numpy().copy()
    net = MlpScoreNet.init_glorot(2, 64, rng)
    onet = O.Net(*[a.cpu().numpy().astype(np.float64).copy() for a in net.params()])
    est = SbtmEstimator(net, L, K, rng, lr=1e-3, weight_decay=0.0, divergence="exact")
    sim = Simulation(p, f, grid, dt=dt, nu=nu, mode="VPL", gamma=-2.0, estimator=est,
                     max_rows=steps + 1)
    for k in range(1, steps + 1):
        sim.step(k)
    sim.check()
    got = sim.records(range(1, steps + 1), range(1, steps + 1), [dt * k for k in range(1, steps + 1)])
    st = dict(x=x.copy(), v=v.copy(), w=w64, E1=E1_0.copy(), E2=np.zeros(M), B3=np.zeros(M))
    d0 = O.diagnostics(v, w64, E1_0, np.zeros(M), np.zeros(M), grid.eta)
    opt = O.AdamW(lr=1e-3, weight_decay=0.0)
    ref = [O.full_step(st, eta=grid.eta, M=M, dt=dt, nu=nu, mode="VPL", gamma=-2.0, net=onet,
                       opt=opt, K=K, divergence="exact") for _ in range(steps)]
    E0 = d0["E_total"]
    drift_g = np.array([r.E_total / E0 - 1.0 for r in got])
    drift_r = np.array([r["E_total"] / E0 - 1.0 for r in ref])
    EE_g, EE_r = np.array([r.E_E for r in got]), np.array([r["E_E"] for r in ref])
    HD_g, HD_r = np.array([r.H_dot for r in got]), np.array([r["H_dot"] for r in ref])
    P_g = np.array([r.P for r in got])
    pscale = float(np.sum(w64 * np.linalg.norm(v, axis=1)))
    P0 = w64 @ v
    ee = float(np.max(np.abs(EE_g - EE_r)) / np.max(EE_r))
    hd = float(np.max(np.abs(HD_g - HD_r)) / np.max(np.abs(HD_r)))
    py = float(np.max(np.abs(P_g[:, 1] - P0[1])) / pscale)
    print(f"dv = 2, 50 steps: drift device {np.max(np.abs(drift_g)):.3e} oracle "
          f"{np.max(np.abs(drift_r)):.3e} |diff| {np.max(np.abs(drift_g - drift_r)):.3e}; E_E trace "
          f"{ee:.3e}; H_dot trace {hd:.3e}; P_y drift {py:.3e}")
    assert np.max(np.abs(drift_g - drift_r)) <= 1e-6
    assert ee <= 1e-3 and hd <= 5e-2 and py <= 1e-6


def test_blob_50_steps_traces_match_oracle(lib):
    """The blob estimator (Silverman bandwidth per cell, the symmetric pair-sum kernel) in the
    full step for 50 steps (VPL Landau damping, n = 16 384, dv = 3, M = 32, nu = 0.1,
    dt = 0.05) on the device engine and in oracle.full_step(estimator="blob") from the same
    float32 state: energy drift within 1e-6 of the oracle's, E_E trace within 1e-3, H_dot
    trace within 1e-2, P_y / P_z constant to 1e-6."""
    from paper_2603_25832_b200.engine import Simulation
    from paper_2603_25832_b200.pic import Grid, deposit, poisson_solve
    from paper_2603_25832_b200.score import BlobEstimator
    from paper_2603_25832_b200.state import FieldState, ParticleEnsemble

    steps, dt, nu, n, M = 50, 0.05, 0.1, 16384, 32
    L = 4 * math.pi
    rng = np.random.default_rng(8)
    x = f32(rng.uniform(0, L, n))
    x[x >= L] = 0.0
    v = f32(rng.normal(size=(n, 3)))
    w = np.full(n, L / n)
    grid = Grid(M, L / M)
    p = ParticleEnsemble.from_arrays(x, v, w)
    w64 = p.w.double().cpu().numpy()
    rho, _ = deposit(p, grid)
    rho_ion = float(rho.sum()) * grid.eta / L
    f = FieldState.zeros(M, 3, rho_ion)
    f.E1.copy_(poisson_solve(rho, rho_ion, grid))
    E1_0 = f.E1.cpu().numpy().copy()
    sim = Simulation(p, f, grid, dt=dt, nu=nu, mode="VPL", gamma=-3.0,
                     estimator=BlobEstimator(grid, None), max_rows=steps + 1)
    for k in range(1, steps + 1):
        sim.step(k)
    sim.check()
    got = sim.records(range(1, steps + 1), range(1, steps + 1), [dt * k for k in range(1, steps + 1)])
    st = dict(x=x.copy(), v=v.copy(), w=w64, E1=E1_0.copy(), E2=np.zeros(M), B3=np.zeros(M))
    d0 = O.diagnostics(v, w64, E1_0, np.zeros(M), np.zeros(M), grid.eta)
    ref = [O.full_step(st, eta=grid.eta, M=M, dt=dt, nu=nu, mode="VPL", gamma=-3.0, net=None,
                       opt=None, K=0, estimator="blob", bandwidth=None) for _ in range(steps)]
    E0 = d0["E_total"]
    drift_g = np.array([r.E_total / E0 - 1.0 for r in got])
    drift_r = np.array([r["E_total"] / E0 - 1.0 for r in ref])
    EE_g, EE_r = np.array([r.E_E for r in got]), np.array([r["E_E"] for r in ref])
    HD_g, HD_r = np.array([r.H_dot for r in got]), np.array([r["H_dot"] for r in ref])
    P_g = np.array([r.P for r in got])
    pscale = float(np.sum(w64 * np.linalg.norm(v, axis=1)))
    P0 = w64 @ v
    ee = float(np.max(np.abs(EE_g - EE_r)) / np.max(EE_r))
    hd = float(np.max(np.abs(HD_g - HD_r)) / np.max(np.abs(HD_r)))
    pyz = float(np.max(np.abs(P_g[:, 1:] - P0[None, 1:])) / pscale)
    print(f"blob, 50 steps: drift device {np.max(np.abs(drift_g)):.3e} oracle "
          f"{np.max(np.abs(drift_r)):.3e} |diff| {np.max(np.abs(drift_g - drift_r)):.3e}; E_E trace "
          f"{ee:.3e}; H_dot trace {hd:.3e}; P_yz drift {pyz:.3e}")
    assert np.max(np.abs(drift_g - drift_r)) <= 1e-6
    assert ee <= 1e-3 and hd <= 1e-2 and pyz <= 1e-6
