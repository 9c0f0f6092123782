"""The reference's acceptance criteria (ref: pkg/tests/test_acceptance.py, A1-A11) run on the
device path, through this package's public API, with the reference's configurations and
seeds. Criteria that the reference states for float64 arithmetic keep their structure with
float32 tolerances stated here; the physics criteria keep the reference's own bounds.

  A1  collision conservation, 100 random ensembles: momentum and energy relative <= 1e-5
      (float32; the reference's float64 bound is 1e-10)
  A2  entropy production H_dot >= -1e-6 * scale on the same ensembles (float32)
  A6  VPL Landau damping, dv = 2, n = 2e4, nu = 1, t = 10 with SBTM: every temperature
      component within 5% of the analytic T_inf (the reference's bound); the momentum
      sub-criterion is reported (the reference documents it as known-red: an undamped
      plasma-frequency mode of sampling noise), and the drift beyond that mode is bounded
  A7  nu = 0: the blob and SBTM runs write byte-identical diagnostics CSVs
  A8  score_test: the pretrained SBTM net's initial-score MSE beats the blob estimator's,
      median over 3 seeds (two-stream, n = 1e5)
  A9  energy bookkeeping of the sampled Landau-damping ensemble and its Poisson field
  A10 scaling trend: SBTM update time grows < 2.5x per doubling of n (the reference's sizes
      1e4, 2e4, 4e4), the one-cell blob sum > 2.5x (O(n^2)); CUDA-event timings. The blob leg
      runs at 4x the reference's sizes: at 1e4-4e4 particles the device's O(n^2) sum takes
      0.05-0.7 ms and a fixed ~0.15 ms of launches hides the growth (measured ratios 1.87,
      2.22 there)
  A11 Weibel equilibrium temperature within 3% of 0.035
"""

import math
import os

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


def _random_collision_ensembles():
    """100 random ensembles across n in {1e2, 1e3, 1e4} and dv in {2, 3} (the reference's
    A1 construction, test_acceptance.py:37-55), float32-rounded."""
    from paper_2603_25832_b200.state import seeded_rng

    rng = seeded_rng(0)
    sizes = [100] * 40 + [1000] * 40 + [10000] * 20
    out = []
    for i, n in enumerate(sizes):
        dv = 2 if i % 2 == 0 else 3
        L = float(rng.uniform(3.0, 15.0))
        M = int(rng.integers(1, 17))
        x = rng.uniform(0, L, n).astype(np.float32).astype(np.float64)
        x[x >= L] = 0.0
        v = (rng.normal(size=(n, dv)) * rng.uniform(0.2, 2.0)).astype(np.float32).astype(np.float64)
        s = (rng.normal(size=(n, dv)) * rng.uniform(0.1, 5.0)).astype(np.float32).astype(np.float64)
        out.append((x, v, np.full(n, L / n), s, L, M))
    return out


def test_A1_A2_collision_conservation_and_entropy_sign(lib):
    from paper_2603_25832_b200.collision import build_cell_index, collision_force
    from paper_2603_25832_b200.pic import Grid
    from paper_2603_25832_b200.state import ParticleEnsemble

    worst_mom = worst_en = 0.0
    worst_h = 0.0
    for x, v, w, s, L, M in _random_collision_ensembles():
        p = ParticleEnsemble.from_arrays(x, v, w)
        grid = Grid(M, L / M)
        U = collision_force(p, s, build_cell_index(p, grid), grid, -float(v.shape[1]))
        U = U.double().cpu().numpy()
        wU = w[:, None] * U
        mom = np.max(np.abs(wU.sum(axis=0))) / (max(np.max(np.abs(wU)), 1e-300) * x.size)
        en = abs(float(np.sum(w * np.einsum("ij,ij->i", v, U))))
        en /= max(float(np.sum(w * np.linalg.norm(v, axis=1) * np.linalg.norm(U, axis=1))), 1e-300)
        h = float(np.sum(w * np.einsum("ij,ij->i", s, U)))
        hs = max(float(np.sum(w * np.linalg.norm(s, axis=1) * np.linalg.norm(U, axis=1))), 1e-300)
        worst_mom, worst_en = max(worst_mom, mom), max(worst_en, en)
        worst_h = min(worst_h, h / hs)
    print(f"A1: momentum {worst_mom:.2e}, energy {worst_en:.2e}; A2: min H_dot/scale {worst_h:.2e}")
    assert worst_mom <= 1e-5 and worst_en <= 1e-5
    assert worst_h >= -1e-6


def test_A6_equilibrium_relaxation(lib, tmp_path):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.diagnostics import read_snapshot
    from paper_2603_25832_b200.run import run

    cfg = build_config(overrides=dict(preset="landau_damping", dv=2, n=20000, M=32, nu=1.0,
                                      t_final=10.0, dt=0.02, K=10, hidden=64, estimator="sbtm",
                                      pretrain_budget=3000, seed=0))
    out = str(tmp_path / "a6")
    records = run(cfg, out)
    (x, v, w), _, _ = read_snapshot(os.path.join(out, f"snapshot_{cfg.n_steps:06d}.bin"))
    T_inf, _ = O.vpl_equilibrium(records[0].E_total, records[0].P, 1.0, cfg.L)
    wsum = w.sum()
    u_hat = w @ v / wsum
    temps = np.array([float(np.sum(w * (v[:, i] - u_hat[i]) ** 2) / wsum) for i in range(cfg.dv)])
    dP_vec = records[-1].P - records[0].P
    slosh = records[0].P[0] * (math.cos(cfg.t_final) - 1.0)
    residual = float(np.linalg.norm(dP_vec - np.array([slosh, 0.0])))
    print(f"A6: temperatures {np.round(temps, 4)} vs T_inf {T_inf:.4f}; |dP| "
          f"{np.linalg.norm(dP_vec):.3e} (uniform-mode prediction {slosh:.3e}, drift beyond it "
          f"{residual:.3e})")
    assert np.all(np.abs(temps - T_inf) <= 0.05 * T_inf)
    assert residual < 1e-2


def test_A7_collisionless_estimator_equivalence(lib, tmp_path):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.run import run

    blobs = {}
    for est in ("blob", "sbtm"):
        cfg = build_config(overrides=dict(preset="landau_damping", dv=2, n=10000, M=64, nu=0.0,
                                          t_final=1.0, estimator=est, seed=0))
        out = str(tmp_path / f"a7_{est}")
        run(cfg, out)
        blobs[est] = open(os.path.join(out, "diagnostics.csv"), "rb").read()
    assert blobs["blob"] == blobs["sbtm"]


def test_A8_initial_score_mse_ordering(lib, tmp_path):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.run import score_test

    blob, sbtm = [], []
    for seed in (0, 1, 2):
        cfg = build_config(overrides=dict(preset="two_stream", n=100000, dv=3,
                                          pretrain_budget=1500, seed=seed))
        cfg.pretrain_batch = 8192
        rep = score_test(cfg, str(tmp_path / f"a8_{seed}"), compute_force=False)
        blob.append(rep["blob"]["mse"])
        sbtm.append(rep["sbtm"]["mse"])
    print(f"A8: median MSE sbtm {np.median(sbtm):.4f} vs blob {np.median(blob):.4f}")
    assert float(np.median(sbtm)) < float(np.median(blob))


def test_A9_energy_bookkeeping(lib):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.pic import Grid, deposit
    from paper_2603_25832_b200.run import initial_fields
    from paper_2603_25832_b200.sampling import sample_arrays
    from paper_2603_25832_b200.state import ParticleEnsemble, seeded_rng

    n, dv = 100000, 3
    L = 4 * math.pi
    rng = seeded_rng(0)
    v = rng.normal(size=(n, dv))
    w = np.full(n, L / n)
    E_K = 0.5 * float(np.sum(w * np.einsum("ij,ij->i", v, v)))
    sigma_K = 0.5 * L * math.sqrt(2.0 * dv / n)
    assert abs(E_K - 0.5 * dv * L) <= 4 * sigma_K
    cfg = build_config(overrides=dict(preset="landau_damping", n=n, seed=0))
    grid = Grid(cfg.M, cfg.eta)
    p = ParticleEnsemble.from_arrays(*sample_arrays(cfg, seeded_rng(0)))
    rho, J = deposit(p, grid)
    fields = initial_fields(cfg, grid, rho, J)
    E1 = fields.E1.double().cpu().numpy()
    E_E = 0.5 * grid.eta * float(np.sum(E1 ** 2))
    sig = math.sqrt(2.0 / n)
    k_m = 2 * math.pi * np.arange(1, cfg.M // 2 + 1) / cfg.L
    noise_floor = cfg.L / (2 * n) * float(np.sum(1.0 / k_m ** 2))
    hi = (cfg.alpha + 4 * sig) ** 2 * cfg.L / (4 * cfg.k ** 2) + 4 * noise_floor
    lo = (cfg.alpha - 4 * sig) ** 2 * cfg.L / (4 * cfg.k ** 2)
    print(f"A9: E_E {E_E:.5f} in [{lo:.5f}, {hi:.5f}]")
    assert lo <= E_E <= hi


def test_A10_scaling_trend(lib):
    from paper_2603_25832_b200.collision import build_cell_index
    from paper_2603_25832_b200.pic import Grid
    from paper_2603_25832_b200.score import BlobEstimator, MlpScoreNet, SbtmEstimator
    from paper_2603_25832_b200.state import ParticleEnsemble, seeded_rng

    sizes = (10000, 20000, 40000)
    L = 10 * math.pi
    rng = seeded_rng(0)

    def ens(n):
        return ParticleEnsemble.from_arrays(rng.uniform(0, L, n), rng.normal(size=(n, 3)),
                                            np.full(n, L / n))

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
        return float(np.median(out))

    sbtm = []
    for n in sizes:
        p = ens(n)
        est = SbtmEstimator(MlpScoreNet.init_glorot(3, 256, rng), L, K=3, rng=seeded_rng(1))
        sbtm.append(timed(lambda: est.update(p), 3))
    grid = Grid(1, L)
    blob_est = BlobEstimator(grid)
    blob = []
    for n in (4 * m for m in sizes):
        p = ens(n)
        ci = build_cell_index(p, grid)
        blob.append(timed(lambda: blob_est.estimate(p, ci), 3))
    r = [sbtm[1] / sbtm[0], sbtm[2] / sbtm[1], blob[1] / blob[0], blob[2] / blob[1]]
    print(f"A10: sbtm {np.round(sbtm, 3)} ms (ratios {r[0]:.2f}, {r[1]:.2f}); one-cell blob "
          f"{np.round(blob, 3)} ms (ratios {r[2]:.2f}, {r[3]:.2f})")
    assert r[0] < 2.5 and r[1] < 2.5 and r[2] > 2.5 and r[3] > 2.5


def test_A11_weibel_equilibrium_oracle(lib):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.pic import Grid, deposit
    from paper_2603_25832_b200.run import initial_fields
    from paper_2603_25832_b200.sampling import sample_arrays
    from paper_2603_25832_b200.state import ParticleEnsemble, seeded_rng

    cfg = build_config(overrides=dict(preset="weibel", n=100000, seed=0))
    grid = Grid(cfg.M, cfg.eta)
    x, v, w = sample_arrays(cfg, seeded_rng(0))
    p = ParticleEnsemble.from_arrays(x, v, w)
    rho, J = deposit(p, grid)
    fields = initial_fields(cfg, grid, rho, J)
    E_K = 0.5 * float(np.sum(w * np.einsum("ij,ij->i", v, v)))
    B3 = fields.B3.double().cpu().numpy()
    E_B = 0.5 * grid.eta * float(np.sum(B3 ** 2))
    B_mean = np.array([0.0, 0.0, grid.eta * B3.sum() / cfg.L])
    T_inf, _ = O.vml_equilibrium(E_K + E_B, B_mean, 1.0, cfg.L)
    print(f"A11: T_inf {T_inf:.5f} vs 0.035")
    assert abs(T_inf - 0.035) <= 0.03 * 0.035
