"""Analysis mode: the t = 0 score comparison (reference: run.py:134-185).

For every requested estimator the run is re-seeded and re-sampled, the score estimated on
device (blob KDE, or the SBTM net pretrained on the analytic score), the weighted MSE
against the analytic score reported, and a CSV written with columns x, v*, s_est*, s_true*
(and U* from the Landau kernel when requested), 17 significant digits.
"""

from __future__ import annotations

import json
import os

import numpy as np

from .collision import build_cell_index, collision_force
from .config import SimConfig
from .pic import Grid
from .sampling import sample_arrays
from .score import MlpScoreNet, SbtmEstimator, blob_score
from .state import ParticleEnsemble, seeded_rng


def _estimate(name: str, config: SimConfig, particles, ci, grid, score_fn, rng):
    if name == "blob":
        return blob_score(particles, ci, grid, config.fixed_bandwidth())
    if name == "sbtm":
        net = MlpScoreNet.init_glorot(config.dv, config.hidden, rng)
        est = SbtmEstimator(net, config.L, config.K, rng, lr=config.lr,
                            weight_decay=config.weight_decay)
        est.pretrain(particles, score_fn, budget=config.pretrain_budget,
                     batch=config.pretrain_batch, lr=config.pretrain_lr)
        return est.estimate(particles)
    raise ValueError(f"unknown estimator: {name!r}")


def score_test(config: SimConfig, out_dir: str, *, compute_force: bool = True,
               estimators=("blob", "sbtm")) -> dict:
    from .run import initial_score_fn

    config.validate()
    if config.preset == "custom":
        raise ValueError("score_test needs a preset with an analytic initial score")
    os.makedirs(out_dir, exist_ok=True)
    grid = Grid(config.M, config.eta)
    score_fn = initial_score_fn(config)
    summary = {}
    for name in estimators:
        rng = seeded_rng(config.seed)
        particles = ParticleEnsemble.from_arrays(*sample_arrays(config, rng))
        ci = build_cell_index(particles, grid)
        s_true = score_fn(particles.x, particles.v)
        s_est = _estimate(name, config, particles, ci, grid, score_fn, rng)
        diff = s_est.double() - s_true.double()
        w = particles.w.double()
        mse = float((w * (diff * diff).sum(1)).sum() / w.sum())
        x, v, _ = particles.to_numpy()
        blocks = [("x", x[:, None]), ("v", v), ("s_est", s_est.double().cpu().numpy()),
                  ("s_true", s_true.double().cpu().numpy())]
        if compute_force:
            U = collision_force(particles, s_est, ci, grid, config.gamma)
            blocks.append(("U", U.double().cpu().numpy()))
        header = [lbl if lbl == "x" else f"{lbl}{i + 1}" for lbl, arr in blocks
                  for i in range(arr.shape[1])]
        table = np.concatenate([arr for _, arr in blocks], axis=1)
        csv_path = os.path.join(out_dir, f"score_test_{name}.csv")
        with open(csv_path, "w", encoding="utf-8", newline="\n") as fh:
            fh.write(",".join(header) + "\n")
            for row in table:
                fh.write(",".join(format(val, ".17g") for val in row) + "\n")
        summary[name] = {"mse": mse, "csv": csv_path}
    with open(os.path.join(out_dir, "score_test_report.json"), "w", encoding="utf-8") as fh:
        fh.write(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    return summary
