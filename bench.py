#!/usr/bin/env python
"""Benchmark of the B200 per-timestep hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4] [--impl ours|reference]

Workload (default c4 = BASELINE config 4, the largest single-GPU configuration): Landau
damping 1D3V, SBTM, n = 2^24 particles, M = 1024 cells on L = 4 pi, nu = 0.1, dt = 0.05,
K = 10 exact-divergence ISM steps per time step with BASELINE's score MLP
"(x, v) -> 2x128 SiLU -> R^3" (tcgen05 hidden GEMMs), Adam lr 1e-3 (AdamW, wd = 0).
A step is one full Algorithm-1 step (push, bin, deposit + field, K ISM steps, score, Landau
collision + push, diagnostics) over the synthetic ensemble (seeded sampler, random-init net).
The same line carries config 3 (Weibel, full Maxwell VML, n = 2^22) as `config3_vml`, config 4
with the blob estimator (h = 0.025) as `config4_blob` and config 4 with the reference's own
softsign network as `reference_net_variant`.

  value  = particle-steps/s, device-timed with CUDA events per step (L2 flushed between
           timed steps by a 256 MiB write outside the timed windows), max over ranks.
           N > 1: strong scaling — the same n = 2^24 particles split by cell range.
  e2e    = same metric through Simulation.step_host with pinned HOST buffers: H2D of x, v,
           the step, D2H of x, v, the diagnostics row and the error flags, and the flag check
           run() does, every step.
  roofline: the kernel with the largest share of the step (the Landau pair kernel at c4)
           against the FP32 peak measured in-run by spic_fp32_probe.
  cpu_baseline: the float64 oracle port (oracle/, C + OpenMP) on a bounded sample of the same
           workload, rank 0, N = 1 only.
`--impl reference` times that CPU port alone (the reference arm; the reference itself is pure
Python + numba and is not shipped to the GPU box), on the same config dict.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FLOP_PER_PAIR = 38.0        # ordered pair kernel, per ordered live pair
FLOP_PER_UPAIR = 41.0       # antisymmetric kernel, per unordered live pair


def pair_flops(live_ordered: float, n: int) -> float:
    """Algorithmic FLOP of one pair-kernel launch. The default (antisymmetric) kernel evaluates
    each unordered live pair once: 41 FLOP x (live - n) / 2 (live counts ordered pairs incl.
    the n self pairs); SPIC_LANDAU_VARIANT=o/s selects the ordered kernel (38 per ordered pair)."""
    if os.environ.get("SPIC_LANDAU_VARIANT"):
        return FLOP_PER_PAIR * live_ordered
    return FLOP_PER_UPAIR * max(live_ordered - n, 0.0) / 2.0


PAIR_KERNEL = ("spic_landau (k_landau_x2, ordered pairs)" if os.environ.get("SPIC_LANDAU_VARIANT")
               else "spic_landau (k_landau_sym, unordered pairs)")
METRIC = "particle-steps/s (full VML step, SBTM)"

WORKLOADS = {
    # BASELINE configs as named, incl. their score MLP "(x,v) -> 2x128 SiLU -> R^3"
    # (extension M1: tcgen05 hidden GEMMs). "...ss" = the same config with the reference's own
    # softsign 1x128 network (the only network the reference has; like-for-like with its arm).
    "c2": dict(workload="config2_two_stream_sbtm", preset="two_stream", mode="VPL", n=1 << 20,
               M=128, L=10 * math.pi, alpha=0.001, k=0.2, c=2.4, nu=0.05, dt=0.05, K=10,
               hidden=128, lr=1e-3, weight_decay=0.0, divergence="exact", estimator="sbtm",
               net="silu"),
    "c0": dict(workload="config0_landau_damping_sbtm", preset="landau_damping", mode="VPL",
               n=65536, M=64, L=4 * math.pi, alpha=0.01, k=0.5, c=0.0, nu=0.1, dt=0.05, K=10,
               hidden=128, lr=1e-3, weight_decay=0.0, divergence="exact", estimator="sbtm",
               net="silu"),
    "c4": dict(workload="config4_landau_damping_sbtm_n2^24", preset="landau_damping", mode="VPL",
               n=1 << 24, M=1024, L=4 * math.pi, alpha=0.01, k=0.5, c=0.0, nu=0.1, dt=0.05,
               K=10, hidden=128, lr=1e-3, weight_decay=0.0, divergence="exact",
               estimator="sbtm", net="silu"),
    "c2blob": dict(workload="config2_two_stream_blob", preset="two_stream", mode="VPL",
                   n=1 << 20, M=128, L=10 * math.pi, alpha=0.001, k=0.2, c=2.4, nu=0.05,
                   dt=0.05, K=0, hidden=128, lr=1e-3, weight_decay=0.0, divergence="exact",
                   estimator="blob", bandwidth="silverman"),
    "c4blob": dict(workload="config4_landau_damping_blob_n2^24", preset="landau_damping",
                   mode="VPL", n=1 << 24, M=1024, L=4 * math.pi, alpha=0.01, k=0.5, c=0.0,
                   nu=0.1, dt=0.05, K=0, hidden=128, lr=1e-3, weight_decay=0.0,
                   divergence="exact", estimator="blob", bandwidth=0.025),
}
# BASELINE config 3: Weibel, full Maxwell (VML), anisotropic Maxwellian T = (0.01, 0.04, 0.04),
# seeded B_z noise of amplitude 1e-4 (extension samplers)
WORKLOADS["c3"] = dict(workload="config3_weibel_vml_sbtm", preset="weibel", mode="VML",
                       n=1 << 22, M=256, L=2 * math.pi / 1.25, alpha=0.0, k=1.25, c=0.0,
                       beta=0.01, alpha_B=0.0, nu=0.01, dt=0.02, K=10, hidden=128, lr=1e-3,
                       weight_decay=0.0, divergence="exact", estimator="sbtm", net="silu",
                       sampler="anisotropic", temps=(0.01, 0.04, 0.04), b3_noise=1e-4)
for _k in ("c0", "c2", "c3", "c4"):
    WORKLOADS[_k + "ss"] = dict(WORKLOADS[_k], net="softsign",
                                workload=WORKLOADS[_k]["workload"] + "_reference_softsign_net")
NET_LABEL = {"silu": "SiLU 2x128 (BASELINE's MLP; extension M1, tcgen05 split-BF16 hidden GEMMs)",
             "softsign": "softsign 1x128 (the reference's network)"}
# per particle per ISM step: G1 [W2 h1 | B d1], G2 [W2^T da2 | B^T y2], G3 [da2 h1^T, y2 d1^T]
SILU_GEMM_FLOP_PER_PARTICLE = 3 * 2 * (2 * 128 * 128)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


def make_config(wl: dict, seed: int):
    from paper_2603_25832_b200.config import SimConfig

    keys = {f for f in SimConfig.__dataclass_fields__}
    kw = {k: v for k, v in wl.items() if k in keys}
    if "bandwidth" in kw:
        kw["bandwidth"] = str(kw["bandwidth"])
    return SimConfig(seed=seed, t_final=wl["dt"], **kw)


# ------------------------------------------------------------------------------------------
# CPU baseline: the oracle port on a bounded sample
# ------------------------------------------------------------------------------------------

def cpu_sample_plan(wl: dict) -> dict:
    """Bounded CPU sample of one step of the workload (about 10-30 s on 16 host cores):
    the pair kernels on every `cell_stride`-th cell (about 1.3e10 stencil pairs), the SiLU ISM
    on `ism_particles` particles (numpy float64), the softsign ISM on up to 65 536; everything
    else (push, deposit, field, bin, softsign forward) on all n. Each sampled stage is scaled
    up by its factor."""
    n, M = wl["n"], wl["M"]
    stencil_pairs = 3.0 * n * n / M if M >= 3 else float(n) * n
    cell_stride = int(max(1, min(M, round(stencil_pairs / 1.3e10))))
    if wl.get("net") == "silu":
        ism = min(n, 16384)
        fwd_stride = max(1, n // (1 << 18))
    else:
        ism = min(n, 65536)
        fwd_stride = 1
    return {"cell_stride": cell_stride, "ism_particles": ism, "forward_stride": fwd_stride}


def cpu_sample_step(wl: dict, host_state: dict, plan: dict, *, seed: int = 0):
    """Seconds for one full step of the workload on the host cores, measured on the bounded
    sample of cpu_sample_plan() and scaled up stage by stage."""
    from oracle import oracle as O

    x, v, w = host_state["x"], host_state["v"], host_state["w"]
    E1, E2, B3 = host_state["E1"], host_state["E2"], host_state["B3"]
    M, L = wl["M"], wl["L"]
    eta = L / M
    n = x.shape[0]
    cell_stride = plan["cell_stride"]
    t = {}
    t0 = time.perf_counter()
    x1, v1 = O.push(x, v, E1, E2, B3, eta, M, wl["dt"])
    rho, J = O.deposit(x1, v1, w, eta, M)
    O.vpl_field_step(E1, J, wl["dt"]) if wl["mode"] == "VPL" else O.maxwell_step(E1, E2, B3, J, eta, wl["dt"])
    O.build_cell_index(x1, eta, M)
    t["push_deposit_field_bin"] = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    sub = np.sort(rng.choice(n, size=plan["ism_particles"], replace=False)) \
        if plan["ism_particles"] < n else np.arange(n)
    if wl["estimator"] == "sbtm" and wl.get("net") == "silu":
        from oracle import silu_oracle as SO

        params = SO.glorot(128, rng)
        u = SO.inputs(x1[sub], v1[sub], L)
        m, v2 = np.zeros_like(params), np.zeros_like(params)
        t0 = time.perf_counter()
        for k in range(wl["K"]):
            _, g = SO.ism_loss_and_grad(params, u, w[sub], 128)
            params, m, v2 = SO.adamw_step(params, g, m, v2, k + 1, wl["lr"],
                                          weight_decay=wl["weight_decay"])
        t["ism"] = (time.perf_counter() - t0) * (n / len(sub))
        t0 = time.perf_counter()
        fsub = np.arange(0, n, plan["forward_stride"])
        s = np.zeros_like(v1)
        s[fsub] = SO.forward(params, SO.inputs(x1[fsub], v1[fsub], L), 128, with_div=False)[0]
        t["forward"] = (time.perf_counter() - t0) * (n / len(fsub))
    elif wl["estimator"] == "sbtm":
        net = O.Net.glorot(v.shape[1], wl["hidden"], rng)
        opt = O.AdamW(lr=wl["lr"], weight_decay=wl["weight_decay"])
        t0 = time.perf_counter()
        O.sbtm_update(net, opt, x1[sub], v1[sub], w[sub], wl["K"], L=L, divergence=wl["divergence"])
        t["ism"] = (time.perf_counter() - t0) * (n / len(sub))
        t0 = time.perf_counter()
        s = O.mlp_forward(net, x1 / L, v1)
        t["forward"] = time.perf_counter() - t0
    else:
        t0 = time.perf_counter()
        s = O.blob_score(x1, v1, w, eta, M, wl.get("bandwidth"), cell_stride=cell_stride)
        t["blob"] = (time.perf_counter() - t0) * cell_stride
    t0 = time.perf_counter()
    O.collision_force(x1, v1, w, s, eta, M, -3.0, cell_stride=cell_stride)
    t["collision"] = (time.perf_counter() - t0) * cell_stride
    return sum(t.values()), t


_SAMPLE_CACHE: dict = {}


def sample_workload(wl: dict, cfg, rng):
    """Initial particles of a workload: the reference's preset sampler, or BASELINE config 3's
    anisotropic Maxwellian; plus the seeded B3 noise (None unless the workload has one).
    Memoised per (workload sampling parameters, seed): a variant line of the same config (e.g.
    the softsign network) reuses the ensemble and continues from the same rng state."""
    key = (wl["preset"], wl["n"], wl["M"], wl["L"], wl.get("sampler"), wl.get("b3_noise"),
           cfg.seed)
    hit = _SAMPLE_CACHE.get(key)
    if hit is not None:
        rng.bit_generator.state = hit[1]
        return hit[0]
    res = _sample_workload(wl, cfg, rng)
    _SAMPLE_CACHE.clear()
    _SAMPLE_CACHE[key] = (res, rng.bit_generator.state)
    return res


def _sample_workload(wl: dict, cfg, rng):
    from paper_2603_25832_b200.sampling import anisotropic_ensemble, sample_arrays, seeded_b3_noise

    if wl.get("sampler") == "anisotropic":
        x, v, w = anisotropic_ensemble(cfg.n, cfg.L, wl["temps"], rng)
    else:
        x, v, w = sample_arrays(cfg, rng)
    b3 = seeded_b3_noise(cfg.M, wl["b3_noise"], rng) if wl.get("b3_noise") else None
    return x, v, w, b3


def host_initial_state(wl: dict, seed: int):
    from oracle import oracle as O

    cfg = make_config(wl, seed)
    x, v, w, b3 = sample_workload(wl, cfg, np.random.default_rng(seed))
    x = x.astype(np.float32).astype(np.float64)
    v = v.astype(np.float32).astype(np.float64)
    M, L = wl["M"], wl["L"]
    eta = L / M
    rho, _ = O.deposit(x, v, w, eta, M)
    rho_ion = float(rho.sum() * eta / L)
    E1 = O.poisson_solve(rho, rho_ion, eta) if wl["mode"] == "VPL" else np.zeros(M)
    return dict(x=x, v=v, w=w, E1=E1, E2=np.zeros(M), B3=b3 if b3 is not None else np.zeros(M))


def cpu_baseline_line(wl: dict, seed: int, reps: int = 1, warm: int = 0):
    from oracle import oracle as O

    st = host_initial_state(wl, seed)
    plan = cpu_sample_plan(wl)
    for _ in range(warm):
        cpu_sample_step(wl, st, plan, seed=seed)
    times, parts = [], None
    wall0 = time.perf_counter()
    for _ in range(reps):
        T, parts = cpu_sample_step(wl, st, plan, seed=seed)
        times.append(T)
    sample_seconds = (time.perf_counter() - wall0) / max(reps, 1)
    T = statistics.mean(times)
    n = wl["n"]
    live = O.count_live_pairs(st["x"], wl["L"] / wl["M"], wl["M"]) if n <= (1 << 21) else None
    net = wl.get("net")
    sample = (f"oracle/ float64 C+OpenMP port of the reference path; per step: push/deposit/"
              f"field/bin on all n; the pair kernel on every {plan['cell_stride']}-th cell "
              f"(x{plan['cell_stride']}); ")
    if wl["estimator"] == "blob":
        sample += f"the blob score on the same cells (x{plan['cell_stride']})"
    elif net == "silu":
        sample += (f"the SiLU 2x128 score net as the float64 numpy restatement "
                   f"oracle/silu_oracle.py (the reference has no such network): K ISM steps on "
                   f"{plan['ism_particles']} particles (x{n / plan['ism_particles']:.0f}), "
                   f"forward on every {plan['forward_stride']}-th particle "
                   f"(x{plan['forward_stride']})")
    else:
        sample += (f"the reference's softsign score net: K ISM steps on "
                   f"{plan['ism_particles']} particles (x{n / plan['ism_particles']:.0f}), "
                   f"forward on all n")
    scale = {"pair_cells": plan["cell_stride"], "ism": n / plan["ism_particles"],
             "forward": plan["forward_stride"] if net == "silu" else 1}
    return dict(value=n / T, unit="particle-steps/s", cores=O.num_threads(), kind="port",
                sample=sample, extrapolated=True, sample_seconds=sample_seconds,
                scale_factors=scale, seconds_per_step=T, stage_seconds=parts,
                pair_interactions_per_s=(live / parts["collision"]) if live else None)


def bench_config(wl: dict, world: int) -> dict:
    """The `config` dict of a bench line; identical for the GPU arm and the reference arm."""
    return {"workload": wl["workload"], "n": wl["n"], "M": wl["M"], "L": wl["L"],
            "mode": wl["mode"], "estimator": wl["estimator"], "K_ism": wl["K"],
            "hidden": wl["hidden"], "net": NET_LABEL[wl.get("net", "softsign")]
            if wl["estimator"] == "sbtm" else None,
            "bandwidth": wl.get("bandwidth"), "divergence": wl["divergence"],
            "nu": wl["nu"], "dt": wl["dt"],
            "l2": "flushed between timed steps (256 MiB write + read-back, outside timed windows)",
            "parallelism": ("single GPU" if world == 1 else
                            f"cell-range decomposition of the same n over {world} ranks (NCCL): "
                            "migration, halo, rho/J and ISM-gradient allreduces")}


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.stop_ev = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.max_mhz = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self.stop_ev.wait(0.1)

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.th.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def fp32_peak_tflops(torch, _lib) -> float:
    import ctypes

    out = torch.zeros(4096, device="cuda")
    flop = ctypes.c_double(0.0)
    best = 0.0
    for it in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("spic_fp32_probe", 1 << 14, 148 * 4, _lib.ptr(out), ctypes.byref(flop),
                  _lib.stream_handle())
        e1.record()
        e1.synchronize()
        if it:
            best = max(best, flop.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def make_estimator_for(wl: dict, cfg, rng, device, grid):
    from paper_2603_25832_b200.score import BlobEstimator, MlpScoreNet, SbtmEstimator

    if wl["estimator"] == "sbtm" and wl.get("net") == "silu":
        from paper_2603_25832_b200.silu_net import SiluEstimator, SiluScoreNet

        net = SiluScoreNet.init_glorot(rng, device=device)
        return SiluEstimator(net, cfg.L, cfg.K, rng, lr=cfg.lr, weight_decay=cfg.weight_decay)
    if wl["estimator"] == "sbtm":
        net = MlpScoreNet.init_glorot(cfg.dv, cfg.hidden, rng, device=device)
        return SbtmEstimator(net, cfg.L, cfg.K, rng, lr=cfg.lr, weight_decay=cfg.weight_decay,
                             divergence=cfg.divergence, rademacher=cfg.rademacher)
    bw = wl["bandwidth"]
    return BlobEstimator(grid, None if bw == "silverman" else float(bw))


def build_sim(wl: dict, seed: int, device):
    import torch

    from paper_2603_25832_b200.engine import Simulation
    from paper_2603_25832_b200.pic import Grid, deposit, poisson_solve
    from paper_2603_25832_b200.run import initial_fields
    from paper_2603_25832_b200.state import ParticleEnsemble

    cfg = make_config(wl, seed)
    rng = np.random.default_rng(seed)
    x, v, w, b3 = sample_workload(wl, cfg, rng)
    grid = Grid(cfg.M, cfg.eta)
    p = ParticleEnsemble.from_arrays(x, v, w, device=device)
    rho, J = deposit(p, grid)
    fields = initial_fields(cfg, grid, rho, J)
    if b3 is not None:
        fields.B3.copy_(torch.as_tensor(b3, dtype=fields.B3.dtype, device=fields.B3.device))
    est = make_estimator_for(wl, cfg, rng, device, grid)
    sim = Simulation(p, fields, grid, dt=cfg.dt, nu=cfg.nu, mode=cfg.mode, gamma=cfg.gamma,
                     estimator=est, max_rows=4)
    del torch
    return sim


def variant_line(torch, device, wl: dict, seed: int, steps: int = 3) -> dict:
    """Graph-replayed full steps of another network variant of the same workload (CUDA
    events, L2 flushed between steps): particle-steps/s and ms per step."""
    sim = build_sim(wl, seed, device)
    n = wl["n"]
    for _ in range(3):
        sim.step(0)
    torch.cuda.synchronize()
    sim.check()
    sim.capture(row=3)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    total = 0.0
    for _ in range(steps):
        l2_flush(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sim.replay(1)
        e1.record()
        e1.synchronize()
        total += e0.elapsed_time(e1)
    sim.check()
    return {"workload": wl["workload"], "net": NET_LABEL[wl.get("net", "softsign")],
            "value": n * steps / (total * 1e-3), "unit": "particle-steps/s",
            "ms_per_step": total / steps}


def silu_kernel_roofline(torch, device, sim, wl: dict, key: str, reps: int = 10) -> dict:
    """The SiLU ISM kernel (spic_silu_ism_partials: k_silu + its fixed-order column reduce)
    timed on the stream it runs on over `reps` launches on the step's own cell-sorted records.
    achieved = algorithmic GEMM FLOP (3 x 2 x 2*128*128 per particle) / launch time;
    peak = the measured bf16 tensor peak / 3 (split-BF16 executes three bf16 products per
    fp32-accurate product)."""
    from paper_2603_25832_b200.silu_net import _silu_partials

    net, n, L = sim.trainer.net, wl["n"], wl["L"]
    if hasattr(sim, "ci"):  # the single-GPU engine's cell-sorted records of the last step
        xv, sw = sim.ci.xv, sim.ci.sw
    else:  # decomposed run: the same record count on this rank, seeded synthetic values
        g = torch.Generator(device=device).manual_seed(7)
        xv = torch.rand(n, 4, device=device, generator=g) * torch.tensor([L, 1, 1, 1], device=device)
        sw = torch.full((n, 4), L / n, device=device)
    _silu_partials(net, xv, sw, n, L)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _silu_partials(net, xv, sw, n, L)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bf16 = float(peaks["bf16_tflops"])
    flop = SILU_GEMM_FLOP_PER_PARTICLE * n
    achieved = flop / (ms * 1e-3) / 1e12
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "silu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(key)
        except Exception:  # noqa: BLE001
            traffic = None
    return {"bound": "tensor", "kernel": "spic_silu_ism_partials (k_silu, tcgen05)",
            "achieved": achieved, "peak": bf16 / 3.0, "unit": "TFLOP/s",
            "frac": achieved / (bf16 / 3.0), "traffic": traffic, "flop_per_launch": flop,
            "launch_ms": ms, "launches_per_step": wl["K"],
            "bf16_tflops_executed": 3.0 * achieved, "bf16_peak": bf16,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst) / 3 split-BF16 passes"}


def config1_microbench(torch, device, n: int = 131072, reps: int = 3) -> dict:
    """BASELINE config 1: one cell, co-located x (so w psi = 1/n), v from the equal mixture of
    N((+-1.5, 0, 0), I3), exact mixture score; all n^2 ordered pairs are live. Times the pair
    kernel alone (CUDA events) and checks momentum / energy conservation of U."""
    from paper_2603_25832_b200 import _lib
    from paper_2603_25832_b200.collision import build_cell_index, landau_sorted
    from paper_2603_25832_b200.pic import Grid
    from paper_2603_25832_b200.state import ParticleEnsemble

    rng = np.random.default_rng(1)
    L = 2.0
    v = rng.normal(size=(n, 3))
    v[:, 0] += np.where(rng.random(n) < 0.5, 1.5, -1.5)
    s = -v.copy()
    s[:, 0] = -v[:, 0] + 1.5 * np.tanh(1.5 * v[:, 0])
    p = ParticleEnsemble.from_arrays(np.full(n, 1.0), v, np.full(n, L / n), device=device)
    grid = Grid(1, L)
    ci = build_cell_index(p, grid)
    sp = torch.as_tensor(s, dtype=torch.float32, device=device).t().contiguous()
    _lib.call("spic_gather_scores", _lib.ptr(sp), n, _lib.ptr(ci.perm), n, 3, _lib.ptr(ci.sw), None,
              _lib.stream_handle())
    U = torch.empty(3, n, dtype=torch.float32, device=device)
    landau_sorted(ci, p, grid, -3.0, U)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        landau_sorted(ci, p, grid, -3.0, U)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    Us = U.double().cpu().numpy().T
    vs = ci.xv[:, 1:4].double().cpu().numpy()
    wU = (L / n) * Us
    mom = float(np.max(np.abs(wU.sum(0))) / (np.max(np.abs(wU)) * n))
    en = abs(float(np.sum((L / n) * np.einsum("ij,ij->i", vs, Us))))
    en /= float(np.sum((L / n) * np.linalg.norm(vs, axis=1) * np.linalg.norm(Us, axis=1)))
    pairs = float(n) * n
    return {"n": n, "ms": ms, "pair_interactions_per_s": pairs / (ms * 1e-3),
            "tflops": pair_flops(pairs, n) / (ms * 1e-3) / 1e12,
            "ordered_equivalent_tflops": FLOP_PER_PAIR * pairs / (ms * 1e-3) / 1e12,
            "momentum_rel": mom, "energy_rel": en}


def l2_flush(buf) -> None:
    """Evict L2 between timed regions: write a 256 MiB buffer (twice L2), then read it back so
    the lines left in L2 are clean — otherwise the timed kernel that follows pays for writing
    back up to 126 MB of the flush's dirty lines."""
    buf.zero_()
    buf.view(-1, 4096).amax(dim=1)


def hbm_peak_gbs() -> float:
    """Measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs); the profiling recipe's fallback
    6650 GB/s only when the driver-written file is absent."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6650.0


def hbm_microbench(torch, device, peak_gbs: float, n: int = 1 << 24, M: int = 1024,
                   reps: int = 5) -> dict:
    """HBM-bound kernels at config-4 size (n = 2^24, M = 1024: 400+ MB of particle state,
    beyond the 126 MB L2): push (interpolate + Lorentz + advance + wrap), binning, deposit.
    Each launch is timed alone with CUDA events after an L2 flush. Algorithmic bytes per
    particle: push 24 (read + write x, v0, v1; the Lorentz step with B = (0, 0, B3) leaves v2
    as it is — SURVEY §8(d) counts 32 with v2), binning 52, deposit 16 (the
    x, v record; uniform weights)."""
    from paper_2603_25832_b200 import _lib
    from paper_2603_25832_b200.collision import auto_sub_cells, build_cell_index
    from paper_2603_25832_b200.pic import Grid, deposit_from_index
    from paper_2603_25832_b200.state import ParticleEnsemble, new_flags

    rng = np.random.default_rng(3)
    L = 4 * math.pi
    p = ParticleEnsemble.from_arrays(rng.uniform(0, L, n).astype(np.float32),
                                     rng.normal(size=(n, 3)).astype(np.float32),
                                     np.full(n, L / n, np.float32), device=device)
    grid = Grid(M, L / M)
    S = auto_sub_cells(n, M)
    E = [torch.zeros(M, dtype=torch.float64, device=device) for _ in range(3)]
    flags = new_flags(device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    ci = build_cell_index(p, grid, S)
    st = _lib.stream_handle()

    def timed(fn):
        out = []
        for _ in range(reps + 1):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
        return statistics.median(out[1:])

    res = {"n": n, "M": M, "sub_cells": S, "l2": "flushed before every timed launch",
           "peak_gbs": peak_gbs}
    for name, fn, bpp in (
            ("push", lambda: _lib.call("spic_push", _lib.ptr(p.x), _lib.ptr(p.vp), n, n, 3,
                                       _lib.ptr(E[0]), _lib.ptr(E[1]), _lib.ptr(E[2]), M,
                                       float(grid.eta), 0.0, _lib.ptr(flags), st), 24),
            ("bin", lambda: build_cell_index(p, grid, S, out=ci), 52),
            ("deposit", lambda: deposit_from_index(ci, p, grid), 16)):
        ms = timed(fn)
        gbs = bpp * n / (ms * 1e-3) / 1e9
        res[name] = {"ms": ms, "bytes_per_particle": bpp, "achieved_gbs": gbs,
                     "frac": gbs / peak_gbs}
    return res


def build_dist_sim(wl: dict, seed: int, device, world: int, host_staged: bool = False):
    """The workload's own problem (n, M, L fixed: strong scaling, as BASELINE configs 3 and 4
    define their 2/4/8-GPU runs) decomposed into cell ranges, one per rank; the ranges are
    balanced on the initial cell counts."""
    from paper_2603_25832_b200.dist_engine import DistSimulation
    from paper_2603_25832_b200.parallel import CellPartition, Comm
    from paper_2603_25832_b200.pic import Grid, deposit
    from paper_2603_25832_b200.run import initial_fields
    from paper_2603_25832_b200.state import ParticleEnsemble

    cfg = make_config(wl, seed)
    rng = np.random.default_rng(seed)
    x, v, w, b3 = sample_workload(wl, cfg, rng)
    grid = Grid(cfg.M, cfg.eta)
    comm = Comm(host_staged=host_staged)
    cell = np.minimum(np.floor(x.astype(np.float32).astype(np.float64) / grid.eta).astype(np.int64) % cfg.M,
                      cfg.M - 1)
    part = CellPartition.balanced(np.bincount(cell, minlength=cfg.M), world)
    lo, hi = part.owned(comm.rank)
    own = np.nonzero((cell >= lo) & (cell < hi))[0]
    # global initial fields from the full ensemble (identical on every rank)
    pfull = ParticleEnsemble.from_arrays(x, v, w, device=device)
    rho, J = deposit(pfull, grid)
    fields = initial_fields(cfg, grid, rho, J)
    if b3 is not None:
        import torch

        fields.B3.copy_(torch.as_tensor(b3, dtype=fields.B3.dtype, device=fields.B3.device))
    del pfull
    est = make_estimator_for(wl, cfg, rng, device, grid)
    sim = DistSimulation(x[own], v[own], w[own], own, fields, grid, dt=cfg.dt, nu=cfg.nu,
                         mode=cfg.mode, gamma=cfg.gamma, estimator=est, comm=comm, partition=part,
                         n_global=cfg.n, max_rows=4)
    return sim


def live_pairs(sim, dist_mode: bool) -> float:
    """Ordered live pairs (|dx| < eta) of this rank's pair kernel. Decomposed runs count the
    rank's own particles only (pairs with the halo cells left out: a slight undercount)."""
    from paper_2603_25832_b200.collision import count_live_pairs

    if not dist_mode:
        return float(count_live_pairs(sim.ci, sim.p, sim.grid))
    if getattr(sim, "ci_own", None) is None:
        return 0.0
    return float(count_live_pairs(sim.ci_own, sim.buf.view(sim.n_own, sim.uniform_w), sim.grid))


def allreduce_max(dist, t, host_staged: bool):
    """MAX over ranks of a small device tensor (host-staged for the gloo test backend)."""
    if host_staged:
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t


def evaluated_pairs(cell_start, sub_start, M: int, S: int, TI: int = 512) -> float:
    """Unordered pairs the antisymmetric kernel evaluates in one launch ("count
    41 FLOP per evaluated unordered pair"): per target tile [t0, t1) of a cell, its forward
    window (the rest of the cell, len1, plus the next cell's prefix through the sub-cell of
    the tile's last record, len2 — the k_sym_tiles rule, landau_sym.cu) and the tile's own
    unordered pairs (the diagonal block, counted once although the kernel evaluates it
    one-sided in both orders). Host numpy on the cell / sub-cell starts; M >= 3."""
    cs = np.asarray(cell_start, dtype=np.int64)
    ss = np.asarray(sub_start, dtype=np.int64) if S > 1 else None
    total = 0.0
    for c in range(M):
        a, e = int(cs[c]), int(cs[c + 1])
        cn = (c + 1) % M
        for t0 in range(a, e, TI):
            t1 = min(t0 + TI, e)
            tl = t1 - t0
            if ss is not None:
                sub = ss[c * S:(c + 1) * S]
                b = int(np.searchsorted(sub, t1 - 1, side="right")) - 1
                len2 = int(ss[cn * S + b + 1] - cs[cn])
            else:
                len2 = int(cs[cn + 1] - cs[cn])
            total += tl * ((e - t1) + len2) + tl * (tl - 1) / 2.0
    return total


def main():
    args = parse_args()
    wl = WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        # bounded: each CPU step is a sampled step (a few seconds on 16 host cores); at most 3
        # timed sample steps and 1 warm-up so any --steps/--warmup finishes in minutes
        reps, warm = min(max(1, args.steps), 3), min(max(0, args.warmup), 1)
        line = cpu_baseline_line(wl, args.seed, reps=reps, warm=warm)
        out = {"metric": METRIC, "value": line["value"], "unit": "particle-steps/s",
               "impl": "reference", "n_gpus": args.gpus, "steps": reps, "warmup": warm,
               "requested_steps": args.steps, "requested_warmup": args.warmup,
               "ms_per_step": 1e3 * line["seconds_per_step"], "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": bench_config(wl, 1),
               "cpu_baseline": {k: line[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                     "extrapolated", "sample_seconds",
                                                     "scale_factors")},
               "extrapolated": True, "sample_seconds": line["sample_seconds"],
               "scale_factors": line["scale_factors"],
               "e2e": {"value": line["value"], "unit": "particle-steps/s",
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
               "pair_interactions_per_s": line["pair_interactions_per_s"],
               "stage_seconds": line["stage_seconds"]}
        print(json.dumps(out))
        return 0

    import torch

    from paper_2603_25832_b200 import _lib
    
    # SPIC_DIST_BACKEND=gloo (test only): every rank on cuda:0 with host-staged collectives, so
    # the multi-rank bench path can be exercised on one GPU (NCCL refuses two ranks per device);
    # its timings are not bench numbers
    backend = os.environ.get("SPIC_DIST_BACKEND", "nccl")
    share_gpu = backend == "gloo"
    if share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    # SPIC_FORCE_DIST=1: the decomposed (NCCL) path even at one rank — a one-GPU check of the
    # multi-GPU bench path (process group, DistSimulation, max-over-ranks timing)
    dist_mode = world > 1 or os.environ.get("SPIC_FORCE_DIST") == "1"
    if dist_mode:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    _lib.load(build_if_missing=False)

    # N = 1: the single-GPU engine. N > 1: the cell-range decomposition of the same problem
    # (strong scaling) over NCCL.
    sim = (build_dist_sim(wl, args.seed, device, world, host_staged=share_gpu) if dist_mode
           else build_sim(wl, args.seed, device))
    n = wl["n"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)

    for _ in range(max(3, args.warmup)):
        sim.step(0)
    torch.cuda.synchronize()
    sim.check()
    # the timed steps replay a CUDA graph of the step (one launch per step; the eager path is
    # identical kernel for kernel, see tests/test_gpu_parity.py::test_cuda_graph_replay_*)
    use_graph = not dist_mode and not os.environ.get("SPIC_NO_GRAPH")
    if use_graph:
        sim.capture(row=3)
    live0 = live_pairs(sim, dist_mode)
    peak = fp32_peak_tflops(torch, _lib)

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sim.time_collision = not use_graph
    sim.collision_events.clear()
    launches0 = _lib.query("spic_launch_count")
    evs = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if use_graph:
                sim.replay(1)
            else:
                sim.step(1)
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
    launches = _lib.query("spic_launch_count") - launches0
    if use_graph:
        # graph replays do not pass through the host launch counter: count the captured
        # kernels of one eager step (same sequence) and time the pair kernel eagerly
        c0 = _lib.query("spic_launch_count")
        sim.time_collision = True
        for _ in range(3):
            sim.step(2)
        torch.cuda.synchronize()
        launches = args.steps * (_lib.query("spic_launch_count") - c0) // 3
    sim.time_collision = False
    sim.check()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    coll_ms = [a.elapsed_time(b) for a, b in sim.collision_events]
    live1 = live_pairs(sim, dist_mode)
    live = 0.5 * (live0 + live1)
    evald = None
    if not dist_mode and not os.environ.get("SPIC_LANDAU_VARIANT") and sim.grid.M >= 3:
        try:
            evald = evaluated_pairs(sim.ci.cell_start.cpu().numpy(), sim.ci.sub_start.cpu().numpy(),
                                    sim.grid.M, sim.S,
                                    TI=int(_lib.query("spic_landau_tile_targets", sim.grid.M)))
        except Exception:  # noqa: BLE001
            evald = None
    t = torch.tensor([total_ms, statistics.mean(coll_ms) if coll_ms else float("nan")],
                     dtype=torch.float64, device=device)
    if dist:
        allreduce_max(dist, t, share_gpu)
        dist.barrier()
    total_ms, coll_avg_ms = float(t[0]), float(t[1])
    value = n * args.steps / (total_ms * 1e-3)  # n = the whole job's particles (strong scaling)

    # end to end through the public host-buffer API
    e2e = None
    if not args.no_e2e and not dist_mode:
        dv = sim.p.dv
        xh = torch.empty(n, dtype=torch.float32).pin_memory()
        vh = torch.empty(dv, n, dtype=torch.float32).pin_memory()
        dh = torch.empty(sim.diag.shape[1], dtype=torch.float64).pin_memory()
        fh = torch.empty(sim.flags.shape[0], dtype=torch.int32).pin_memory()
        xh.copy_(sim.p.x)
        vh.copy_(sim.p.vp)
        torch.cuda.synchronize()
        sim.step_host(2, xh, vh, dh, fh)  # warm
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            sim.step_host(2, xh, vh, dh, fh)
            stream.synchronize()       # the per-step flag read run() does (ref: run.py:107-108)
            sim.check_host(fh.numpy())
        e1.record()
        e1.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
        if dist:
            allreduce_max(dist, te, share_gpu)
        e2e = {"value": n * args.steps / (float(te[0]) * 1e-3), "unit": "particle-steps/s",
               "h2d_bytes_per_step": int(xh.numel() * 4 + vh.numel() * 4),
               "d2h_bytes_per_step": int(xh.numel() * 4 + vh.numel() * 4 + dh.numel() * 8
                                         + fh.numel() * 4),
               "flags_checked_every_step": True}
        sim.check()
    elif not args.no_e2e:
        # decomposed engine: each rank's particles through DistSimulation.step_host. The pinned
        # host buffers are sized from the all-reduced largest rank count plus the most a rank
        # can receive over the timed steps (two boundary messages per step), capped at the
        # whole job — so no rank can fail inside the collective loop on capacity; any other
        # error propagates (torchrun then stops every rank) instead of desynchronising them.
        dv = sim.dv
        nmax = torch.tensor([float(sim.n)], dtype=torch.float64, device=device)
        allreduce_max(dist, nmax, share_gpu)
        cap = int(min(n, int(nmax[0]) + (args.steps + 2) * 2 * (sim.mcap + 1))) + 64
        xh = torch.empty(cap, dtype=torch.float32).pin_memory()
        vh = torch.empty(dv, cap, dtype=torch.float32).pin_memory()
        dh = torch.empty(sim.diag.shape[1], dtype=torch.float64).pin_memory()
        n0 = sim.n
        xh[:n0].copy_(sim.buf.x[:n0])
        vh[:, :n0].copy_(sim.buf.vp[:, :n0])
        torch.cuda.synchronize()
        sim.step_host(2, xh, vh, dh)  # warm
        torch.cuda.synchronize()
        dist.barrier()
        counts = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            counts.append(sim.step_host(2, xh, vh, dh))
        e1.record()
        e1.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
        allreduce_max(dist, te, share_gpu)
        nb = int(statistics.mean(counts)) * 4 * (1 + dv)
        e2e = {"value": n * args.steps / (float(te[0]) * 1e-3),
               "unit": "particle-steps/s", "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb + dh.numel() * 8,
               "note": "per rank: its own particles in and out every step (rank 0's bytes)"}
        sim.check()

    flop_launch = pair_flops(live, n)
    achieved = flop_launch / (coll_avg_ms * 1e-3) / 1e12
    silu_rf = None
    if wl["estimator"] == "sbtm" and wl.get("net") == "silu":
        silu_rf = silu_kernel_roofline(torch, device, sim, wl, args.workload)
        t = torch.tensor([silu_rf["launch_ms"]], dtype=torch.float64, device=device)
        if dist:
            allreduce_max(dist, t, share_gpu)
        silu_rf["launch_ms"] = float(t[0])
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "landau_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(args.workload)
        except Exception:  # noqa: BLE001
            traffic = None
    out = {
        "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded reference sampler; random-init score net, no pretraining)",
        "config": bench_config(wl, world),
        "engine": {"sub_cells": sim.S, "cuda_graph": use_graph, "dist_path": dist_mode,
                   "backend": (backend if dist_mode else None)},
        "pair_interactions_per_s": world * live / (coll_avg_ms * 1e-3),
        "live_pairs_per_step": live,
        "collision_ms": coll_avg_ms,
        "roofline_pair": {"bound": "fp32", "kernel": PAIR_KERNEL,
                          "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                          "frac": achieved / peak, "traffic": traffic,
                          "ordered_equivalent_frac": FLOP_PER_PAIR * live / (coll_avg_ms * 1e-3)
                          / 1e12 / peak,
                          "evaluated_unordered_pairs": evald,
                          "frac_evaluated": (FLOP_PER_UPAIR * evald / (coll_avg_ms * 1e-3) / 1e12
                                             / peak) if evald else None,
                          "flop_per_launch": flop_launch, "launch_ms": coll_avg_ms,
                          "launches_per_step": 1,
                          "peak_source": "measured in-run: spic_fp32_probe (FFMA2 chains, "
                                         "592 CTAs)"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    # `roofline` = the kernel with the largest share of the step: with the SiLU net the K = 10
    # ISM launches (tensor cores) edge out the pair kernel; otherwise the pair kernel
    out["roofline"] = out["roofline_pair"]
    if silu_rf is not None:
        out["roofline_silu"] = silu_rf
        if silu_rf["launch_ms"] * silu_rf["launches_per_step"] > coll_avg_ms:
            out["roofline"] = silu_rf
    if world == 1:
        try:
            mb = config1_microbench(torch, device)
            mb["frac_of_fp32_peak"] = mb["tflops"] / peak
            out["config1_microbench"] = mb
        except Exception as exc:  # noqa: BLE001
            out["config1_microbench"] = {"error": str(exc)}
        try:
            out["hbm_kernels"] = hbm_microbench(torch, device, hbm_peak_gbs())
        except Exception as exc:  # noqa: BLE001
            out["hbm_kernels"] = {"error": str(exc)}
    if world == 1 and args.workload == "c4":
        # BASELINE config 3 (the VML config: Weibel, full Maxwell) in the same run
        try:
            out["config3_vml"] = variant_line(torch, device, WORKLOADS["c3"], args.seed)
            out["config3_vml"]["config"] = bench_config(WORKLOADS["c3"], 1)
        except Exception as exc:  # noqa: BLE001
            out["config3_vml"] = {"error": str(exc)}
    if world == 1 and args.workload == "c4":
        # BASELINE config 4 is to be run "with both the SBTM and the blob estimator"
        try:
            out["config4_blob"] = variant_line(torch, device, WORKLOADS["c4blob"], args.seed)
            out["config4_blob"]["config"] = bench_config(WORKLOADS["c4blob"], 1)
        except Exception as exc:  # noqa: BLE001
            out["config4_blob"] = {"error": str(exc)}
    if world == 1 and args.workload + "ss" in WORKLOADS:
        # the same config with the reference's own softsign network (like-for-like with the
        # reference arm, which has no SiLU network)
        try:
            out["reference_net_variant"] = variant_line(torch, device,
                                                        WORKLOADS[args.workload + "ss"], args.seed)
        except Exception as exc:  # noqa: BLE001
            out["reference_net_variant"] = {"error": str(exc)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line = cpu_baseline_line(wl, args.seed)
            out["cpu_baseline"] = {k: line[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                        "extrapolated", "sample_seconds",
                                                        "scale_factors")}
            out["cpu_baseline"]["pair_interactions_per_s"] = line["pair_interactions_per_s"]
        except Exception as exc:  # noqa: BLE001
            out["cpu_baseline"] = {"error": str(exc)}
    if rank == 0:
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
