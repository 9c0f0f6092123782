"""Full-length runs of the BASELINE configurations on one GPU (the step counts BASELINE.json
names: config 0 100 steps, config 2 400, config 3 500), graph-replayed engine steps with the
diagnostics row of every step kept on device, then read once. Reports the conservation and
field-energy traces the north star asks for at the bench sizes:

  * energy: max_t |E_total(t) / E_total(0) - 1| (collisions conserve energy; the PIC scheme's
    own drift and float32 rounding remain)
  * momentum: VPL — P_y, P_z drift relative to sum w|v| (no force on them); VML — all three
  * field energy: E_E (VPL) / E_B (VML) at t = 0, its maximum and when, and at the end
    (the instability growth / Landau damping trace)
  * entropy production H_dot: min over the run (>= 0 for a dissipative collision operator)

    python tools/long_run.py [--workloads c0,c2,c3] > profiles/r2_long_runs.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STEPS = {"c0": 100, "c2": 400, "c3": 500, "c0ss": 100, "c2ss": 400}


def main():
    import numpy as np
    import torch

    import bench
    from paper_2603_25832_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="c0,c2,c3")
    args = ap.parse_args()
    _lib.load(build_if_missing=False)
    dev = torch.device("cuda", 0)
    out = []
    for key in args.workloads.split(","):
        wl = bench.WORKLOADS[key]
        steps = STEPS[key]
        sim = bench.build_sim(wl, 0, dev)
        sim.diag = torch.zeros(steps + 1, sim.diag.shape[1], dtype=torch.float64, device=dev)
        p = sim.p
        w = p.w.double()
        v0 = p.vp.double()
        E_K0 = float(0.5 * (w * (v0 * v0).sum(0)).sum())
        E1 = sim.f.E1.double()
        E2, B3 = sim.f.E2.double(), sim.f.B3.double()
        eta = sim.grid.eta
        E_E0 = float(0.5 * eta * (E1 * E1).sum())
        E_B0 = float(0.5 * eta * ((E2 * E2).sum() + (B3 * B3).sum())) if wl["mode"] == "VML" else 0.0
        P0 = (w * v0).sum(1).cpu().numpy()
        pscale = float((w * v0.norm(dim=0)).sum())
        sim.step(1)  # eager first step (sizes scratch), then graph replays into rows 2..steps
        torch.cuda.synchronize()
        sim.check()
        sim.capture(row=0)
        t0 = time.perf_counter()
        for k in range(2, steps + 1):
            sim.replay(k)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        sim.check()
        D = sim.diag[1:steps + 1].cpu().numpy()
        E_tot0 = E_K0 + E_E0 + E_B0
        E_tot = D[:, 4] + D[:, 0] + D[:, 1]
        drift = np.abs(E_tot / E_tot0 - 1.0)
        P = D[:, 5:8]
        field = D[:, 1] if wl["mode"] == "VML" else D[:, 0]
        k_max = int(np.argmax(field))
        out.append({
            "workload": wl["workload"], "steps": steps, "dt": wl["dt"], "n": wl["n"],
            "net": bench.NET_LABEL[wl.get("net", "softsign")],
            "wall_s_graph_replays": wall,
            "energy_drift_max": float(drift.max()), "energy_drift_end": float(drift[-1]),
            "momentum_drift_max_rel": ({"P_y": float(np.abs(P[:, 1] - P0[1]).max() / pscale),
                                        "P_z": float(np.abs(P[:, 2] - P0[2]).max() / pscale)}
                                       if wl["mode"] == "VPL" else
                                       {c: float(np.abs(P[:, i] - P0[i]).max() / pscale)
                                        for i, c in enumerate(("P_x", "P_y", "P_z"))}),
            "field_energy": {"kind": "E_B" if wl["mode"] == "VML" else "E_E",
                             "t0": E_B0 if wl["mode"] == "VML" else E_E0,
                             "max": float(field[k_max]), "t_max": (k_max + 1) * wl["dt"],
                             "end": float(field[-1]),
                             "trace_every_10": [float(a) for a in field[::10]]},
            "H_dot_min": float(D[:, 3].min()), "H_dot_end": float(D[-1, 3]),
        })
        print(json.dumps(out[-1]), flush=True)
        del sim
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
