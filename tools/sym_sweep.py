"""Time the antisymmetric pair kernel configurations (SPIC_SYM_CFG) and the ordered kernel on
one workload's cell-sorted records (CUDA events, warm). Prints one JSON object.

    python tools/sym_sweep.py [--workload c2ss] [--cfgs 0,1,2,3,4] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2603_25832_b200 import _lib
    from paper_2603_25832_b200.collision import landau_sorted

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2ss")
    ap.add_argument("--cfgs", default="0,5,6,7,8")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload]
    dev = torch.device("cuda", 0)
    _lib.load(build_if_missing=False)
    sim = bench.build_sim(wl, 0, dev)
    for _ in range(2):
        sim.step(0)
    torch.cuda.synchronize()
    p, g, ci = sim.p, sim.grid, sim.ci

    def timeit(env):
        os.environ.pop("SPIC_SYM_CFG", None)
        os.environ.pop("SPIC_LANDAU_VARIANT", None)
        os.environ.update(env)
        U = torch.empty(3, p.n, dtype=torch.float32, device=dev)
        landau_sorted(ci, p, g, sim.gamma, U)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            landau_sorted(ci, p, g, sim.gamma, U)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / args.reps, U

    out = {"workload": wl["workload"]}
    ms, Uo = timeit({"SPIC_LANDAU_VARIANT": "o"})
    out["ordered_ms"] = ms
    for c in args.cfgs.split(","):
        ms, U = timeit({"SPIC_SYM_CFG": c})
        err = float((U - Uo).norm() / Uo.norm())
        out[f"sym{c}_ms"] = ms
        out[f"sym{c}_relerr_vs_ordered"] = err
    print(json.dumps(out))


if __name__ == "__main__":
    main()
