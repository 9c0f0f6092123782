"""Per-op device timings (CUDA events, warm, averaged) of the step engine's kernels at one
workload; used to iterate on individual kernels. Prints one JSON object.

    python tools/bench_kernels.py [--workload c2] [--reps 20]
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
    from paper_2603_25832_b200.collision import build_cell_index, landau_sorted
    from paper_2603_25832_b200.pic import FIELD_VPL, deposit_from_index

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload]
    dev = torch.device("cuda", 0)
    _lib.load(build_if_missing=False)
    sim = bench.build_sim(wl, 0, dev)
    for _ in range(3):
        sim.step(0)
    torch.cuda.synchronize()
    p, g, ci = sim.p, sim.grid, sim.ci
    n = p.n
    st = _lib.stream_handle()

    def timeit(fn, reps=args.reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {}
    out["push_ms"] = timeit(lambda: _lib.call(
        "spic_push", _lib.ptr(p.x), _lib.ptr(p.vp), n, n, p.dv, _lib.ptr(sim.f.E1), _lib.ptr(sim.f.E2),
        _lib.ptr(sim.f.B3), g.M, float(g.eta), 0.0, _lib.ptr(sim.flags), st))
    out["bin_ms"] = timeit(lambda: build_cell_index(p, g, sim.S, out=ci))
    out["deposit_field_ms"] = timeit(lambda: deposit_from_index(
        ci, p, g, fields=sim.f, field_mode=FIELD_VPL, dt=0.0, diag_out=sim.diag[3, 0:3], flags=sim.flags))
    if sim.trainer is not None and getattr(sim.trainer.net, "arch", "") == "silu":
        from paper_2603_25832_b200.silu_net import _silu_partials

        tr = sim.trainer
        out["ism_partials_ms"] = timeit(lambda: _silu_partials(tr.net, ci.xv, ci.sw, n, tr.L))
        out["forward_ms"] = timeit(lambda: sim.est.estimate_sorted(ci, n))
        out["sbtm_update_K_ms"] = timeit(lambda: tr.run(n, ci=ci, flags=sim.flags), reps=3)
    elif sim.trainer is not None:
        from paper_2603_25832_b200.score import DIV_EXACT, _finalize, _partials

        net, tr = sim.trainer.net, sim.trainer
        holder = {}

        def part():
            holder["buf"] = _partials(net, DIV_EXACT, n=n, x_scale=1.0 / tr.L, xv=ci.xv, sw=ci.sw)

        out["ism_partials_ms"] = timeit(part)
        out["ism_finalize_ms"] = timeit(lambda: _finalize(net, holder["buf"], n, DIV_EXACT, opt=tr.opt,
                                                          reset_lr=True, apply_step=False))
        out["mlp_forward_ms"] = timeit(lambda: sim.est.estimate_sorted(ci, n))
        out["sbtm_update_K_ms"] = timeit(lambda: tr.run(n, ci=ci, flags=sim.flags), reps=3)
    else:
        from paper_2603_25832_b200.score import blob_sorted

        out["blob_ms"] = timeit(lambda: blob_sorted(ci, p, g, sim.est.bandwidth, sim.flags,
                                                    sim.bad_pid, sim.h_cell), reps=5)
    out["landau_ms"] = timeit(lambda: landau_sorted(ci, p, g, sim.gamma, sim.U_sorted,
                                                    nsplit=sim.opt.landau_split), reps=5)
    out["step_ms"] = timeit(lambda: sim.step(1), reps=5)
    out["workload"] = wl["workload"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
