"""A/B of the HBM-bound kernels (push, binning, deposit) at config-4 size, one process, each
variant selected by its environment switch (read per call). Prints one JSON object per run.

    python tools/hbm_ab.py SPIC_PUSH_VARIANT=1/2 SPIC_DEP_CFG=1024,4,6/512,4,7
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2603_25832_b200 import _lib

    _lib.load(build_if_missing=False)
    dev = torch.device("cuda", 0)
    sweeps = [a.split("=", 1) for a in sys.argv[1:]] or [["SPIC_PUSH_VARIANT", "2"]]
    peak = bench.hbm_peak_gbs()
    # practical ceilings at the same byte counts (torch's own vectorised elementwise kernels)
    import statistics

    n = 1 << 24
    t = torch.zeros(3, n, device=dev)
    u = torch.zeros(3, n, device=dev)
    r = torch.zeros(4 * n, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn, reps=9):
        out = []
        for _ in range(reps + 1):
            bench.l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
        return statistics.median(out[1:])

    for name, fn, nbytes in (("inplace_add_24B", lambda: t.add_(1.0), 24 * n),
                             ("copy_12B_to_12B", lambda: u.copy_(t), 24 * n),
                             ("read_16B_sum", lambda: r.sum(), 16 * n)):
        ms = timed(fn)
        print(json.dumps({"ceiling": name, "ms": ms, "gbs": nbytes / (ms * 1e-3) / 1e9,
                          "frac": nbytes / (ms * 1e-3) / 1e9 / peak}), flush=True)
    for key, vals in sweeps:
        for val in vals.split("/"):
            os.environ[key] = val
            r = bench.hbm_microbench(torch, dev, peak, reps=9)
            print(json.dumps({key: val, **{k: r[k] for k in ("push", "bin", "deposit")}}),
                  flush=True)
            del os.environ[key]


if __name__ == "__main__":
    main()
