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
    for key, vals in sweeps:
        for val in vals.split("/"):
            os.environ[key] = val
            r = bench.hbm_microbench(torch, dev, peak, reps=9)
            print(json.dumps({key: val, **{k: r[k] for k in ("push", "bin", "deposit")}}),
                  flush=True)
            del os.environ[key]


if __name__ == "__main__":
    main()
