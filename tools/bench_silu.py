"""Device timings of the SiLU score network kernels (extension M1) at config-0 and config-2
particle counts: ISM partials (+ fixed-order reduction), finalize, forward. Prints one JSON
object per size with the tensor-pipe throughput of the hidden GEMMs.

    python tools/bench_silu.py [--reps 20]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# per particle per ISM step: G1, G2, G3 with two 128 x 128 products each (primal + divergence)
GEMM_FLOP_PER_PARTICLE = 3 * 2 * (2 * 128 * 128)
SPLIT_PASSES = 3  # hi*hi + hi*lo + lo*hi


def main():
    import numpy as np
    import torch

    from paper_2603_25832_b200 import _lib
    from paper_2603_25832_b200.score import AdamW
    from paper_2603_25832_b200.silu_net import (SiluScoreNet, _silu_finalize, _silu_partials,
                                                records)

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--sizes", default="65536,1048576")
    args = ap.parse_args()
    _lib.load(build_if_missing=False)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bf16_peak = float(peaks["bf16_tflops"])
    dev = torch.device("cuda", 0)
    for n in (int(a) for a in args.sizes.split(",")):
        L = 4 * math.pi if n <= 65536 else 10 * math.pi
        rng = np.random.default_rng(0)
        net = SiluScoreNet.init_glorot(rng, device=dev)
        x = rng.uniform(0, L, n)
        v = rng.normal(size=(n, 3))
        xv, sw = records(x, v, np.full(n, L / n), L, dev)
        opt = AdamW(lr=1e-3, weight_decay=0.0, device=dev)

        def timeit(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                fn()
            e1.record()
            e1.synchronize()
            return e0.elapsed_time(e1) / args.reps

        holder = {}

        def part():
            holder["b"] = _silu_partials(net, xv, sw, n, L)

        t_part = timeit(part)
        t_fin = timeit(lambda: _silu_finalize(net, holder["b"], n, opt, apply_step=True))
        out = sw.clone()
        t_fwd = timeit(lambda: _lib.call("spic_silu_forward", _lib.ptr(net.params32), 128,
                                         _lib.ptr(xv), _lib.ptr(sw), n, float(1 / L),
                                         _lib.ptr(out), _lib.stream_handle()))
        alg = GEMM_FLOP_PER_PARTICLE * n / (t_part * 1e-3) / 1e12
        print(json.dumps({
            "n": n, "ism_partials_ms": t_part, "finalize_ms": t_fin, "forward_ms": t_fwd,
            "ism_step_ms": t_part + t_fin,
            "gemm_tflops_algorithmic": alg,
            "tensor_bf16_tflops": alg * SPLIT_PASSES,
            "tensor_frac_of_bf16_peak": alg * SPLIT_PASSES / bf16_peak,
            "bf16_peak_tflops": bf16_peak,
        }))


if __name__ == "__main__":
    main()
