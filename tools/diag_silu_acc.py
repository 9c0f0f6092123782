"""Diagnostic: SiLU ISM gradient accuracy vs accumulation length and data (config 3)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from test_gpu_parity_at_size import bench_ensemble, _silu_oracle_chunked, f32, relL2
from oracle import silu_oracle as so
from paper_2603_25832_b200 import _lib
from paper_2603_25832_b200.silu_net import SiluScoreNet, silu_ism_loss_and_grad
_lib.load()
for tag in ("c3", "c2"):
    x, v, w, wl = bench_ensemble(tag)
    L = wl["L"]
    rng = np.random.default_rng(5)
    params = so.glorot(128, rng)
    params[4 * 128:5 * 128] = rng.normal(0, 0.3, 128)
    params[-3:] = rng.normal(0, 0.3, 3)
    params = f32(params)
    net = SiluScoreNet(); net.set_flat(params)
    n = x.shape[0]
    for parts in (1, 4, 16):
        g = 0
        for k in range(parts):
            a, b = k * n // parts, (k + 1) * n // parts
            _, gk = silu_ism_loss_and_grad(net, x[a:b], v[a:b], w[a:b], L)
            g = g + gk.cpu().numpy()
        if parts == 1:
            rl, rg = _silu_oracle_chunked(params, x, v, w, L)
        sl = net._slices()
        out = []
        for (a, b, _), name in zip(sl, ("W1", "b1", "W2", "b2", "W3", "b3")):
            out.append(f"{name} {relL2(g[a:b], rg[a:b]):.2e}")
        a, b, _ = sl[0]
        W1g, W1r = g[a:b].reshape(128, 4), rg[a:b].reshape(128, 4)
        cols = " ".join(f"{relL2(W1g[:, c], W1r[:, c]):.2e}(|{np.linalg.norm(W1r[:, c]):.2e}|)" for c in range(4))
        print(f"{tag} n={n} parts={parts}: " + ", ".join(out) + f" | W1 cols {cols}", flush=True)
