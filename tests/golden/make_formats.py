"""Byte-level fixtures of the reference's on-disk formats, written by the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_formats.py

For one seeded state it runs scorepic's own writers — write_diagnostics_csv, write_snapshot
(+ JSON sidecar), save_checkpoint, write_manifest — and stores the inputs and the produced
bytes in tests/golden/formats.npz (particle values are float32-exact so the float32 device
state reproduces them). Nothing here is imported at test time.
"""

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from scorepic import diagnostics, score  # noqa: E402
from scorepic.config import build_config, write_manifest  # noqa: E402
from scorepic.state import DiagnosticsRecord, FieldState, ParticleEnsemble  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(2603)
    n, dv, M = 37, 3, 8
    L = 2.0
    x = rng.uniform(0, L, n).astype(np.float32).astype(np.float64)
    v = rng.normal(size=(n, dv)).astype(np.float32).astype(np.float64)
    w = np.full(n, L / n, dtype=np.float32).astype(np.float64)
    E1, E2, B3 = rng.normal(size=(3, M))
    p = ParticleEnsemble(x=x, v=v, w=w)
    f = FieldState(E1=E1, E2=E2, B3=B3, rho=np.zeros(M), J=np.zeros((dv, M)), rho_ion=0.0)
    recs = []
    for k in range(4):
        vals = rng.normal(size=7) * 10.0 ** rng.integers(-12, 6, size=7)
        recs.append(DiagnosticsRecord(step=k, t=0.05 * k, E_K=vals[0], E_E=vals[1], E_B=vals[2],
                                      E_total=vals[0] + vals[1] + vals[2], H_dot=vals[3],
                                      P=vals[4:7].copy(), E_l2=abs(vals[1]) ** 0.5))
    rec_arr = np.array([[r.step, r.t, r.E_K, r.E_E, r.E_B, r.E_total, r.H_dot, *r.P, r.E_l2]
                        for r in recs])
    net = score.MlpScoreNet.init_glorot(dv, 16, rng)
    net.b1[:] = rng.normal(size=net.b1.shape)
    net.b2[:] = rng.normal(size=net.b2.shape)
    cfg = build_config(overrides=dict(preset="weibel", n=4096, M=16, dt=0.05, t_final=0.25,
                                      seed=11))
    with tempfile.TemporaryDirectory() as d:
        diagnostics.write_diagnostics_csv(recs, os.path.join(d, "diagnostics.csv"))
        diagnostics.write_snapshot(p, f, 3, 0.15, os.path.join(d, "snap.bin"), config=cfg)
        score.save_checkpoint(net, os.path.join(d, "net.sbtm"))
        write_manifest(cfg, d, ["a warning"])

        def rd(name):
            with open(os.path.join(d, name), "rb") as fh:
                return np.frombuffer(fh.read(), dtype=np.uint8)

        out = dict(x=x, v=v, w=w, E1=E1, E2=E2, B3=B3, records=rec_arr,
                   W1=net.W1, b1=net.b1, W2=net.W2, b2=net.b2,
                   csv=rd("diagnostics.csv"), snap=rd("snap.bin"), snap_json=rd("snap.bin.json"),
                   ckpt=rd("net.sbtm"), manifest=rd("manifest.json"))
    np.savez_compressed(os.path.join(OUT, "formats.npz"), **out)
    print("wrote", os.path.join(OUT, "formats.npz"))


if __name__ == "__main__":
    main()
