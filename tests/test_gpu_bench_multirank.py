"""The multi-rank path of bench.py (what the driver launches under torchrun for N > 1) run end to
end at world size 2 and 3 on the one GPU of this pool: SPIC_DIST_BACKEND=gloo puts every rank
on cuda:0 with host-staged collectives (NCCL refuses two ranks per device), everything else —
cell-range decomposition of the same n, DistSimulation steps, max-over-ranks timing, the
per-rank host-buffer e2e loop, rank 0's single JSON line — is the production path. Timings of
this mode are not bench numbers; the test checks that the path completes and reports."""

import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_bench_multirank_path_completes(world):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, SPIC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_free_port()), "bench.py", "--gpus", str(world), "--workload", "c0",
           "--steps", "2", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == world and out["value"] > 0 and out["scaling"] == "strong"
    assert out["engine"]["dist_path"] and out["engine"]["backend"] == "gloo"
    assert out["gpu_launches"] > 0
    assert out["e2e"] and out["e2e"].get("value", 0) > 0, out["e2e"]
    assert out["config"]["n"] == 65536
