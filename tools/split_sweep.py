import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2603_25832_b200 import _lib
from paper_2603_25832_b200.collision import landau_sorted
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dev = torch.device("cuda", 0)
_lib.load(build_if_missing=False)
sim = bench.build_sim(wl, 0, dev)
for _ in range(3): sim.step(0)
torch.cuda.synchronize()
out = {}
for ns in [0, 1, 2, 3, 4, 5, 6, 8, 10, 12, 16]:
    landau_sorted(sim.ci, sim.p, sim.grid, -3.0, sim.U_sorted, nsplit=ns)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): landau_sorted(sim.ci, sim.p, sim.grid, -3.0, sim.U_sorted, nsplit=ns)
    e1.record(); e1.synchronize()
    out[ns] = e0.elapsed_time(e1) / 5
print(json.dumps(out))
