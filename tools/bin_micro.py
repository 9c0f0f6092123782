"""Binning alone at config-4 size (n = 2^24, M = 1024, S = 16) for launch-list profiling."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import math  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_25832_b200 import _lib  # noqa: E402
from paper_2603_25832_b200.collision import auto_sub_cells, build_cell_index  # noqa: E402
from paper_2603_25832_b200.pic import Grid  # noqa: E402
from paper_2603_25832_b200.state import ParticleEnsemble  # noqa: E402

_lib.load()
n, M = 1 << 24, 1024
rng = np.random.default_rng(3)
L = 4 * math.pi
dev = torch.device("cuda", 0)
p = ParticleEnsemble.from_arrays(rng.uniform(0, L, n).astype(np.float32),
                                 rng.normal(size=(n, 3)).astype(np.float32),
                                 np.full(n, L / n, np.float32), device=dev)
g = Grid(M, L / M)
S = auto_sub_cells(n, M)
ci = build_cell_index(p, g, S)
for _ in range(3):
    build_cell_index(p, g, S, out=ci)
torch.cuda.synchronize()
print("ok", S)
