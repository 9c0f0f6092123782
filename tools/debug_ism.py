import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2603_25832_b200 import _lib
from paper_2603_25832_b200.score import MlpScoreNet, ism_loss_and_grad, _partials, DIV_EXACT, _vec, _planes
g = np.load("tests/golden/mlp_ism.npz")
for k in range(4):
    p = f"c{k}_"
    W1 = g[p+"W1"]; H = W1.shape[0]; dv = g[p+"W2"].shape[0]
    net = MlpScoreNet(dv, H)
    net.set_params([g[p+"W1"], g[p+"b1"], g[p+"W2"], g[p+"b2"]])
    x, v, w = g[p+"x"], g[p+"v"], g[p+"w"]
    loss, grads = ism_loss_and_grad(net, x, v, w, divergence="exact")
    n = len(x)
    buf = _partials(net, DIV_EXACT, n=n, x_scale=1.0, x=_vec(x, "cuda"), vp=_planes(v, "cuda"), w=_vec(w, "cuda"), ldz=n)
    rows = buf.view(torch.float64)
    width = 1 + net.n_params + H
    off = int(_lib.query("spic_ism_row_offset", n, H, dv)) // 8
    print(k, "H", H, "n", n, "loss", loss, "ref", float(g[p+"exact_loss"]), "row0 loss", float(rows[0]), "reduced", float(rows[off]), "nblk", off // width)
