"""The BASELINE "2 x 128 SiLU" score network (extension M1) on the B200 tensor cores.

BASELINE configs 0 and 2 name the score MLP "(x, v) in R^4 -> 2 x 128 SiLU -> R^3"; the
reference itself ships only the one-hidden-layer softsign net (ref: score.py:38-71). This
module adds the deeper network behind the same estimator plug-in surface (estimate / update /
warnings, ref: score.py:591-623) and the same device training loop contract as SbtmTrainer,
so the step engines and run() drive either network. Kernels: spic_silu_forward,
spic_silu_ism_partials (tcgen05 split-BF16 hidden GEMMs), spic_silu_mse_partials
(pretraining), spic_silu_finalize (AdamW with the reference's restore-and-halve recovery).
Only the exact divergence is supported.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .collision import CellIndex
from .score import DIV_EXACT, AdamW, SbtmEstimator, _planes, _vec
from .state import ParticleEnsemble, new_flags

SILU_HIDDEN = 128


class SiluScoreNet:
    """Flat float64 master parameters W1[H][4], b1[H], W2[H][H], b2[H], W3[3][H], b3[3] on
    device plus the float32 working copy the kernels read."""

    arch = "silu"

    def __init__(self, dv: int = 3, hidden: int = SILU_HIDDEN, device=None):
        if dv != 3 or hidden != SILU_HIDDEN:
            raise ValueError(f"the SiLU network needs dv = 3 and hidden = {SILU_HIDDEN}")
        self.dv, self.hidden = dv, hidden
        dev = device or _lib.require_cuda()
        P = int(_lib.query("spic_silu_num_params", hidden))
        self.params64 = torch.zeros(P, dtype=torch.float64, device=dev)
        self.params32 = torch.zeros(P, dtype=torch.float32, device=dev)

    def _slices(self):
        H = self.hidden
        shapes = ((H, 4), (H,), (H, H), (H,), (3, H), (3,))
        out, o = [], 0
        for sh in shapes:
            k = int(np.prod(sh))
            out.append((o, o + k, sh))
            o += k
        return tuple(out)

    def params(self) -> list:
        return [self.params64[a:b].view(*shape) for a, b, shape in self._slices()]

    def set_flat(self, flat) -> None:
        t = torch.as_tensor(np.asarray(flat) if not isinstance(flat, torch.Tensor) else flat,
                            dtype=torch.float64, device=self.params64.device)
        self.params64.copy_(t.reshape(-1))
        self.refresh32()

    def refresh32(self) -> None:
        self.params32.copy_(self.params64)

    @classmethod
    def init_glorot(cls, rng: np.random.Generator, device=None) -> "SiluScoreNet":
        """Glorot-uniform W1, W2, W3 (drawn in that order from `rng`), zero biases."""
        net = cls(device=device)
        H = net.hidden
        parts = []
        for fan_out, fan_in in ((H, 4), (H, H), (3, H)):
            lim = np.sqrt(6.0 / (fan_in + fan_out))
            parts.append(rng.uniform(-lim, lim, size=(fan_out, fan_in)))
        flat = np.concatenate([parts[0].ravel(), np.zeros(H), parts[1].ravel(), np.zeros(H),
                               parts[2].ravel(), np.zeros(3)])
        net.set_flat(flat)
        return net

    @property
    def n_params(self) -> int:
        return int(self.params64.numel())

    def numpy_params(self) -> np.ndarray:
        return self.params64.cpu().numpy().copy()


def records(x, v, w, L: float, dev):
    """(xv, sw) float4 records of pid-order arrays (the kernels' input format)."""
    vp = _planes(v, dev)
    n = vp.shape[1]
    xs = _vec(x, dev, n)
    ws = _vec(w, dev, n) if w is not None else torch.zeros(n, dtype=torch.float32, device=dev)
    xv = torch.stack([xs, vp[0], vp[1], vp[2]], dim=1).contiguous()
    sw = torch.zeros(n, 4, dtype=torch.float32, device=dev)
    sw[:, 3] = ws
    return xv, sw


def silu_forward(net: SiluScoreNet, x, v, L: float) -> torch.Tensor:
    """Scores (n, 3) at positions x in [0, L) and velocities v (n, 3)."""
    dev = net.params32.device
    xv, sw = records(x, v, None, L, dev)
    n = xv.shape[0]
    _lib.call("spic_silu_forward", _lib.ptr(net.params32), net.hidden, _lib.ptr(xv), _lib.ptr(sw),
              n, float(1.0 / L), _lib.ptr(sw), _lib.stream_handle())
    return sw[:, :3]


def _silu_partials(net: SiluScoreNet, xv, sw, n: int, L: float):
    buf, nb = _lib.scratch("silu", _lib.query("spic_silu_scratch_bytes", n))
    _lib.call("spic_silu_ism_partials", _lib.ptr(net.params32), net.hidden, _lib.ptr(xv),
              _lib.ptr(sw), n, float(1.0 / L), _lib.ptr(buf), nb, _lib.stream_handle())
    return buf


def _silu_mse_partials(net: SiluScoreNet, n: int, *, x, vp, w, Z, ldz: int, idx=None,
                       inv_wsum: float, ldv: int, x_scale: float = 1.0):
    buf, nb = _lib.scratch("silu", _lib.query("spic_silu_scratch_bytes", n))
    _lib.call("spic_silu_mse_partials", _lib.ptr(net.params32), net.hidden, _lib.ptr(x),
              _lib.ptr(vp), ldv, _lib.ptr(w), n, float(x_scale), _lib.ptr(Z), ldz, _lib.ptr(idx),
              float(inv_wsum), _lib.ptr(buf), nb, _lib.stream_handle())
    return buf


def _silu_finalize(net: SiluScoreNet, buf, n: int, opt: AdamW, *, reset_lr=False,
                   apply_step=False, grads_out=None, loss_out=None, flags=None, mse=False):
    opt._ensure(net.n_params)
    _lib.call("spic_silu_finalize", _lib.ptr(buf), n, net.hidden, int(mse), _lib.ptr(net.params64),
              _lib.ptr(opt.m), _lib.ptr(opt.v), _lib.ptr(opt.state), float(opt.betas[0]),
              float(opt.betas[1]), float(opt.eps), float(opt.weight_decay), int(reset_lr),
              int(apply_step), _lib.ptr(net.params32), _lib.ptr(grads_out), _lib.ptr(loss_out),
              _lib.ptr(flags), _lib.stream_handle())


def silu_ism_loss_and_grad(net: SiluScoreNet, x, v, w, L: float):
    """(loss, flat float64 grads) of sum_p w_p (|s_p|^2 + 2 div_p), exact divergence."""
    dev = net.params64.device
    xv, sw = records(x, v, w, L, dev)
    n = xv.shape[0]
    buf = _silu_partials(net, xv, sw, n, L)
    g = torch.empty(net.n_params, dtype=torch.float64, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    _silu_finalize(net, buf, n, AdamW(device=dev), grads_out=g, loss_out=loss)
    lv = float(loss.item())
    if not np.isfinite(lv):
        raise RuntimeError("training divergence")
    return lv, g


class SiluTrainer:
    """K exact-divergence ISM steps on device (same contract as score.SbtmTrainer.run)."""

    def __init__(self, net: SiluScoreNet, optimizer: AdamW, K: int, L: float):
        self.net, self.opt, self.K, self.L = net, optimizer, K, L
        dev = net.params64.device
        self.losses = torch.zeros(max(K, 1), dtype=torch.float64, device=dev)
        optimizer._ensure(net.n_params)
        self._z_free = torch.cuda.Event() if torch.cuda.is_available() else None

    def mode(self) -> int:
        return DIV_EXACT

    def draw_shared_probes(self) -> None:  # exact divergence draws nothing
        return None

    def run(self, n: int, *, ci: CellIndex | None = None, particles: ParticleEnsemble | None = None,
            flags=None, reduce_row=None, gid=None, n_global: int | None = None,
            draw: bool = True) -> None:
        if ci is not None:
            xv, sw = ci.xv, ci.sw
        else:
            xv, sw = records(particles.x, particles.v, particles.w, self.L,
                             self.net.params32.device)
        for k in range(self.K):
            buf = _silu_partials(self.net, xv, sw, n, self.L)
            if reduce_row is not None:
                off = int(_lib.query("spic_silu_row_offset", n)) // 8
                reduce_row(buf.view(torch.float64)[off:off + 1 + self.net.n_params])
            _silu_finalize(self.net, buf, n, self.opt, reset_lr=(k == 0), apply_step=True,
                           loss_out=self.losses[k:k + 1], flags=flags)


class SiluEstimator(SbtmEstimator):
    """SBTM estimator over the SiLU network (exact divergence only)."""

    def __init__(self, net: SiluScoreNet, L: float, K: int, rng: np.random.Generator, *,
                 lr: float = 2e-4, weight_decay: float = 1e-4, divergence: str = "exact",
                 rademacher: str = "shared"):
        if divergence != "exact":
            raise ValueError("the SiLU network supports divergence = 'exact' only")
        super().__init__(net, L, K, rng, lr=lr, weight_decay=weight_decay,
                         divergence=divergence, rademacher=rademacher)

    def make_trainer(self) -> SiluTrainer:
        return SiluTrainer(self.net, self.optimizer, self.K, self.L)

    def estimate(self, particles: ParticleEnsemble, cell_index=None) -> torch.Tensor:
        return silu_forward(self.net, particles.x, particles.v, self.L)

    def estimate_sorted(self, ci: CellIndex, n: int) -> None:
        _lib.call("spic_silu_forward", _lib.ptr(self.net.params32), self.net.hidden,
                  _lib.ptr(ci.xv), _lib.ptr(ci.sw), n, float(1.0 / self.L), _lib.ptr(ci.sw),
                  _lib.stream_handle())

    def update(self, particles: ParticleEnsemble, cell_index=None) -> None:
        flags = new_flags(self.net.params64.device)
        tr = self.make_trainer()
        tr.run(particles.n, ci=cell_index, particles=particles, flags=flags)
        f = flags.cpu().numpy()
        lr = self.optimizer.lr
        for _ in range(int(f[_lib.FLAG_LR_HALVINGS])):
            lr *= 0.5
            self.warnings.append(f"training divergence: learning rate halved to {lr:g}")
        if f[_lib.FLAG_TRAIN_FATAL]:
            raise RuntimeError("training divergence")

    # pretrain: inherited; score.pretrain dispatches to the SiLU MSE kernels for this net
