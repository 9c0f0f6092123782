"""Velocity-score estimators on the B200: SBTM network + ISM training, and the blob KDE.

Operator/plug-in API of the reference (ref: score.py:34-623) over device kernels:
  * MlpScoreNet: flat float64 master parameters on device (W1, b1, W2, b2 are views) plus a
    float32 working copy the kernels read.
  * ism_loss_and_grad / mse_loss_and_grad: spic_ism_partials_ex + spic_sbtm_finalize_ex.
  * sbtm_update: K device steps (partials -> finalize with AdamW and restore-and-halve).
  * blob_score: spic_blob (per-cell Silverman bandwidth or a fixed one).
Rademacher probes and pretraining minibatch permutations are drawn from the run's host
PCG64 stream in the reference's order (bit-identical draws), then uploaded.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .collision import CellIndex, build_cell_index
from .pic import Grid, raise_for_flags
from .state import ParticleEnsemble, new_flags

DIV_EXACT, DIV_SHARED, DIV_PER_PARTICLE, DIV_MSE = 0, 1, 2, 3


def softsign(z):
    return z / (1.0 + abs(z))


class MlpScoreNet:
    """s(u) = W2 softsign(W1 u + b1) + b2, u = [x; v] (ref: score.py:38-71)."""

    def __init__(self, dv: int, hidden: int, device=None):
        self.dv, self.hidden = dv, hidden
        dev = device or _lib.require_cuda()
        P = int(_lib.query("spic_mlp_num_params", hidden, dv))
        self.params64 = torch.zeros(P, dtype=torch.float64, device=dev)
        self.params32 = torch.zeros(P, dtype=torch.float32, device=dev)

    # flat layout W1[H][1+dv], b1[H], W2[dv][H], b2[dv]
    def _slices(self):
        H, dv = self.hidden, self.dv
        o1 = H * (1 + dv)
        o2 = o1 + H
        o3 = o2 + dv * H
        return ((0, o1, (H, 1 + dv)), (o1, o2, (H,)), (o2, o3, (dv, H)), (o3, o3 + dv, (dv,)))

    def params(self) -> list:
        return [self.params64[a:b].view(*shape) for a, b, shape in self._slices()]

    def _set(self, i: int, value) -> None:
        a, b, shape = self._slices()[i]
        t = torch.as_tensor(np.asarray(value) if not isinstance(value, torch.Tensor) else value,
                            dtype=torch.float64, device=self.params64.device)
        self.params64[a:b].copy_(t.reshape(-1))
        self.refresh32()

    W1 = property(lambda self: self.params()[0], lambda self, v: self._set(0, v))
    b1 = property(lambda self: self.params()[1], lambda self, v: self._set(1, v))
    W2 = property(lambda self: self.params()[2], lambda self, v: self._set(2, v))
    b2 = property(lambda self: self.params()[3], lambda self, v: self._set(3, v))

    def refresh32(self) -> None:
        self.params32.copy_(self.params64)

    @classmethod
    def init_glorot(cls, dv: int, hidden: int, rng: np.random.Generator,
                    device=None) -> "MlpScoreNet":
        """Glorot-uniform W1 then W2 from `rng`, zero biases (same draws as score.py:50-58)."""
        net = cls(dv, hidden, device)
        d_in = 1 + dv
        lim1 = np.sqrt(6.0 / (d_in + hidden))
        lim2 = np.sqrt(6.0 / (hidden + dv))
        net.W1 = rng.uniform(-lim1, lim1, size=(hidden, d_in))
        net.W2 = rng.uniform(-lim2, lim2, size=(dv, hidden))
        return net

    def copy_params(self) -> list:
        return [p.clone() for p in self.params()]

    def set_params(self, params: list) -> None:
        for i, p in enumerate(params):
            self._set(i, p)

    @property
    def n_params(self) -> int:
        return int(self.params64.numel())

    def numpy_params(self) -> list:
        return [p.cpu().numpy().copy() for p in self.params()]


def _planes(v, dev, dtype=torch.float32) -> torch.Tensor:
    t = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v))
    t = t.to(device=dev, dtype=dtype)
    if t.ndim == 1:
        t = t.view(-1, 1)
    return t.t().contiguous()


def _vec(a, dev, n=None) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float64))
    t = t.to(device=dev, dtype=torch.float32).reshape(-1)
    if n is not None and t.numel() == 1:
        t = t.expand(n)
    return t.contiguous()


def mlp_forward(net: MlpScoreNet, x, v) -> torch.Tensor:
    """Network output at (x, v) for arrays (n,), (n, dv) (ref: score.py:80-86)."""
    dev = net.params32.device
    vp = _planes(v, dev)
    n = vp.shape[1]
    xs = _vec(x, dev, n)
    s = torch.empty(net.dv, n, dtype=torch.float32, device=dev)
    _lib.call("spic_mlp_forward", _lib.ptr(net.params32), net.hidden, net.dv, None, _lib.ptr(xs),
              _lib.ptr(vp), n, n, 1.0, None, _lib.ptr(s), n, _lib.stream_handle())
    return s.t()


def _partials(net: MlpScoreNet, mode: int, *, n: int, x_scale: float, xv=None, sw=None, x=None,
              vp=None, w=None, Z=None, ldz=0, idx=None, inv_wsum=0.0, ldv=None):
    buf, nb = _lib.scratch("ism", _lib.query("spic_ism_scratch_bytes", n, net.hidden, net.dv))
    _lib.call("spic_ism_partials_ex", _lib.ptr(net.params32), net.hidden, net.dv, mode,
              _lib.ptr(xv), _lib.ptr(sw), _lib.ptr(x), _lib.ptr(vp), ldv if ldv is not None else n,
              _lib.ptr(w), n, float(x_scale), _lib.ptr(Z), ldz, _lib.ptr(idx), float(inv_wsum),
              _lib.ptr(buf), nb, _lib.stream_handle())
    return buf


def _finalize(net: MlpScoreNet, buf, n: int, div_mode: int, *, z=None, opt: "AdamW" = None,
              reset_lr: bool = False, apply_step: bool = False, grads_out=None, loss_out=None,
              flags=None):
    dev = net.params64.device
    if opt is None:
        opt = AdamW(device=dev)
    opt._ensure(net)
    _lib.call("spic_sbtm_finalize_ex", _lib.ptr(buf), n, net.hidden, net.dv, div_mode, _lib.ptr(z),
              _lib.ptr(net.params64), _lib.ptr(opt.m), _lib.ptr(opt.v), _lib.ptr(opt.state),
              float(opt.betas[0]), float(opt.betas[1]), float(opt.eps), float(opt.weight_decay),
              int(reset_lr), int(apply_step), _lib.ptr(net.params32), _lib.ptr(grads_out),
              _lib.ptr(loss_out), _lib.ptr(flags), _lib.stream_handle())


def _split_grads(net: MlpScoreNet, g: torch.Tensor) -> list:
    return [g[a:b].view(*shape) for a, b, shape in net._slices()]


def ism_loss_and_grad(net: MlpScoreNet, x, v, w, *, divergence: str = "hutchinson", z=None):
    """Loss sum_p w_p (|s_p|^2 + 2 div_p) and its gradients (ref: score.py:303-338)."""
    dev = net.params32.device
    vp = _planes(v, dev)
    n = vp.shape[1]
    xs, ws = _vec(x, dev, n), _vec(w, dev, n)
    Zt, zs = None, None
    if divergence == "exact":
        mode = DIV_EXACT
    elif divergence == "hutchinson":
        if z is None:
            raise ValueError("hutchinson divergence needs a Rademacher draw z")
        za = z if isinstance(z, torch.Tensor) else torch.as_tensor(np.asarray(z, dtype=np.float64))
        if za.ndim == 1:
            mode, zs = DIV_SHARED, za.to(device=dev, dtype=torch.float32).contiguous()
        else:
            mode, Zt = DIV_PER_PARTICLE, _planes(za, dev)
    else:
        raise ValueError(f"unknown divergence mode: {divergence!r}")
    buf = _partials(net, mode, n=n, x_scale=1.0, x=xs, vp=vp, w=ws,
                    Z=zs if mode == DIV_SHARED else Zt, ldz=n)
    g = torch.empty(net.n_params, dtype=torch.float64, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    _finalize(net, buf, n, mode, z=zs, grads_out=g, loss_out=loss)
    lv = float(loss.item())
    if not np.isfinite(lv):
        raise RuntimeError("training divergence")
    return lv, _split_grads(net, g)


def mse_loss_and_grad(net: MlpScoreNet, x, v, w, target):
    """sum_p w_p |s_p - y_p|^2 / sum_p w_p and gradients (ref: score.py:254-300, 341-350)."""
    dev = net.params32.device
    vp = _planes(v, dev)
    n = vp.shape[1]
    xs, ws = _vec(x, dev, n), _vec(w, dev, n)
    T = _planes(target, dev)
    inv_wsum = 1.0 / float(ws.double().sum())
    buf = _partials(net, DIV_MSE, n=n, x_scale=1.0, x=xs, vp=vp, w=ws, Z=T, ldz=n, inv_wsum=inv_wsum)
    g = torch.empty(net.n_params, dtype=torch.float64, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    _finalize(net, buf, n, DIV_MSE, grads_out=g, loss_out=loss)
    lv = float(loss.item())
    if not np.isfinite(lv):
        raise RuntimeError("training divergence")
    return lv, _split_grads(net, g)


class AdamW:
    """Adam with decoupled weight decay and bias correction (ref: score.py:358-386).

    Device state: m, v (float64 [P]) and state = [t, lr_current, base_lr, 0]."""

    def __init__(self, lr: float = 2e-4, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 1e-4, device=None):
        self.lr, self.betas, self.eps, self.weight_decay = lr, betas, eps, weight_decay
        self.device = device
        self.m = self.v = None
        self.state = None

    def _ensure(self, net_or_P) -> None:
        P = net_or_P.n_params if isinstance(net_or_P, MlpScoreNet) else int(net_or_P)
        dev = self.device or _lib.require_cuda()
        if self.m is None or self.m.numel() != P:
            self.m = torch.zeros(P, dtype=torch.float64, device=dev)
            self.v = torch.zeros(P, dtype=torch.float64, device=dev)
            self.state = torch.tensor([0.0, self.lr, self.lr, 0.0], dtype=torch.float64, device=dev)
            self._lr_on_device = self.lr
        if self._lr_on_device != self.lr:  # base lr changed on the host (not during capture)
            self.state[2] = float(self.lr)
            self._lr_on_device = self.lr

    @property
    def t(self) -> int:
        return 0 if self.state is None else int(self.state[0].item())

    def step(self, params, grads) -> None:
        """One AdamW step on a network's parameters (params = net or net.params())."""
        net = params if isinstance(params, MlpScoreNet) else None
        if net is None:
            raise TypeError("AdamW.step expects the MlpScoreNet (or its params) on device")
        self._ensure(net)
        g = torch.cat([torch.as_tensor(q, dtype=torch.float64, device=net.params64.device).reshape(-1)
                       for q in grads])
        _lib.call("spic_adamw_step", _lib.ptr(net.params64), _lib.ptr(g), _lib.ptr(self.m),
                  _lib.ptr(self.v), net.n_params, _lib.ptr(self.state), float(self.betas[0]),
                  float(self.betas[1]), float(self.eps), float(self.weight_decay),
                  _lib.ptr(net.params32), _lib.stream_handle())


def draw_probe(rng: np.random.Generator, shape) -> np.ndarray:
    """Rademacher draw exactly as the reference (ref: score.py:565)."""
    return rng.integers(0, 2, size=shape).astype(np.float64) * 2.0 - 1.0


class SbtmTrainer:
    """Device loop of sbtm_update without host syncs (used by the step engine)."""

    def __init__(self, net: MlpScoreNet, optimizer: AdamW, K: int, L: float, divergence: str,
                 rademacher: str, rng: np.random.Generator):
        self.net, self.opt, self.K, self.L = net, optimizer, K, L
        self.divergence, self.rademacher, self.rng = divergence, rademacher, rng
        dev = net.params64.device
        self.losses = torch.zeros(max(K, 1), dtype=torch.float64, device=dev)
        self.z_shared = torch.zeros(max(K, 1), 3, dtype=torch.float32, device=dev)
        self._pinned_z = torch.zeros(max(K, 1), 3, dtype=torch.float32).pin_memory() \
            if torch.cuda.is_available() else None
        optimizer._ensure(net)
        self._z_free = torch.cuda.Event() if torch.cuda.is_available() else None

    def draw_shared_probes(self) -> None:
        """K shared Rademacher probes from the host stream into the pinned staging buffer.
        Waits until the previous step's H2D copy of that buffer has executed (the host may
        run ahead of the device by several steps)."""
        if self.mode() != DIV_SHARED or not self.K:
            return
        self._z_free.synchronize()
        dv = self.net.dv
        zs = np.stack([draw_probe(self.rng, (dv,)) for _ in range(self.K)])
        self._pinned_z[: self.K, :dv].copy_(torch.from_numpy(zs.astype(np.float32)))

    def mode(self) -> int:
        if self.divergence == "exact":
            return DIV_EXACT
        return DIV_SHARED if self.rademacher == "shared" else DIV_PER_PARTICLE

    def run(self, n: int, *, ci: CellIndex | None = None, particles: ParticleEnsemble | None = None,
            flags=None, reduce_row=None, gid=None, n_global: int | None = None,
            draw: bool = True) -> None:
        """K ISM steps. reduce_row(row) (optional) is applied to the reduced float64 row
        [loss, grads, Phi] before each finalize (the cross-rank allreduce); gid (optional)
        maps sorted records to global particle ids for per-particle probes drawn over
        n_global particles. draw=False (CUDA-graph capture) leaves the shared probes to a
        separate draw_shared_probes() call before every replay."""
        mode = self.mode()
        dv = self.net.dv
        Zp = None
        if mode == DIV_SHARED and self.K:
            if draw:
                self.draw_shared_probes()
            self.z_shared.copy_(self._pinned_z, non_blocking=True)
            if draw:  # (under graph capture the replayer records the event instead)
                self._z_free.record()
        for k in range(self.K):
            if mode == DIV_PER_PARTICLE:
                Zp = _planes(draw_probe(self.rng, (n_global or n, dv)), self.net.params32.device)
            zk = self.z_shared[k] if mode == DIV_SHARED else None
            if ci is not None:
                idx = None
                if mode == DIV_PER_PARTICLE:
                    idx = ci.perm if gid is None else gid
                buf = _partials(self.net, mode, n=n, x_scale=1.0 / self.L, xv=ci.xv, sw=ci.sw,
                                Z=zk if mode == DIV_SHARED else Zp,
                                ldz=Zp.shape[1] if Zp is not None else n, idx=idx)
            else:
                buf = _partials(self.net, mode, n=n, x_scale=1.0 / self.L, x=particles.x,
                                vp=particles.vp, w=particles.w,
                                Z=zk if mode == DIV_SHARED else Zp, ldz=n)
            if reduce_row is not None:
                off = int(_lib.query("spic_ism_row_offset", n, self.net.hidden, dv)) // 8
                width = 1 + self.net.n_params + self.net.hidden
                reduce_row(buf.view(torch.float64)[off:off + width])
            _finalize(self.net, buf, n, mode, z=zk, opt=self.opt, reset_lr=(k == 0),
                      apply_step=True, loss_out=self.losses[k:k + 1], flags=flags)


def sbtm_update(net: MlpScoreNet, optimizer: AdamW, particles: ParticleEnsemble, K: int, *,
                L: float, rng: np.random.Generator, divergence: str = "hutchinson",
                rademacher: str = "shared", warnings: list | None = None,
                cell_index: CellIndex | None = None) -> list:
    """K full-batch ISM steps with restore-and-halve recovery (ref: score.py:547-588)."""
    if K <= 0:
        return []
    flags = new_flags(net.params64.device)
    tr = SbtmTrainer(net, optimizer, K, L, divergence, rademacher, rng)
    tr.run(particles.n, ci=cell_index, particles=particles, flags=flags)
    f = flags.cpu().numpy()
    halvings = int(f[_lib.FLAG_LR_HALVINGS])
    if warnings is not None:
        lr = optimizer.lr
        for _ in range(halvings):
            lr *= 0.5
            warnings.append(f"training divergence: learning rate halved to {lr:g}")
    if f[_lib.FLAG_TRAIN_FATAL]:
        raise RuntimeError("training divergence")
    return [float(a) for a in tr.losses[:K].cpu().numpy()]


@dataclass
class PretrainResult:
    final_mse: float
    steps: int
    converged: bool
    tol: float


def pretrain(net, particles: ParticleEnsemble, analytic_score, *, L: float,
             rng: np.random.Generator, budget: int = 10000, batch: int = 4096, lr: float = 1e-3,
             weight_decay: float = 1e-4, tol: float | None = None,
             eval_every: int = 100) -> PretrainResult:
    """Minibatch AdamW fit of the net to a known score (ref: score.py:402-445); the
    minibatch permutations come from `rng` in the reference's order."""
    dev = net.params64.device
    n = particles.n
    xn = (particles.x.double() / L).float().contiguous()
    target = analytic_score(particles.x, particles.v)
    T = _planes(target, dev)
    w64 = particles.w.double()
    wsum = float(w64.sum())
    w_host = particles.w.double().cpu().numpy()
    if tol is None:
        tol = 1e-3 * float((w64 * (T.double() ** 2).sum(0)).sum()) / wsum
    opt = AdamW(lr=lr, weight_decay=weight_decay, device=dev)
    opt._ensure(net.n_params)
    flags = new_flags(dev)
    loss_buf = torch.empty(1, dtype=torch.float64, device=dev)
    idx_dev = torch.empty(n, dtype=torch.int32, device=dev)
    if getattr(net, "arch", "softsign") == "silu":  # extension M1: same loop, SiLU kernels
        from .silu_net import _silu_finalize, _silu_mse_partials

        def mse_partials(nb, idx, inv):
            return _silu_mse_partials(net, nb, x=xn, vp=particles.vp, w=particles.w, Z=T, ldz=n,
                                      idx=idx, inv_wsum=inv, ldv=n)

        def mse_finalize(buf, nb, **kw):
            _silu_finalize(net, buf, nb, kw.pop("opt", None) or AdamW(device=dev), mse=True, **kw)
    else:
        def mse_partials(nb, idx, inv):
            return _partials(net, DIV_MSE, n=nb, x_scale=1.0, x=xn, vp=particles.vp,
                             w=particles.w, Z=T, ldz=n, idx=idx, inv_wsum=inv, ldv=n)

        def mse_finalize(buf, nb, **kw):
            _finalize(net, buf, nb, DIV_MSE, **kw)

    def full_mse() -> float:
        buf = mse_partials(n, None, 1.0 / wsum)
        mse_finalize(buf, n, loss_out=loss_buf)
        return float(loss_buf.item())

    mse = full_mse()
    steps = 0
    perm = None
    while mse >= tol and steps < budget:
        stop = False
        for lo in range(0, n, batch):
            if steps >= budget:
                stop = True
                break
            if lo == 0:
                perm = rng.permutation(n)
                idx_dev.copy_(torch.from_numpy(perm.astype(np.int32)))
            hi = min(lo + batch, n)
            nb = hi - lo
            inv = 1.0 / float(w_host[perm[lo:hi]].sum())
            buf = mse_partials(nb, idx_dev[lo:hi], inv)
            mse_finalize(buf, nb, opt=opt, reset_lr=True, apply_step=True, flags=flags)
            steps += 1
            if steps % eval_every == 0:
                raise_for_flags(flags)
                mse = full_mse()
                if mse < tol:
                    stop = True
                    break
        if stop:
            break
    raise_for_flags(flags)
    mse = full_mse()
    return PretrainResult(final_mse=mse, steps=steps, converged=mse < tol, tol=tol)


# ------------------------------------------------------------------------------------------
# blob (KDE) estimator
# ------------------------------------------------------------------------------------------

def silverman_bandwidth(v) -> float:
    """sigma_hat (4/((dv+2) m))^(1/(dv+4)), mean per-component ddof=1 std; 1.0 fallback
    (ref: score.py:493-500). Device float64 reduction."""
    t = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v))
    t = t.to(device=_lib.require_cuda(), dtype=torch.float64)
    m, dv = t.shape
    sigma = float(t.std(dim=0, unbiased=True).mean()) if m > 1 else 0.0
    h = sigma * (4.0 / ((dv + 2) * m)) ** (1.0 / (dv + 4))
    return h if h > 0 and np.isfinite(h) else 1.0


def blob_sorted(ci: CellIndex, particles: ParticleEnsemble, grid: Grid, bandwidth: float | None,
                flags, bad_pid, h_cell=None) -> None:
    """Blob scores into ci.sw (sorted order); errors are left in flags / bad_pid."""
    n, dv = particles.n, particles.dv
    dev = particles.x.device
    if h_cell is None:
        h_cell = torch.empty(grid.M, dtype=torch.float32, device=dev)
    buf, nb = _lib.scratch("pairs", _lib.query("spic_blob_scratch_bytes", n, grid.M, dv))
    _lib.call("spic_blob", _lib.ptr(ci.xv), _lib.ptr(ci.sw), _lib.ptr(ci.perm), n, dv,
              _lib.ptr(ci.cell_start), _lib.ptr(ci.sub_start) if ci.S > 1 else None, grid.M, ci.S,
              float(grid.eta), float(bandwidth) if bandwidth is not None else -1.0,
              float(particles.uniform_w), _lib.ptr(h_cell), _lib.ptr(bad_pid), _lib.ptr(flags),
              _lib.ptr(buf), nb, _lib.stream_handle())


def _raise_isolated(flags, bad_pid) -> None:
    if flags.cpu().numpy()[_lib.FLAG_ISOLATED]:
        idx = int(bad_pid.item()) & 0xFFFFFFFF
        raise ValueError(f"isolated particle in velocity space (particle {idx})")


def blob_score(particles: ParticleEnsemble, cell_index: CellIndex, grid: Grid,
               bandwidth: float | None = None) -> torch.Tensor:
    """KDE score at every particle, (n, dv) in particle order (ref: score.py:503-523)."""
    dev = particles.x.device
    flags = new_flags(dev)
    bad = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    blob_sorted(cell_index, particles, grid, bandwidth, flags, bad)
    _raise_isolated(flags, bad)
    s = torch.empty(particles.n, particles.dv, dtype=torch.float32, device=dev)
    s[cell_index.perm.long()] = cell_index.sw[:, : particles.dv]
    return s


class BlobEstimator:
    """Stateless KDE score provider; update() is a no-op (ref: score.py:526-540)."""

    def __init__(self, grid: Grid, bandwidth: float | None = None):
        self.grid = grid
        self.bandwidth = bandwidth
        self.warnings: list[str] = []

    def estimate(self, particles: ParticleEnsemble, cell_index: CellIndex | None = None):
        if cell_index is None:
            cell_index = build_cell_index(particles, self.grid)
        return blob_score(particles, cell_index, self.grid, self.bandwidth)

    def update(self, particles: ParticleEnsemble, cell_index: CellIndex | None = None):
        pass


class SbtmEstimator:
    """Neural score provider: estimate() is a forward pass, update() trains
    (ref: score.py:591-623)."""

    def __init__(self, net: MlpScoreNet, L: float, K: int, rng: np.random.Generator, *,
                 lr: float = 2e-4, weight_decay: float = 1e-4, divergence: str = "hutchinson",
                 rademacher: str = "shared"):
        self.net, self.L, self.K, self.rng = net, L, K, rng
        self.divergence, self.rademacher = divergence, rademacher
        self.optimizer = AdamW(lr=lr, weight_decay=weight_decay, device=net.params64.device)
        self.warnings: list[str] = []

    def make_trainer(self) -> SbtmTrainer:
        """The device training loop the step engines drive."""
        return SbtmTrainer(self.net, self.optimizer, self.K, self.L, self.divergence,
                           self.rademacher, self.rng)

    def estimate(self, particles: ParticleEnsemble, cell_index=None) -> torch.Tensor:
        xn = (particles.x.double() / self.L).float()
        return mlp_forward(self.net, xn, particles.v)

    def estimate_sorted(self, ci: CellIndex, n: int) -> None:
        """Scores into the sorted records ci.sw (the engine's fused path)."""
        _lib.call("spic_mlp_forward", _lib.ptr(self.net.params32), self.net.hidden, self.net.dv,
                  _lib.ptr(ci.xv), None, None, n, n, float(1.0 / self.L), _lib.ptr(ci.sw), None, n,
                  _lib.stream_handle())

    def update(self, particles: ParticleEnsemble, cell_index=None) -> None:
        sbtm_update(self.net, self.optimizer, particles, self.K, L=self.L, rng=self.rng,
                    divergence=self.divergence, rademacher=self.rademacher,
                    warnings=self.warnings, cell_index=cell_index)

    def pretrain(self, particles: ParticleEnsemble, analytic_score, *, budget: int = 10000,
                 batch: int = 4096, lr: float = 1e-3) -> PretrainResult:
        res = pretrain(self.net, particles, analytic_score, L=self.L, rng=self.rng, budget=budget,
                       batch=batch, lr=lr, weight_decay=self.optimizer.weight_decay)
        if not res.converged:
            self.warnings.append(f"pretraining budget exhausted: mse {res.final_mse:.3e} "
                                 f"above tol {res.tol:.3e} after {res.steps} steps")
        return res


# ------------------------------------------------------------------------------------------
# SBTM checkpoint (flat little-endian binary, ref: score.py:631-657)
# ------------------------------------------------------------------------------------------
CHECKPOINT_MAGIC = b"SBTM"
CHECKPOINT_VERSION = 1


def save_checkpoint(net: MlpScoreNet, path: str) -> None:
    """magic "SBTM", u32 version, u32 H, u32 dv, then W1, b1, W2, b2 as <f8 (row-major)."""
    import struct

    body = net.params64.cpu().numpy().astype("<f8").tobytes()
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC + struct.pack("<III", CHECKPOINT_VERSION, net.hidden, net.dv) + body)


def load_checkpoint(path: str, device=None) -> MlpScoreNet:
    import struct

    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:4] != CHECKPOINT_MAGIC:
        raise ValueError(f"bad checkpoint magic: {raw[:4]!r}")
    version, hidden, dv = struct.unpack_from("<III", raw, 4)
    if version != CHECKPOINT_VERSION:
        raise ValueError(f"unsupported checkpoint version: {version}")
    net = MlpScoreNet(dv, hidden, device)
    P = net.n_params
    if len(raw) < 16 + 8 * P:
        raise ValueError("truncated checkpoint")
    if len(raw) > 16 + 8 * P:
        raise ValueError("trailing bytes in checkpoint")
    net.params64.copy_(torch.from_numpy(np.frombuffer(raw, dtype="<f8", offset=16).copy()))
    net.refresh32()
    return net
