"""TEST INFRASTRUCTURE ONLY — the parity oracle for the scorepic hot path.

Float64 CPU restatement of the reference (`/root/reference/pkg/src/scorepic`, cited as
``ref: file:line``). Heavy loops live in ``oracle.c`` (built into ``oracle/build/liboracle.so``
by ``oracle/Makefile``); the small O(M) / O(P) pieces are restated here in numpy.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` leg and
``--impl reference``) may import this module, and only as the checker / CPU baseline. The
product package ``paper_2603_25832_b200`` never imports it.

Pinning: ``tests/golden/make_golden.py`` runs the reference itself (in the build container)
and stores inputs/outputs under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks
every function here against those vectors.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

EPS_Z = 1e-12  # ref: kernels.py:7


def build() -> str:
    """Compile oracle.c (gcc, OpenMP). Test infrastructure only."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        P = ctypes.c_void_p
        sig = {
            "oracle_cell_of": (None, [P, i64, d, i64, P]),
            "oracle_build_cell_index": (None, [P, i64, d, i64, P, P]),
            "oracle_collision_force": (i32, [P, P, P, P, i64, i32, i64, d, d, P]),
            "oracle_collision_force_sampled": (i32, [P, P, P, P, i64, i32, i64, d, d, i64, P]),
            "oracle_count_live_pairs": (i64, [P, i64, i64, d]),
            "oracle_silverman_bandwidth": (d, [P, i64, i32]),
            "oracle_blob_score": (i32, [P, P, P, i64, i32, i64, d, d, P, P, P]),
            "oracle_blob_score_sampled": (i32, [P, P, P, i64, i32, i64, d, d, i64, P, P, P]),
            "oracle_mlp_forward": (None, [P, P, i64, i32, i64, P, P, P, P, P]),
            "oracle_ism_kernel": (d, [P, P, P, i64, i32, i64, P, P, P, P, P, P, P, P]),
            "oracle_mse_kernel": (d, [P, P, P, i64, i32, i64, P, P, P, P, P, d, P]),
            "oracle_deposit": (None, [P, P, P, i64, i32, i64, d, P, P]),
            "oracle_push": (i32, [P, P, i64, i32, P, P, P, i64, d, d]),
            "oracle_maxwell_step": (None, [P, P, P, P, i64, d, d]),
            "oracle_vpl_field_step": (None, [P, P, i64, d]),
            "oracle_num_threads": (i32, []),
            "oracle_set_num_threads": (None, [i32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_num_threads(t: int) -> None:
    lib().oracle_set_num_threads(int(t))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ------------------------------------------------------------------------------------------
# state / grid (ref: state.py:14-27, pic.py:14-30)
# ------------------------------------------------------------------------------------------

def wrap_position(x, L):
    """x mod L in [0, L); values rounding to L fold to 0 (ref: state.py:14-27)."""
    if L <= 0:
        raise ValueError("domain length must be positive")
    x = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite position")
    out = np.mod(x, L)
    return np.where(out >= L, 0.0, out)


def cell_of(x, eta: float, M: int) -> np.ndarray:
    x = _f64(x)
    out = np.empty(x.shape[0], dtype=np.int64)
    lib().oracle_cell_of(_p(x), x.shape[0], float(eta), int(M), _p(out))
    return out


def build_cell_index(x, eta: float, M: int):
    """(perm, starts): stable argsort by cell id and bin boundaries (ref: collision.py:39-46)."""
    x = _f64(x)
    n = x.shape[0]
    perm = np.empty(n, dtype=np.int64)
    starts = np.empty(M + 1, dtype=np.int64)
    lib().oracle_build_cell_index(_p(x), n, float(eta), int(M), _p(perm), _p(starts))
    return perm, starts


# ------------------------------------------------------------------------------------------
# collision (ref: collision.py:49-116)
# ------------------------------------------------------------------------------------------

def collision_force(x, v, w, s, eta: float, M: int, gamma: float, cell_stride: int = 1):
    x, v, w, s = _f64(x), _f64(v), _f64(w), _f64(s)
    n, dv = v.shape
    U = np.zeros((n, dv))
    rc = lib().oracle_collision_force_sampled(_p(x), _p(v), _p(w), _p(s), n, dv, int(M),
                                              float(eta), float(gamma), int(cell_stride), _p(U))
    if rc != 0:
        raise ValueError("invalid score input")
    return U


def count_live_pairs(x, eta: float, M: int) -> int:
    x = _f64(x)
    return int(lib().oracle_count_live_pairs(_p(x), x.shape[0], int(M), float(eta)))


def collision_push(v, U, nu: float, dt: float):
    """v <- v - (dt*nu) U (ref: collision.py:113-116)."""
    return _f64(v) - (dt * nu) * _f64(U)


# ------------------------------------------------------------------------------------------
# blob (ref: score.py:453-523)
# ------------------------------------------------------------------------------------------

def silverman_bandwidth(v) -> float:
    v = _f64(v)
    m, dv = v.shape
    return float(lib().oracle_silverman_bandwidth(_p(v), m, dv))


def blob_score(x, v, w, eta: float, M: int, bandwidth: float | None = None,
               cell_stride: int = 1, return_den: bool = False):
    x, v, w = _f64(x), _f64(v), _f64(w)
    n, dv = v.shape
    s = np.zeros((n, dv))
    den = np.zeros(n)
    bad = np.zeros(1, dtype=np.int64)
    h = -1.0 if bandwidth is None else float(bandwidth)
    rc = lib().oracle_blob_score_sampled(_p(x), _p(v), _p(w), n, dv, int(M), float(eta), h,
                                         int(cell_stride), _p(s), _p(den), _p(bad))
    if rc != 0:
        raise ValueError(f"isolated particle in velocity space (particle {int(bad[0])})")
    return (s, den) if return_den else s


# ------------------------------------------------------------------------------------------
# SBTM network, ISM loss, AdamW (ref: score.py:38-120, 128-386, 547-588)
# ------------------------------------------------------------------------------------------

@dataclass
class Net:
    W1: np.ndarray  # (H, 1+dv)
    b1: np.ndarray  # (H,)
    W2: np.ndarray  # (dv, H)
    b2: np.ndarray  # (dv,)

    @property
    def H(self) -> int:
        return self.W1.shape[0]

    @property
    def dv(self) -> int:
        return self.W2.shape[0]

    def params(self):
        return [self.W1, self.b1, self.W2, self.b2]

    def copy(self) -> "Net":
        return Net(*[p.copy() for p in self.params()])

    @classmethod
    def glorot(cls, dv: int, H: int, rng: np.random.Generator) -> "Net":
        """Glorot-uniform W1 then W2 from the same stream, zero biases (ref: score.py:50-58)."""
        d_in = 1 + dv
        lim1 = np.sqrt(6.0 / (d_in + H))
        lim2 = np.sqrt(6.0 / (H + dv))
        W1 = rng.uniform(-lim1, lim1, size=(H, d_in))
        W2 = rng.uniform(-lim2, lim2, size=(dv, H))
        return cls(W1, np.zeros(H), W2, np.zeros(dv))


def mlp_forward(net: Net, x, v) -> np.ndarray:
    x, v = _f64(x), _f64(v)
    n, dv = v.shape
    S = np.empty((n, dv))
    W1, b1, W2, b2 = (_f64(p) for p in net.params())
    lib().oracle_mlp_forward(_p(x), _p(v), n, dv, net.H, _p(W1), _p(b1), _p(W2), _p(b2), _p(S))
    return S


def _split_grads(g: np.ndarray, H: int, dv: int):
    o1 = H * (1 + dv)
    o2 = o1 + H
    o3 = o2 + dv * H
    return [g[:o1].reshape(H, 1 + dv).copy(), g[o1:o2].copy(),
            g[o2:o3].reshape(dv, H).copy(), g[o3:].copy()]


def ism_loss_and_grad(net: Net, x, v, w, *, divergence: str = "exact", z=None):
    """Loss sum_p w_p (|s_p|^2 + 2 div_p) and gradients (ref: score.py:303-338)."""
    x, v, w = _f64(x), _f64(v), _f64(w)
    n, dv = v.shape
    H = net.H
    W1, b1, W2, b2 = (_f64(p) for p in net.params())
    P = H * (1 + dv) + H + dv * H + dv
    g = np.zeros(P)
    Phi = np.zeros(H)
    if divergence == "exact":
        coef = np.einsum("ih,hi->h", W2, W1[:, 1:])
        loss = lib().oracle_ism_kernel(_p(x), _p(v), _p(w), n, dv, H, _p(W1), _p(b1), _p(W2),
                                       _p(b2), _p(_f64(coef)), None, _p(g), _p(Phi))
        gW1, gb1, gW2, gb2 = _split_grads(g, H, dv)
        gW2 += 2.0 * Phi[None, :] * W1[:, 1:].T
        gW1[:, 1:] += 2.0 * Phi[:, None] * W2.T
    elif divergence == "hutchinson":
        if z is None:
            raise ValueError("hutchinson divergence needs a Rademacher draw z")
        z = _f64(z)
        if z.ndim == 1:
            t = W1[:, 1:] @ z
            r = W2.T @ z
            loss = lib().oracle_ism_kernel(_p(x), _p(v), _p(w), n, dv, H, _p(W1), _p(b1),
                                           _p(W2), _p(b2), _p(_f64(r * t)), None, _p(g), _p(Phi))
            gW1, gb1, gW2, gb2 = _split_grads(g, H, dv)
            gW2 += 2.0 * np.outer(z, t * Phi)
            gW1[:, 1:] += 2.0 * np.outer(r * Phi, z)
        else:
            loss = lib().oracle_ism_kernel(_p(x), _p(v), _p(w), n, dv, H, _p(W1), _p(b1),
                                           _p(W2), _p(b2), None, _p(z), _p(g), None)
            gW1, gb1, gW2, gb2 = _split_grads(g, H, dv)
    else:
        raise ValueError(f"unknown divergence mode: {divergence!r}")
    if not np.isfinite(loss):
        raise RuntimeError("training divergence")
    return float(loss), [gW1, gb1, gW2, gb2]


def mse_loss_and_grad(net: Net, x, v, w, target):
    """Weighted score MSE and gradients (ref: score.py:254-300, 341-350)."""
    x, v, w, target = _f64(x), _f64(v), _f64(w), _f64(target)
    n, dv = v.shape
    H = net.H
    W1, b1, W2, b2 = (_f64(p) for p in net.params())
    P = H * (1 + dv) + H + dv * H + dv
    g = np.zeros(P)
    loss = lib().oracle_mse_kernel(_p(x), _p(v), _p(w), n, dv, H, _p(W1), _p(b1), _p(W2), _p(b2),
                                   _p(target), 1.0 / float(w.sum()), _p(g))
    if not np.isfinite(loss):
        raise RuntimeError("training divergence")
    return float(loss), _split_grads(g, H, dv)


class AdamW:
    """Decoupled weight decay, bias-corrected Adam (ref: score.py:358-386)."""

    def __init__(self, lr=2e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=1e-4):
        self.lr, self.betas, self.eps, self.weight_decay = lr, betas, eps, weight_decay
        self.m = self.v = None
        self.t = 0

    def step(self, params, grads):
        if self.m is None:
            self.m = [np.zeros_like(p) for p in params]
            self.v = [np.zeros_like(p) for p in params]
        b1, b2 = self.betas
        self.t += 1
        bc1 = 1.0 - b1 ** self.t
        bc2 = 1.0 - b2 ** self.t
        for p, g, m, v in zip(params, grads, self.m, self.v):
            if self.weight_decay:
                p -= self.lr * self.weight_decay * p
            m *= b1
            m += (1.0 - b1) * g
            v *= b2
            v += (1.0 - b2) * g * g
            p -= self.lr * (m / bc1) / (np.sqrt(v / bc2) + self.eps)


def sbtm_update(net: Net, opt: AdamW, x, v, w, K: int, *, L: float, rng=None,
                divergence: str = "exact", rademacher: str = "shared", warnings=None,
                probes=None):
    """K full-batch ISM steps with restore-and-halve recovery (ref: score.py:547-588).

    `probes`, when given, supplies the K Rademacher draws instead of `rng`.
    """
    xn = _f64(x) / L
    base_lr = opt.lr
    losses = []
    try:
        for k in range(K):
            z = None
            if divergence == "hutchinson":
                if probes is not None:
                    z = probes[k]
                else:
                    size = (v.shape[1],) if rademacher == "shared" else v.shape
                    z = rng.integers(0, 2, size=size).astype(np.float64) * 2.0 - 1.0
            while True:
                saved = [p.copy() for p in net.params()]
                try:
                    loss, grads = ism_loss_and_grad(net, xn, v, w, divergence=divergence, z=z)
                    opt.step(net.params(), grads)
                    if all(np.all(np.isfinite(p)) for p in net.params()):
                        losses.append(loss)
                        break
                    raise RuntimeError("training divergence")
                except RuntimeError:
                    for p, s in zip(net.params(), saved):
                        p[...] = s
                    opt.lr *= 0.5
                    if warnings is not None:
                        warnings.append(f"training divergence: learning rate halved to {opt.lr:g}")
                    if opt.lr < 1e-12:
                        raise
    finally:
        opt.lr = base_lr
    return losses


# ------------------------------------------------------------------------------------------
# PIC (ref: pic.py:33-134)
# ------------------------------------------------------------------------------------------

def deposit(x, v, w, eta: float, M: int):
    x, v, w = _f64(x), _f64(v), _f64(w)
    n, dv = v.shape
    rho = np.empty(M)
    J = np.empty((dv, M))
    lib().oracle_deposit(_p(x), _p(v), _p(w), n, dv, int(M), float(eta), _p(rho), _p(J))
    return rho, J


def push(x, v, E1, E2, B3, eta: float, M: int, dt: float):
    """interpolate -> Lorentz push -> advance + wrap (ref: pic.py:61-93). Returns (x, v)."""
    x, v = _f64(x).copy(), _f64(v).copy()
    n, dv = v.shape
    rc = lib().oracle_push(_p(x), _p(v), n, dv, _p(_f64(E1)), _p(_f64(E2)), _p(_f64(B3)),
                           int(M), float(eta), float(dt))
    if rc != 0:
        raise ValueError("non-finite position")
    return x, v


def maxwell_step(E1, E2, B3, J, eta: float, dt: float):
    E1, E2, B3 = _f64(E1).copy(), _f64(E2).copy(), _f64(B3).copy()
    J = _f64(J)
    M = E1.shape[0]
    lib().oracle_maxwell_step(_p(E1), _p(E2), _p(B3), _p(J), M, float(eta), float(dt))
    return E1, E2, B3


def vpl_field_step(E1, J, dt: float):
    E1 = _f64(E1).copy()
    J = _f64(J)
    lib().oracle_vpl_field_step(_p(E1), _p(J), E1.shape[0], float(dt))
    return E1


def poisson_solve(rho, rho_ion: float, eta: float):
    """Spectral periodic solve of -phi'' = rho - rho_ion, E1 = -phi' (ref: pic.py:118-134)."""
    src = _f64(rho) - rho_ion
    M = src.shape[0]
    if abs(src.sum() * eta) > 1e-8:
        raise ValueError("non-neutral plasma")
    sh = np.fft.rfft(src)
    k = 2.0 * np.pi * np.fft.rfftfreq(M, d=eta)
    Eh = np.zeros_like(sh)
    Eh[1:] = -1j * sh[1:] / k[1:]
    if M % 2 == 0:
        Eh[-1] = 0.0
    return np.fft.irfft(Eh, n=M)


def diagnostics(v, w, E1, E2, B3, eta: float, *, nu: float = 0.0, U=None, s=None):
    """E_K, E_E, E_B, E_total, H_dot, P, E_l2 (ref: diagnostics.py:20-35)."""
    v, w = _f64(v), _f64(w)
    E_K = 0.5 * float(np.sum(w * np.einsum("ij,ij->i", v, v)))
    e2 = float(np.sum(_f64(E1) ** 2 + _f64(E2) ** 2))
    E_E = 0.5 * eta * e2
    E_B = 0.5 * eta * float(np.sum(_f64(B3) ** 2))
    H_dot = 0.0
    if nu > 0 and U is not None and s is not None:
        H_dot = float(np.sum(w * np.einsum("ij,ij->i", _f64(s), _f64(U))))
    return dict(E_K=E_K, E_E=E_E, E_B=E_B, E_total=E_K + E_E + E_B, H_dot=H_dot, P=w @ v,
                E_l2=float(np.sqrt(eta * e2)))


# ------------------------------------------------------------------------------------------
# one full step of Algorithm 1 (ref: run.py:81-118), used by bench.py's reference arm
# ------------------------------------------------------------------------------------------

def full_step(state: dict, *, eta: float, M: int, dt: float, nu: float, mode: str,
              gamma: float, net: Net | None, opt: AdamW | None, K: int,
              divergence: str = "exact", estimator: str = "sbtm",
              bandwidth: float | None = None, cell_stride: int = 1, timers: dict | None = None):
    """Advance `state` (x, v, w, E1, E2, B3) by one step. With cell_stride > 1 the pair
    kernels evaluate only every cell_stride-th cell (a bounded CPU sample)."""
    import time

    def tick(name, t0):
        if timers is not None:
            timers[name] = timers.get(name, 0.0) + time.perf_counter() - t0

    L = M * eta
    t0 = time.perf_counter()
    x, v = push(state["x"], state["v"], state["E1"], state["E2"], state["B3"], eta, M, dt)
    tick("push", t0)
    t0 = time.perf_counter()
    rho, J = deposit(x, v, state["w"], eta, M)
    if mode == "VML":
        E1, E2, B3 = maxwell_step(state["E1"], state["E2"], state["B3"], J, eta, dt)
    else:
        E1, E2, B3 = vpl_field_step(state["E1"], J, dt), state["E2"], state["B3"]
    tick("deposit_field", t0)
    U = s = None
    if nu > 0:
        t0 = time.perf_counter()
        build_cell_index(x, eta, M)
        tick("bin", t0)
        t0 = time.perf_counter()
        if estimator == "sbtm":
            sbtm_update(net, opt, x, v, state["w"], K, L=L, divergence=divergence)
            tick("ism", t0)
            t0 = time.perf_counter()
            s = mlp_forward(net, x / L, v)
        else:
            s = blob_score(x, v, state["w"], eta, M, bandwidth, cell_stride=cell_stride)
        tick("estimate", t0)
        t0 = time.perf_counter()
        U = collision_force(x, v, state["w"], s, eta, M, gamma, cell_stride=cell_stride)
        v = collision_push(v, U, nu, dt)
        tick("collide", t0)
    state.update(x=x, v=v, E1=E1, E2=E2, B3=B3, rho=rho, J=J)
    return diagnostics(v, state["w"], E1, E2, B3, eta, nu=nu, U=U, s=s)


# ------------------------------------------------------------------------------------------
# Long-time equilibrium oracles (ref: equilibrium.py:24-55), used by the acceptance tests
# ------------------------------------------------------------------------------------------

def vpl_equilibrium(initial_energy: float, initial_momentum, rho_ion: float, volume: float):
    """Electrostatic steady state (ref: equilibrium.py:40-55): drift u = P0 / (rho_ion |Omega|),
    T_inf = 2 / (dv rho_ion |Omega|) (E0 - rho_ion |u|^2 |Omega| / 2). Returns (T_inf, u)."""
    P0 = np.asarray(initial_momentum, dtype=np.float64)
    dv = P0.shape[0]
    u = P0 / (rho_ion * volume)
    T = 2.0 / (dv * rho_ion * volume) * (initial_energy - 0.5 * rho_ion * float(u @ u) * volume)
    if not T > 0:
        raise ValueError("inconsistent energy accounting")
    return T, u


def vml_equilibrium(initial_energy: float, B_init_mean, rho_ion: float, volume: float,
                    dv: int = 3):
    """Electromagnetic steady state (ref: equilibrium.py:24-37): zero drift, B_inf = mean B(0),
    T_inf = 2 / (dv rho_ion |Omega|) (E0 - |B_inf|^2 |Omega| / 2). Returns (T_inf, B_inf)."""
    B = np.asarray(B_init_mean, dtype=np.float64).reshape(3)
    T = 2.0 / (dv * rho_ion * volume) * (initial_energy - 0.5 * float(B @ B) * volume)
    if not T > 0:
        raise ValueError("inconsistent energy accounting")
    return T, B
