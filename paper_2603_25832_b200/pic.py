"""Particle-grid transfer, pushes and field solvers on the B200 (ref: pic.py:14-134).

Operator API with the reference's names; every call launches the sm_100a kernels of
libscorepic_b200.so on the current CUDA stream. `interpolate_fields -> lorentz_push ->
advance_positions` is one fused kernel here (`push_particles`); the three reference names are
kept as thin entry points of that kernel where the semantics allow.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .state import FieldState, ParticleEnsemble, new_flags

FIELD_NONE, FIELD_VPL, FIELD_VML = 0, 1, 2


@dataclass(frozen=True)
class Grid:
    M: int
    eta: float

    @property
    def L(self) -> float:
        return self.M * self.eta

    @property
    def centers(self) -> np.ndarray:
        return (np.arange(self.M) + 0.5) * self.eta

    def cell_of(self, x: torch.Tensor) -> torch.Tensor:
        """min(floor(x/eta) mod M, M-1) in float64 on the float32 positions (int32)."""
        x = x.contiguous()
        out = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
        _lib.call("spic_cell_of", _lib.ptr(x), x.shape[0], float(self.eta), int(self.M),
                  _lib.ptr(out), _lib.stream_handle())
        return out


def raise_for_flags(flags, fields=None) -> None:
    """Map device flags (a device tensor, or a host copy of it) to the reference's exceptions.
    With `fields` given, a non-finite field is named as in FieldState.validate
    (ref: state.py:75-78: "non-finite field state: {name}", first of E1, E2, B3, rho, J)."""
    f = flags.cpu().numpy() if isinstance(flags, torch.Tensor) else np.asarray(flags)
    if f[_lib.FLAG_NONFINITE_X]:
        raise ValueError("non-finite position")
    if f[_lib.FLAG_NON_NEUTRAL]:
        raise ValueError("non-neutral plasma")
    if f[_lib.FLAG_BAD_SCORE]:
        raise ValueError("invalid score input")
    if f[_lib.FLAG_TRAIN_FATAL]:
        raise RuntimeError("training divergence")
    if f[_lib.FLAG_NONFINITE_V]:
        raise ValueError("non-finite particle state")
    if f[_lib.FLAG_NONFINITE_FIELD]:
        name = "E1"
        if fields is not None:
            for nm in ("E1", "E2", "B3", "rho", "J"):
                a = getattr(fields, nm, None)
                if a is not None and not bool(torch.isfinite(a).all()):
                    name = nm
                    break
        raise ValueError(f"non-finite field state: {name}")


def push_particles(particles: ParticleEnsemble, fields: FieldState, grid: Grid, dt: float,
                   flags: torch.Tensor | None = None) -> None:
    """interpolate_fields + lorentz_push + advance_positions in one pass (in place)."""
    own = flags is None
    flags = new_flags(particles.x.device) if own else flags
    _lib.call("spic_push", _lib.ptr(particles.x), _lib.ptr(particles.vp), particles.n,
              particles.n, particles.dv, _lib.ptr(fields.E1), _lib.ptr(fields.E2),
              _lib.ptr(fields.B3), grid.M, float(grid.eta), float(dt), _lib.ptr(flags),
              _lib.stream_handle())
    if own:
        f = flags.cpu().numpy()
        if f[_lib.FLAG_NONFINITE_X]:
            raise ValueError("non-finite position")


def interpolate_fields(particles: ParticleEnsemble, fields: FieldState, grid: Grid):
    """E_p (n, dv) = (E1, E2, 0...), B_p (n, 3) = (0, 0, B3) at the particles
    (ref: pic.py:61-74); the hot loop fuses this into push_particles."""
    n, dv = particles.n, particles.dv
    dev = particles.x.device
    Ep = torch.empty(dv, n, dtype=torch.float32, device=dev)
    Bp = torch.empty(3, n, dtype=torch.float32, device=dev)
    _lib.call("spic_interpolate", _lib.ptr(particles.x), n, dv, _lib.ptr(fields.E1),
              _lib.ptr(fields.E2), _lib.ptr(fields.B3), grid.M, float(grid.eta), _lib.ptr(Ep), n,
              _lib.ptr(Bp), n, _lib.stream_handle())
    return Ep.t(), Bp.t()


def lorentz_push(particles: ParticleEnsemble, E_p, B_p, dt: float) -> None:
    """v <- v + dt (E + v x B), B = (0, 0, B3) (ref: pic.py:77-88), in place."""
    n, dv = particles.n, particles.dv
    dev = particles.x.device
    Ep = torch.as_tensor(E_p, dtype=torch.float32, device=dev).t().contiguous()
    Bp = torch.as_tensor(B_p, dtype=torch.float32, device=dev).t().contiguous()
    flags = new_flags(dev)
    _lib.call("spic_lorentz", _lib.ptr(particles.vp), n, n, dv, _lib.ptr(Ep), n, _lib.ptr(Bp), n,
              float(dt), _lib.ptr(flags), _lib.stream_handle())


def advance_positions(particles: ParticleEnsemble, dt: float, L: float) -> None:
    """x <- (x + dt v1) mod L (ref: pic.py:91-93): the fused push with zero fields."""
    M = 1
    z = torch.zeros(M, dtype=torch.float64, device=particles.x.device)
    push_particles(particles, FieldState(z, z, z, z, z.view(1, 1), 0.0), Grid(M, float(L)), dt)


def deposit(particles: ParticleEnsemble, grid: Grid):
    """rho (M,), J (dv, M) float64 (ref: pic.py:43-58): bin, then the deterministic deposit."""
    from .collision import build_cell_index

    ci = build_cell_index(particles, grid)
    return deposit_from_index(ci, particles, grid)


def deposit_from_index(ci, particles: ParticleEnsemble, grid: Grid, fields: FieldState | None = None,
                       field_mode: int = FIELD_NONE, dt: float = 0.0, diag_out=None, flags=None):
    dev = particles.x.device
    rho = fields.rho if fields is not None else torch.empty(grid.M, dtype=torch.float64, device=dev)
    J = fields.J if fields is not None else torch.empty(particles.dv, grid.M, dtype=torch.float64,
                                                        device=dev)
    dummy = torch.zeros(grid.M, dtype=torch.float64, device=dev) if fields is None else None
    E1 = fields.E1 if fields is not None else dummy
    E2 = fields.E2 if fields is not None else dummy
    B3 = fields.B3 if fields is not None else dummy
    buf, nb = _lib.scratch("deposit", _lib.query("spic_deposit_scratch_bytes", grid.M, particles.dv))
    fl = flags if flags is not None else new_flags(dev)
    _lib.call("spic_deposit_field", _lib.ptr(ci.xv), _lib.ptr(ci.sw), particles.n, particles.dv,
              _lib.ptr(ci.cell_start), grid.M, float(grid.eta), float(particles.uniform_w),
              _lib.ptr(rho), _lib.ptr(J), int(field_mode), float(dt), _lib.ptr(E1), _lib.ptr(E2),
              _lib.ptr(B3), _lib.ptr(diag_out), _lib.ptr(fl), _lib.ptr(buf), nb,
              _lib.stream_handle())
    return rho, J


def maxwell_step(fields: FieldState, J: torch.Tensor, dt: float, grid: Grid) -> None:
    """E1 -= dt J1; E2 -= dt(dB3/dx + J2); B3 -= dt dE2/dx with the fresh E2 (ref: pic.py:96-110)."""
    J = J.to(torch.float64).contiguous()
    _lib.call("spic_field_step", _lib.ptr(fields.E1), _lib.ptr(fields.E2), _lib.ptr(fields.B3),
              _lib.ptr(J), grid.M, float(grid.eta), float(dt), FIELD_VML, None, None,
              _lib.stream_handle())


def vpl_field_step(fields: FieldState, J: torch.Tensor, dt: float) -> None:
    """E1 -= dt J1 (ref: pic.py:113-115)."""
    J = J.to(torch.float64).contiguous()
    M = fields.E1.shape[0]
    _lib.call("spic_field_step", _lib.ptr(fields.E1), _lib.ptr(fields.E2), _lib.ptr(fields.B3),
              _lib.ptr(J), M, 1.0, float(dt), FIELD_VPL, None, None, _lib.stream_handle())


def poisson_solve(rho: torch.Tensor, rho_ion: float, grid: Grid) -> torch.Tensor:
    """Periodic spectral solve of -phi'' = rho - rho_ion, E1 = -phi' (ref: pic.py:118-134)."""
    rho = rho.to(torch.float64).contiguous()
    E1 = torch.empty(grid.M, dtype=torch.float64, device=rho.device)
    flags = new_flags(rho.device)
    _lib.call("spic_poisson", _lib.ptr(rho), float(rho_ion), grid.M, float(grid.eta), _lib.ptr(E1),
              _lib.ptr(flags), _lib.stream_handle())
    if flags.cpu().numpy()[_lib.FLAG_NON_NEUTRAL]:
        raise ValueError("non-neutral plasma")
    return E1
