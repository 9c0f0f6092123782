"""Cell index and the binned Landau collision operator on the B200 (ref: collision.py:22-116).

`build_cell_index` runs the deterministic counting sort (spic_bin); with the default S = 1
its permutation is bit-identical to the reference's stable argsort, and it also gathers the
cell-sorted float4 records the pair kernels stream. `collision_force` runs the tiled
pair kernel (spic_landau) and scatters U back to particle order.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .pic import Grid
from .state import ParticleEnsemble, new_flags


def auto_sub_cells(n: int, M: int) -> int:
    """Sub-cell sort depth S (power of two <= 64): keys M*S <= 32768 (the binning kernel's
    shared-memory histogram) and >= ~64 particles per sub-cell. Finer sub-cells let the pair
    kernels skip more of the stencil beyond eta of a target tile."""
    S = 1
    while S < 64 and M * S * 2 <= 32768 and n // (M * S * 2) >= 64:
        S *= 2
    return S


class CellIndex:
    """Per-cell particle lists (ref: collision.py:22-36), held on device.

    perm[k] = particle index at sorted position k; cell_start[c]..cell_start[c+1] is cell c.
    xv/sw are the cell-sorted float4 records (x', v) and (s, w)."""

    def __init__(self, perm, cell_start, sub_start, M: int, S: int, xv, sw):
        self.perm, self.cell_start, self.sub_start = perm, cell_start, sub_start
        self.M, self.S, self.xv, self.sw = M, S, xv, sw

    @property
    def bins(self) -> list:
        """Reference-style list of ascending-pid int64 arrays per cell (host copy)."""
        perm = self.perm.cpu().numpy().astype(np.int64)
        cs = self.cell_start.cpu().numpy()
        out = [perm[cs[c]:cs[c + 1]] for c in range(self.M)]
        if self.S > 1:  # sub-cell order inside a cell: restore pid order for the API view
            out = [np.sort(b) for b in out]
        return out

    def neighbors(self, c: int) -> np.ndarray:
        cells = []
        for d in (-1, 0, 1):
            cd = (c + d) % self.M
            if cd not in cells:
                cells.append(cd)
        b = self.bins
        return np.concatenate([b[cd] for cd in cells])


def build_cell_index(particles: ParticleEnsemble, grid: Grid, S: int = 1,
                     out: CellIndex | None = None) -> CellIndex:
    n, dv, M = particles.n, particles.dv, grid.M
    dev = particles.x.device
    if out is None:
        out = CellIndex(torch.empty(n, dtype=torch.int32, device=dev),
                        torch.empty(M + 1, dtype=torch.int32, device=dev),
                        torch.empty(M * S + 1, dtype=torch.int32, device=dev), M, S,
                        torch.empty(n, 4, dtype=torch.float32, device=dev),
                        torch.empty(n, 4, dtype=torch.float32, device=dev))
    buf, nb = _lib.scratch("bin", _lib.query("spic_bin_scratch_bytes", n, M, S))
    _lib.call("spic_bin", _lib.ptr(particles.x), _lib.ptr(particles.vp), n, _lib.ptr(particles.w), n,
              dv, float(grid.eta), M, S, _lib.ptr(out.perm), _lib.ptr(out.cell_start),
              _lib.ptr(out.sub_start), _lib.ptr(out.xv), _lib.ptr(out.sw), _lib.ptr(buf), nb,
              _lib.stream_handle())
    return out


def landau_sorted(ci: CellIndex, particles: ParticleEnsemble, grid: Grid, gamma: float,
                  U_sorted: torch.Tensor, nsplit: int = 0) -> torch.Tensor:
    """U in sorted order (dv, n) from the records (scores already in ci.sw)."""
    n, dv = particles.n, particles.dv
    buf, nb = _lib.scratch("pairs", _lib.query("spic_landau_scratch_bytes", n, grid.M, dv, nsplit))
    _lib.call("spic_landau", _lib.ptr(ci.xv), _lib.ptr(ci.sw), n, dv, _lib.ptr(ci.cell_start),
              _lib.ptr(ci.sub_start) if ci.S > 1 else None, grid.M, ci.S, float(grid.eta),
              float(gamma), float(particles.uniform_w), int(nsplit), _lib.ptr(U_sorted),
              _lib.ptr(buf), nb, _lib.stream_handle())
    return U_sorted


def gather_scores_sorted(cell_index: CellIndex, scores, flags=None) -> torch.Tensor:
    """Scatter pid-order scores (n, dv) into the sorted records' s lanes; returns the flags."""
    n = cell_index.perm.numel()
    dev = cell_index.sw.device
    s = scores if isinstance(scores, torch.Tensor) else torch.as_tensor(np.asarray(scores))
    sp = s.to(device=dev, dtype=torch.float32).t().contiguous()  # (dv, n) planes
    dv = sp.shape[0]
    flags = new_flags(dev) if flags is None else flags
    _lib.call("spic_gather_scores", _lib.ptr(sp), n, _lib.ptr(cell_index.perm), n, dv,
              _lib.ptr(cell_index.sw), _lib.ptr(flags), _lib.stream_handle())
    return flags


def collision_force(particles: ParticleEnsemble, scores, cell_index: CellIndex, grid: Grid,
                    gamma: float) -> torch.Tensor:
    """U (n, dv) for every particle (ref: collision.py:92-110); non-finite scores raise."""
    n, dv = particles.n, particles.dv
    dev = particles.x.device
    flags = gather_scores_sorted(cell_index, scores)
    if flags.cpu().numpy()[_lib.FLAG_BAD_SCORE]:
        raise ValueError("invalid score input")
    U_sorted = torch.empty(dv, n, dtype=torch.float32, device=dev)
    landau_sorted(cell_index, particles, grid, gamma, U_sorted)
    U = torch.empty(dv, n, dtype=torch.float32, device=dev)
    buf, nb = _lib.scratch("epilogue", 8 * 2 * 148 * 5 + 64)
    _lib.call("spic_collision_epilogue", _lib.ptr(U_sorted), _lib.ptr(cell_index.sw),
              _lib.ptr(cell_index.perm), n, dv, 0.0, _lib.ptr(particles.vp), n, _lib.ptr(U), n,
              None, _lib.ptr(flags), _lib.ptr(buf), nb, _lib.stream_handle())
    return U.t()


def collision_push(particles: ParticleEnsemble, U: torch.Tensor, nu: float, dt: float) -> None:
    """v <- v - dt nu U (ref: collision.py:113-116). The hot loop fuses this into the
    collision epilogue; this standalone form is a device axpy on the velocity planes."""
    particles.vp.sub_(U.to(particles.vp.dtype).t(), alpha=float(dt * nu))


def count_live_pairs(ci: CellIndex, particles: ParticleEnsemble, grid: Grid) -> int:
    cnt = torch.zeros(1, dtype=torch.int64, device=particles.x.device)
    _lib.call("spic_count_live_pairs", _lib.ptr(ci.xv), particles.n, _lib.ptr(ci.cell_start),
              grid.M, float(grid.eta), _lib.ptr(cnt), _lib.stream_handle())
    return int(cnt.item())
