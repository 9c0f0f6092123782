"""Cell-range domain decomposition across ranks.

One process per GPU. Rank r owns the contiguous cell range [C_r, C_{r+1}) and the particles
in it. Per step the only exchanges are the ones the physics needs (dist_engine.py):

  * deposit     — allreduce(SUM) of the deposited [rho; J] ((1+dv) x M float64);
  * SBTM        — allreduce(SUM) of the reduced ISM loss/gradient row (1 + P + H float64)
                  before every finalize, so every rank applies the identical AdamW step;
  * boundary    — one fixed-size message to each ring neighbour carrying the particles that
                  moved to its side plus the first / last g owned cells (its halo); migration
                  and the halo exchange are this one message;
  * diagnostics — allreduce(SUM) of [H_dot, E_K, P, sum w].

The routines here are device-agnostic (torch tensors + torch.distributed), so the partition
and exchange logic is tested on CPU with the gloo backend (tests/test_parallel_gloo.py); on
the B200 box the same code runs over NCCL with device tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class CellPartition:
    M: int
    bounds: np.ndarray  # (R+1,) cell boundaries, bounds[0] = 0, bounds[R] = M

    @property
    def R(self) -> int:
        return len(self.bounds) - 1

    @classmethod
    def equal(cls, M: int, R: int) -> "CellPartition":
        if R < 1 or M < R:
            raise ValueError(f"cannot split {M} cells over {R} ranks")
        return cls(M, np.array([(r * M) // R for r in range(R + 1)], dtype=np.int64))

    @classmethod
    def balanced(cls, counts, R: int) -> "CellPartition":
        """Contiguous ranges with ~equal particle counts (each rank owns >= 1 cell)."""
        counts = np.asarray(counts, dtype=np.int64)
        M = counts.shape[0]
        if R < 1 or M < R:
            raise ValueError(f"cannot split {M} cells over {R} ranks")
        cum = np.concatenate([[0], np.cumsum(counts)])
        total = cum[-1]
        b = [0]
        for r in range(1, R):
            target = total * r / R
            c = int(np.searchsorted(cum, target, side="left"))
            c = max(c, b[-1] + 1)            # at least one cell per rank
            c = min(c, M - (R - r))          # leave a cell for every later rank
            b.append(c)
        b.append(M)
        return cls(M, np.array(b, dtype=np.int64))

    def owner_table(self) -> np.ndarray:
        own = np.empty(self.M, dtype=np.int32)
        for r in range(self.R):
            own[self.bounds[r]:self.bounds[r + 1]] = r
        return own

    def owned(self, r: int) -> tuple[int, int]:
        return int(self.bounds[r]), int(self.bounds[r + 1])

    def halo_cells(self, r: int) -> tuple[int, int]:
        """(left halo cell, right halo cell) of rank r on the periodic grid."""
        lo, hi = self.owned(r)
        return (lo - 1) % self.M, hi % self.M

    def neighbours(self, r: int) -> tuple[int, int]:
        return (r - 1) % self.R, (r + 1) % self.R


class Comm:
    """torch.distributed helpers (works for gloo/CPU and NCCL/CUDA tensors).

    host_staged=True runs every collective on host copies of device tensors (gloo on CPU):
    several ranks can then share one GPU (NCCL refuses two ranks on one device), which is how
    the multi-rank device path is tested on a single B200."""

    def __init__(self, group=None, host_staged: bool = False):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.size = dist.get_world_size(group) if dist.is_initialized() else 1
        self.host_staged = host_staged

    def _op(self, op: str):
        return {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX}[op]

    def allreduce_(self, t: torch.Tensor, op: str = "sum") -> torch.Tensor:
        if self.size > 1:
            if self.host_staged and t.is_cuda:
                h = t.cpu()
                dist.all_reduce(h, op=self._op(op), group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=self._op(op), group=self.group)
        return t

    def exchange_pair(self, to_left: torch.Tensor, to_right: torch.Tensor,
                      from_left: torch.Tensor, from_right: torch.Tensor,
                      part: "CellPartition") -> None:
        """Fixed-size point-to-point exchange with the ring neighbours: to_left goes to the
        left neighbour (which receives it as its from_right), to_right to the right one. With
        R == 2 both neighbours are one rank; messages between one pair of ranks match in
        posting order, so the receives are posted swapped there."""
        if self.size == 1:
            from_left.copy_(to_right)
            from_right.copy_(to_left)
            return
        left, right = part.neighbours(self.rank)
        staged = self.host_staged and to_left.is_cuda
        sl, sr = (to_left.cpu(), to_right.cpu()) if staged else (to_left, to_right)
        rl = torch.empty_like(sl) if staged else from_left
        rr = torch.empty_like(sr) if staged else from_right
        ops = [dist.P2POp(dist.isend, sl, left, self.group),
               dist.P2POp(dist.isend, sr, right, self.group)]
        recvs = [(rr, right), (rl, left)] if left == right else [(rl, left), (rr, right)]
        ops += [dist.P2POp(dist.irecv, t, peer, self.group) for t, peer in recvs]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if staged:
            from_left.copy_(rl)
            from_right.copy_(rr)
