"""Cell-range domain decomposition across ranks.

One process per GPU. Rank r owns the contiguous cell range [C_r, C_{r+1}) and the particles
in it. Per step the only exchanges are the ones the physics needs:

  * migration   — particles whose new cell is owned elsewhere go to the owner
                  (all-to-all with per-destination counts; in practice only ring
                  neighbours receive anything since dt |v1| << cell width);
  * deposit     — allreduce(SUM) of the deposited rho, J (M x (1+dv) float64);
  * SBTM        — allreduce(SUM) of the reduced ISM loss/gradient row (1 + P + H float64)
                  before every finalize, so every rank applies the identical AdamW step;
  * halo        — the particles of the boundary cells C_r and C_{r+1}-1 go to the left and
                  right neighbours (1-cell halo: the stencil of an owned cell is owned or
                  halo); for the blob estimator the halo scores are exchanged a second time;
  * diagnostics — allreduce(SUM) of [H_dot, E_K, P].

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
    """torch.distributed helpers (works for gloo/CPU and NCCL/CUDA tensors)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.size = dist.get_world_size(group) if dist.is_initialized() else 1

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def alltoallv(self, send: torch.Tensor, counts: torch.Tensor) -> torch.Tensor:
        """Rows of `send` (grouped by destination, counts[d] rows for rank d) -> rows received,
        grouped by source rank in rank order."""
        if self.size == 1:
            return send.clone()
        counts = counts.to(torch.int64)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        sc, rc = counts.cpu().tolist(), recv_counts.cpu().tolist()
        out = torch.empty((sum(rc),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(out, send.contiguous(), output_split_sizes=rc,
                               input_split_sizes=sc, group=self.group)
        return out

    def exchange_halo(self, to_left: torch.Tensor, to_right: torch.Tensor,
                      part: CellPartition) -> tuple[torch.Tensor, torch.Tensor]:
        """Send rows to the left / right neighbour; returns (from_left, from_right), where
        from_left is the left neighbour's `to_right` (its last cell) and vice versa.
        With R == 2 both neighbours are the same rank; point-to-point messages between one
        pair of ranks are matched in posting order, so the receives are posted swapped."""
        if self.size == 1:
            return to_right.clone(), to_left.clone()
        left, right = part.neighbours(self.rank)
        dev, dt, tail = to_left.device, to_left.dtype, tuple(to_left.shape[1:])

        def p2p(sends, recvs):
            ops = [dist.P2POp(dist.isend, t, peer, self.group) for t, peer in sends if t.numel()]
            ops += [dist.P2POp(dist.irecv, t, peer, self.group) for t, peer in recvs if t.numel()]
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()

        n_l = torch.tensor([to_left.shape[0]], dtype=torch.int64, device=dev)
        n_r = torch.tensor([to_right.shape[0]], dtype=torch.int64, device=dev)
        m_l = torch.empty(1, dtype=torch.int64, device=dev)
        m_r = torch.empty(1, dtype=torch.int64, device=dev)
        recv_order = [(m_r, right), (m_l, left)] if left == right else [(m_l, left), (m_r, right)]
        p2p([(n_l, left), (n_r, right)], recv_order)
        from_left = torch.empty((int(m_l.item()),) + tail, dtype=dt, device=dev)
        from_right = torch.empty((int(m_r.item()),) + tail, dtype=dt, device=dev)
        recv_order = [(from_right, right), (from_left, left)] if left == right else \
            [(from_left, left), (from_right, right)]
        p2p([(to_left.contiguous(), left), (to_right.contiguous(), right)], recv_order)
        return from_left, from_right


def route(cells: torch.Tensor, owner: torch.Tensor, R: int):
    """Stable grouping of local rows by destination rank: (order, counts)."""
    dest = owner[cells.long()]
    order = torch.argsort(dest, stable=True)
    counts = torch.bincount(dest, minlength=R)
    return order, counts


def migrate(rows: torch.Tensor, cells: torch.Tensor, owner: torch.Tensor, comm: Comm) -> torch.Tensor:
    """Send every row to the owner of its cell; returns this rank's rows (by source rank)."""
    order, counts = route(cells, owner, comm.size)
    return comm.alltoallv(rows[order], counts)


def boundary_rows(rows_sorted: torch.Tensor, cell_start: np.ndarray, part: CellPartition,
                  rank: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Rows of my first and last owned cells from cell-sorted rows (contiguous slices)."""
    lo, hi = part.owned(rank)
    first = rows_sorted[int(cell_start[lo]):int(cell_start[lo + 1])]
    last = rows_sorted[int(cell_start[hi - 1]):int(cell_start[hi])]
    return first, last
