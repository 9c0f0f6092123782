"""Domain decomposition host logic on CPU with the gloo backend (world sizes 2, 3 and 4):
partitions, the boundary-message cell ranges of dist_engine (send_ranges) and the fixed-size
ring exchange (Comm.exchange_pair, incl. the R = 2 posting-order case), checked by building
each rank's union of own + received particles exactly as DistSimulation does and comparing it
with the global particle set."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_25832_b200.dist_engine import cyclic_segments, intersect_segments, send_ranges
from paper_2603_25832_b200.parallel import CellPartition, Comm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(fn, world, *args):
    port = _free_port()
    # spawn, not fork: the parent may hold an OpenMP pool (oracle tests) that deadlocks
    # in forked children
    mp.start_processes(_entry, args=(fn, world, port, args), nprocs=world, join=True,
                       start_method="spawn")


def _entry(rank, fn, world, port, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def test_partition_balanced_and_equal():
    p = CellPartition.equal(10, 3)
    assert list(p.bounds) == [0, 3, 6, 10]
    assert list(p.owner_table()) == [0, 0, 0, 1, 1, 1, 2, 2, 2, 2]
    assert p.halo_cells(0) == (9, 3) and p.halo_cells(2) == (5, 0)
    counts = np.array([100, 1, 1, 1, 1, 100, 1, 1])
    b = CellPartition.balanced(counts, 2)
    assert b.bounds[0] == 0 and b.bounds[-1] == 8 and 1 <= b.bounds[1] <= 6
    assert np.all(np.diff(CellPartition.balanced(np.ones(5, int), 5).bounds) == 1)


def test_cyclic_segments_and_send_ranges_cover_the_ring():
    assert cyclic_segments(6, 4, 8) == [(6, 8), (0, 2)]
    assert cyclic_segments(2, 3, 8) == [(2, 5), (0, 0)]
    assert cyclic_segments(5, 0, 8) == [(0, 0), (0, 0)]
    assert intersect_segments([(6, 8), (0, 2)], 0, 4) == [(0, 0), (0, 2)]
    for M, R, g in [(16, 2, 1), (16, 2, 2), (9, 3, 1), (64, 4, 2), (1024, 8, 1)]:
        part = CellPartition.equal(M, R)
        for r in range(R):
            lo, hi = part.owned(r)
            (sl, _), (sr, _) = send_ranges(part, r, g)
            cells = np.zeros(M, int)
            for a, b in sl + sr:
                cells[a:b] += 1
            # every cell outside the owned range is sent exactly once; the g boundary cells
            # on each side too (to their neighbour); the interior is kept
            for c in range(M):
                inside = lo <= c < hi
                boundary = inside and (c < lo + g or c >= hi - g)
                want = 1 if (not inside or boundary) else 0
                if inside and g * 2 > hi - lo:
                    continue
                assert cells[c] == want, (M, R, g, r, c, cells[c])


def _exchange_body(rank, world, M, g, seed, balanced):
    """Global particles (gid, cell) are spread over the ranks as they would be after a push:
    rank r holds its own particles, some of them moved up to D cells outside [lo, hi). The
    union own + received must contain every global particle of [lo - g, hi + g) exactly once,
    and the owned count from the headers must equal the global count of [lo, hi)."""
    rng = np.random.default_rng(seed)
    n = 4000
    counts = rng.integers(1, 50, M) if balanced else np.ones(M, int)
    part = CellPartition.balanced(counts, world) if balanced else CellPartition.equal(M, world)
    width = min(np.diff(part.bounds))
    D = max(0, min(3, width - g))
    home = rng.integers(0, M, n)                     # cell before the push (owner = rank)
    moved = (home + rng.integers(-D, D + 1, n)) % M  # cell after the push
    own_rank = part.owner_table()[home]
    gid = np.arange(n)
    lo, hi = part.owned(rank)
    mine = own_rank == rank
    mg, mc = gid[mine], moved[mine]
    order = np.argsort(mc, kind="stable")
    mg, mc = mg[order], mc[order]
    cs = np.searchsorted(mc, np.arange(M + 1), side="left")
    (sl, rl), (sr, rr) = send_ranges(part, rank, g)
    cap = n

    def pack(segs, recv_segs):
        rows = [np.column_stack([mg[cs[a]:cs[b]], mc[cs[a]:cs[b]]]) for a, b in segs if b > a]
        rows = np.concatenate(rows) if rows else np.zeros((0, 2), int)
        owned = sum(cs[b] - cs[a] for a, b in recv_segs if b > a)
        msg = np.full((cap + 1, 2), -1, dtype=np.int64)
        msg[0] = (rows.shape[0], owned)
        msg[1:1 + rows.shape[0]] = rows
        return torch.as_tensor(msg)

    to_l, to_r = pack(sl, rl), pack(sr, rr)
    from_l, from_r = torch.empty_like(to_l), torch.empty_like(to_r)
    Comm().exchange_pair(to_l, to_r, from_l, from_r, part)
    got = [np.column_stack([mg, mc])]
    own_count = int(cs[hi] - cs[lo])
    for m in (from_l.numpy(), from_r.numpy()):
        k, owned = int(m[0, 0]), int(m[0, 1])
        got.append(m[1:1 + k])
        own_count += owned
    union = np.concatenate(got)
    window = [(lo - g + k) % M for k in range(hi - lo + 2 * g)]
    in_win = np.isin(union[:, 1], window)
    ug = union[in_win, 0]
    want = gid[np.isin(moved, window)]
    assert len(ug) == len(np.unique(ug)), "a particle arrived twice"
    assert set(ug.tolist()) == set(want.tolist())
    assert own_count == int(np.sum((moved >= lo) & (moved < hi)))


@pytest.mark.parametrize("world,M,g,balanced", [(2, 16, 1, False), (2, 16, 2, False),
                                                (3, 9, 1, False), (3, 24, 2, True),
                                                (4, 64, 2, True)])
def test_boundary_exchange_builds_the_halo_union(world, M, g, balanced):
    _run(_exchange_body, world, M, g, 11 + world, balanced)


def _allreduce_body(rank, world):
    comm = Comm()
    t = torch.tensor([float(rank + 1), -float(rank)])
    comm.allreduce_(t)
    assert t.tolist() == [sum(range(1, world + 1)), -sum(range(world))]
    m = torch.tensor([rank, 7 - rank], dtype=torch.int32)
    comm.allreduce_(m, op="max")
    assert m.tolist() == [world - 1, 7]


@pytest.mark.parametrize("world", [2, 3])
def test_allreduce_sum_and_max(world):
    _run(_allreduce_body, world)
