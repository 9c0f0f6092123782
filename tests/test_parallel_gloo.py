"""Domain decomposition host logic on CPU with the gloo backend (world sizes 2 and 3):
partition, migration (all-to-all), halo exchange incl. the R = 2 ordering case, and a
decomposed collision step (the float64 oracle as the per-rank compute) against the
single-rank oracle."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_25832_b200.parallel import CellPartition, Comm, migrate


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


def _migration_body(rank, world, M):
    rng = np.random.default_rng(100 + rank)
    n = 500 + 37 * rank
    cells = torch.as_tensor(rng.integers(0, M, n), dtype=torch.int64)
    gid = torch.arange(n, dtype=torch.int64) + 10000 * rank
    rows = torch.stack([gid.double(), cells.double()], 1)
    part = CellPartition.equal(M, world)
    owner = torch.as_tensor(part.owner_table(), dtype=torch.int64)
    got = migrate(rows, cells, owner, Comm())
    lo, hi = part.owned(rank)
    assert torch.all((got[:, 1] >= lo) & (got[:, 1] < hi))
    # every particle arrives exactly once somewhere
    cnt = torch.tensor([got.shape[0]], dtype=torch.int64)
    dist.all_reduce(cnt)
    total = sum(500 + 37 * r for r in range(world))
    assert int(cnt) == total
    # order: by source rank, then source order (deterministic)
    src = (got[:, 0] // 10000).long()
    assert torch.all(src[1:] >= src[:-1])


@pytest.mark.parametrize("world", [2, 3])
def test_migration_alltoall(world):
    _run(_migration_body, world, 11)


def _halo_body(rank, world):
    M = 3 if world == 2 else 7
    part = CellPartition.equal(M, world)
    comm = Comm()
    to_left = torch.tensor([[rank, 0.0]] * (rank + 1))   # my first cell
    to_right = torch.tensor([[rank, 1.0]] * (rank + 2))  # my last cell
    fl, fr = comm.exchange_halo(to_left, to_right, part)
    left, right = part.neighbours(rank)
    # from_left is the left neighbour's last cell, from_right the right neighbour's first
    assert fl.shape[0] == left + 2 and torch.all(fl[:, 0] == left) and torch.all(fl[:, 1] == 1)
    assert fr.shape[0] == right + 1 and torch.all(fr[:, 0] == right) and torch.all(fr[:, 1] == 0)


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_ordering(world):
    _run(_halo_body, world)


def _collision_body(rank, world, n, M, seed):
    """Rank r: own particles (cells [lo, hi)) + 1-cell halos from the neighbours, oracle
    collision on that set, U of own particles compared with the global oracle result."""
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    L = 4 * math.pi
    eta = L / M
    x = rng.uniform(0, L, n)
    v = rng.normal(size=(n, 3))
    s = rng.normal(size=(n, 3)) * 2
    w = np.full(n, L / n)
    U_ref = O.collision_force(x, v, w, s, eta, M, -3.0)
    part = CellPartition.equal(M, world)
    lo, hi = part.owned(rank)
    cell = O.cell_of(x, eta, M)
    own = np.nonzero((cell >= lo) & (cell < hi))[0]
    perm, starts = O.build_cell_index(x[own], eta, M)
    rows = torch.as_tensor(np.column_stack([own[perm], x[own][perm], v[own][perm], s[own][perm]]))
    first = rows[starts[lo]:starts[lo + 1]]
    last = rows[starts[hi - 1]:starts[hi]]
    fl, fr = Comm().exchange_halo(first, last, part)
    hl, hr = part.halo_cells(rank)
    halo = fl if hl == hr else torch.cat([fl, fr])
    idx = np.concatenate([own, halo[:, 0].numpy().astype(np.int64)])
    xs, vs, ss = x[idx], v[idx], s[idx]
    U = O.collision_force(xs, vs, np.full(len(idx), L / n), ss, eta, M, -3.0)
    err = np.max(np.abs(U[: len(own)] - U_ref[own]))
    assert err <= 1e-12 * max(1.0, np.max(np.abs(U_ref))), err


@pytest.mark.parametrize("world,M", [(2, 8), (3, 9), (2, 3)])
def test_decomposed_collision_matches_single_rank(world, M):
    _run(_collision_body, world, 600, M, 7 + world)
