"""Domain-decomposed step engine: one process per GPU, cell ranges per rank.

Rank r owns the cells [lo, hi). Its step (same kernels as engine.Simulation, plus the three
exchange kernels of csrc/dist.cu):

    push (own particles)
    bin them as they are -> records R0            (particles may now sit a few cells outside
                                                    [lo, hi): binning is over all M cells)
    deposit(R0) -> allreduce(rho, J) -> field step (sums over particles: any partition of the
                                                    particles gives the same global sums)
    pack + exchange:  to the left neighbour the R0 records of the cyclic cell range
                      [mid, lo + g), to the right [hi - g, mid) (mid = the far point of the
                      complement arc; g = halo width), as fixed-capacity messages
    SBTM: K x (ISM partials over R0 -> allreduce(reduced row) -> finalize)   (replicated net)
    -- the one host synchronisation of the step: the received row counts, read while the GPU
       still runs the K-loop (so the GPU does not idle) --
    unpack the messages behind the own particles -> bin the union -> scores (SBTM forward over
    the union / blob over the union, whose g = 2 halo cells make the halo scores local)
    -> Landau pair kernel with targets in [lo, hi) -> epilogue: v -= nu dt U for the owned
    targets, written compacted in sorted order as the next step's own particles
    -> allreduce([H_dot, E_K, P, sum w])

Migration is implicit: the owned targets of the union are exactly the particles in [lo, hi)
after the push, wherever they came from. No torch sort / bincount / cat is on the path; the
exchanges are two fixed-size point-to-point messages (no count round-trip), two small
allreduces per step plus one per ISM step. Ranges can be rebalanced on the owned per-cell
counts every `rebalance_every` steps (one allreduce of M counts; boundaries move by at most
a quarter of a neighbour's range per rebalance so the next step's exchange still covers it).
A particle that moves past a whole neighbouring range in one step (dt |v1| > the range width)
is lost; the diagnostics row's sum of weights then drifts from L (ValueError "total particle
weight drifted from L", as the reference's validate, ref: state.py:46-53).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .collision import CellIndex, auto_sub_cells
from .config import DeviceOptions
from .engine import nvtx
from .parallel import CellPartition, Comm
from .pic import FIELD_NONE, FIELD_VML, FIELD_VPL, Grid, deposit_from_index, raise_for_flags
from .score import BlobEstimator, SbtmEstimator, blob_sorted
from .state import DiagnosticsRecord, FieldState, ParticleEnsemble, new_flags

DIAG_W = 9
_NO_PID = torch.iinfo(torch.int64).max


def _round_up(v: int, m: int) -> int:
    return (int(v) + m - 1) // m * m


class _Buffers:
    """Capacity-managed pid-order particle planes of one rank (own particles first, then the
    received ones). The capacity is a multiple of 64 so the velocity planes stay 16-B aligned
    (vectorised push / bulk-copy binning paths)."""

    def __init__(self, cap: int, dv: int, dev):
        cap = _round_up(max(cap, 64), 64)
        self.cap, self.dv, self.dev = cap, dv, dev
        self.x = torch.zeros(cap, dtype=torch.float32, device=dev)
        self.vp = torch.zeros(dv, cap, dtype=torch.float32, device=dev)
        self.w = torch.zeros(cap, dtype=torch.float32, device=dev)
        self.gid = torch.zeros(cap, dtype=torch.int32, device=dev)

    def ensure(self, need: int, keep: int) -> None:
        if need <= self.cap:
            return
        nb = _Buffers(int(need * 1.25) + 1024, self.dv, self.dev)
        nb.x[:keep].copy_(self.x[:keep])
        nb.vp[:, :keep].copy_(self.vp[:, :keep])
        nb.w[:keep].copy_(self.w[:keep])
        nb.gid[:keep].copy_(self.gid[:keep])
        self.__dict__.update(nb.__dict__)

    def view(self, n: int, uniform_w: float) -> ParticleEnsemble:
        # planes with leading dimension cap: pass a (dv, n) view; kernels get ldv = cap
        return ParticleEnsemble(self.x[:n], self.vp[:, :n], self.w[:n], uniform_w)


class _Index:
    """Grow-only cell index (perm, cell_start, sub_start, records) of up to `cap` records."""

    def __init__(self, M: int, S: int, dev):
        self.M, self.S, self.dev, self.cap = M, S, dev, 0
        self.ci = None

    def get(self, n: int) -> CellIndex:
        if self.ci is None or n > self.cap:
            cap = _round_up(int(max(n, 1) * 1.25) + 1024, 64)
            M, S, dev = self.M, self.S, self.dev
            self.ci = CellIndex(torch.empty(cap, dtype=torch.int32, device=dev),
                                torch.empty(M + 1, dtype=torch.int32, device=dev),
                                torch.empty(M * S + 1, dtype=torch.int32, device=dev), M, S,
                                torch.empty(cap, 4, dtype=torch.float32, device=dev),
                                torch.zeros(cap, 4, dtype=torch.float32, device=dev))
            self.cap = cap
        return self.ci


def cyclic_segments(a: int, length: int, M: int) -> list[tuple[int, int]]:
    """Linear cell segments of the cyclic range [a, a + length) (0 <= length <= M)."""
    a %= M
    if length <= 0:
        return [(0, 0), (0, 0)]
    if a + length <= M:
        return [(a, a + length), (0, 0)]
    return [(a, M), (0, a + length - M)]


def intersect_segments(segs, lo: int, hi: int) -> list[tuple[int, int]]:
    out = []
    for a, b in segs:
        c0, c1 = max(a, lo), min(b, hi)
        out.append((c0, c1) if c1 > c0 else (0, 0))
    return out


def send_ranges(part: CellPartition, rank: int, halo: int):
    """(to_left, to_right): the cyclic cell ranges a rank sends to its ring neighbours as two
    linear segments each, and the parts of them the receivers own. to_left = [mid, lo + g),
    to_right = [hi - g, mid), mid = the cell opposite the owned range on the ring."""
    M = part.M
    lo, hi = part.owned(rank)
    comp = M - (hi - lo)
    mid = (hi + comp // 2) % M
    left, right = part.neighbours(rank)
    to_l = cyclic_segments(mid, (lo + halo - mid) % M, M)
    to_r = cyclic_segments(hi - halo, (mid - (hi - halo)) % M, M)
    return ((to_l, intersect_segments(to_l, *part.owned(left))),
            (to_r, intersect_segments(to_r, *part.owned(right))))


def _flat(segs) -> np.ndarray:
    return np.array([segs[0][0], segs[0][1], segs[1][0], segs[1][1]], dtype=np.int32)


class DistSimulation:
    def __init__(self, x, v, w, gid, fields: FieldState, grid: Grid, *, dt: float, nu: float,
                 mode: str, gamma: float, estimator=None, comm: Comm | None = None,
                 partition: CellPartition | None = None, n_global: int | None = None,
                 options: DeviceOptions | None = None, max_rows: int = 1024,
                 halo: int | None = None, msg_capacity: int | None = None,
                 rebalance_every: int = 0):
        self.comm = comm or Comm()
        self.grid, self.f = grid, fields
        self.dt, self.nu, self.mode, self.gamma = float(dt), float(nu), mode, float(gamma)
        self.est = estimator
        self.opt = options or DeviceOptions()
        dev = fields.E1.device
        self.dev = dev
        x, v, w = np.asarray(x), np.asarray(v), np.asarray(w)
        dv = v.shape[1]
        self.dv = dv
        n = x.shape[0]
        self.part = partition or CellPartition.equal(grid.M, self.comm.size)
        self.n_global = int(n_global or n)
        self.uniform_w = float(w[0]) if n and bool(np.all(w == w[0])) else 0.0
        self.halo = int(halo or (2 if isinstance(estimator, BlobEstimator) else 1))
        self.cur = _Buffers(int(1.25 * n) + 1024, dv, dev)
        self.nxt = _Buffers(self.cur.cap, dv, dev)
        self.n = n
        self.cur.x[:n].copy_(torch.as_tensor(x, dtype=torch.float32))
        self.cur.vp[:, :n].copy_(torch.as_tensor(v, dtype=torch.float32).t())
        self.cur.w[:n].copy_(torch.as_tensor(w, dtype=torch.float32))
        self.cur.gid[:n].copy_(torch.as_tensor(np.asarray(gid), dtype=torch.int32))
        self.S = self.opt.sub_cells or auto_sub_cells(max(self.n_global, 1), grid.M)
        self.idx0 = _Index(grid.M, self.S, dev)  # R0: own particles after the push
        self.idx = _Index(grid.M, self.S, dev)   # union: own + received
        self.flags = new_flags(dev)
        self.bad_pid = torch.full((1,), _NO_PID, dtype=torch.int64, device=dev)
        self.h_cell = torch.empty(grid.M, dtype=torch.float32, device=dev)
        self.diag = torch.zeros(max_rows, DIAG_W, dtype=torch.float64, device=dev)
        self.trainer = None
        if isinstance(estimator, SbtmEstimator):
            self.trainer = estimator.make_trainer()
        self._epi, self._epi_n = _lib.scratch("dist_epilogue",
                                              _lib.query("spic_dist_epilogue_scratch_bytes"))
        self.time_collision = False
        self.collision_events: list = []
        self.grid_moments = torch.zeros(1 + dv, grid.M, dtype=torch.float64, device=dev)
        self.U = torch.empty(dv, 1024, dtype=torch.float32, device=dev)
        # fixed-capacity messages (rows); a message that needs more raises at the step's sync
        self.mcap = int(msg_capacity or max(4096, self.n_global // max(4, 2 * self.comm.size)))
        self.send = torch.zeros(2, self.mcap + 1, 8, dtype=torch.float32, device=dev)
        self.recv = torch.zeros(2, self.mcap + 1, 8, dtype=torch.float32, device=dev)
        self._stage = torch.zeros(16, dtype=torch.int32, device=dev)
        self._stage_host = torch.zeros(16, dtype=torch.int32).pin_memory()
        self._ready = torch.cuda.Event()
        self.rebalance_every = int(rebalance_every)
        self.steps_done = 0
        self.host_syncs = 0  # per-step host synchronisations (bench evidence)
        self._set_ranges()

    # ---- partition-dependent constants ------------------------------------------------------
    def _set_ranges(self) -> None:
        r = self.comm.rank
        self.lo, self.hi = self.part.owned(r)
        if self.comm.size > 1 and (self.hi - self.lo) < self.halo:
            raise ValueError(f"rank {r} owns {self.hi - self.lo} cells, fewer than the halo "
                             f"width {self.halo}")
        (sl, rl), (sr, rr) = send_ranges(self.part, r, self.halo)
        self._send_cells = [_flat(sl), _flat(sr)]
        self._recv_cells = [_flat(rl), _flat(rr)]
        self._cs_idx = torch.tensor([self.lo, self.hi], dtype=torch.int64, device=self.dev)

    # ---- helpers ----------------------------------------------------------------------------
    def _bin(self, b: _Buffers, n: int, index: _Index) -> CellIndex:
        ci = index.get(n)
        g = self.grid
        buf, nb = _lib.scratch("bin", _lib.query("spic_bin_scratch_bytes", n, g.M, self.S))
        _lib.call("spic_bin", _lib.ptr(b.x), _lib.ptr(b.vp), b.cap, _lib.ptr(b.w), n, self.dv,
                  float(g.eta), g.M, self.S, _lib.ptr(ci.perm), _lib.ptr(ci.cell_start),
                  _lib.ptr(ci.sub_start), _lib.ptr(ci.xv), _lib.ptr(ci.sw), _lib.ptr(buf), nb,
                  _lib.stream_handle())
        return ci

    def _pack(self, k: int, ci: CellIndex) -> None:
        b = self.cur
        _lib.call("spic_dist_pack", _lib.ptr(b.x), _lib.ptr(b.vp), b.cap, self.dv,
                  None if self.uniform_w > 0 else _lib.ptr(b.w), float(self.uniform_w),
                  _lib.ptr(b.gid), _lib.ptr(ci.perm), _lib.ptr(ci.cell_start), self.grid.M,
                  self._send_cells[k].ctypes.data, self._recv_cells[k].ctypes.data, self.mcap,
                  _lib.ptr(self.send[k]), _lib.stream_handle())

    def rebalance(self) -> None:
        """New cell ranges from the owned per-cell counts (one allreduce + host read)."""
        if self.comm.size == 1 or self.idx.ci is None:
            return
        M = self.grid.M
        cs = self.idx.ci.cell_start.to(torch.int64)
        cnt = torch.zeros(M, dtype=torch.float64, device=self.dev)
        cnt[self.lo:self.hi] = (cs[self.lo + 1:self.hi + 1] - cs[self.lo:self.hi]).double()
        self.comm.allreduce_(cnt)
        new = CellPartition.balanced(cnt.cpu().numpy().astype(np.int64), self.comm.size).bounds
        old = self.part.bounds
        b = old.copy()
        for k in range(1, len(b) - 1):  # move each boundary by <= 1/4 of the narrower side
            lim = max(0, min(old[k] - old[k - 1], old[k + 1] - old[k]) // 4)
            b[k] = int(np.clip(new[k], old[k] - lim, old[k] + lim))
        self.part = CellPartition(M, b)
        self._set_ranges()

    # ---- one step ---------------------------------------------------------------------------
    def step(self, row: int) -> None:
        g, f, comm = self.grid, self.f, self.comm
        dv, st, R = self.dv, _lib.stream_handle(), comm.size
        if self.rebalance_every and self.steps_done and self.steps_done % self.rebalance_every == 0:
            self.rebalance()
        d = self.diag[row]
        d.zero_()
        self._last_row = row
        b, n = self.cur, self.n
        # 1. push own particles
        rng = nvtx("push")
        rng.__enter__()
        _lib.call("spic_push", _lib.ptr(b.x), _lib.ptr(b.vp), b.cap, n, dv, _lib.ptr(f.E1),
                  _lib.ptr(f.E2), _lib.ptr(f.B3), g.M, float(g.eta), self.dt, _lib.ptr(self.flags), st)
        rng.__exit__(None, None, None)
        # 2. bin them where they are (R0), deposit, one allreduce of [rho; J], field step
        with nvtx("bin"):
            ci0 = self._bin(b, n, self.idx0)
        rng = nvtx("deposit")
        rng.__enter__()
        self._n0 = n
        gm = self.grid_moments
        deposit_from_index(ci0, b.view(n, self.uniform_w), g,
                           fields=FieldState(f.E1, f.E2, f.B3, gm[0], gm[1:], f.rho_ion),
                           field_mode=FIELD_NONE, flags=self.flags)
        comm.allreduce_(gm)
        f.rho.copy_(gm[0])
        f.J.copy_(gm[1:])
        fmode = FIELD_VML if self.mode == "VML" else FIELD_VPL
        _lib.call("spic_field_step", _lib.ptr(f.E1), _lib.ptr(f.E2), _lib.ptr(f.B3), _lib.ptr(f.J),
                  g.M, float(g.eta), self.dt, fmode, _lib.ptr(d[0:3]), _lib.ptr(self.flags), st)
        self.steps_done += 1
        rng.__exit__(None, None, None)
        if not (self.nu > 0 and self.est is not None):
            buf, nb = _lib.scratch("moments", _lib.query("spic_moments_scratch_bytes", n))
            _lib.call("spic_moments", _lib.ptr(b.vp), b.cap, _lib.ptr(b.w), n, dv,
                      float(self.uniform_w), _lib.ptr(d[4:9]), _lib.ptr(self.flags), _lib.ptr(buf),
                      nb, st)
            comm.allreduce_(d[3:9])
            return
        # 3. boundary messages (fixed size) to the ring neighbours; counts staged for the host
        rng = nvtx("exchange")
        rng.__enter__()
        if R > 1:
            self._pack(0, ci0)
            self._pack(1, ci0)
            comm.exchange_pair(self.send[0], self.send[1], self.recv[0], self.recv[1], self.part)
            hdr = self.recv[:, 0, :4].contiguous().view(torch.int32)  # (2, 4) headers
            self._stage[0:4].copy_(hdr[0])
            self._stage[4:8].copy_(hdr[1])
            self._stage[8:10].copy_(torch.index_select(ci0.cell_start, 0, self._cs_idx))
            self._stage_host.copy_(self._stage, non_blocking=True)
            self._ready.record()
        rng.__exit__(None, None, None)
        # 4. score training on R0 (gradient rows allreduced before every finalize)
        rng = nvtx("score")
        rng.__enter__()
        if self.trainer is not None:
            gid_sorted = b.gid[:n][ci0.perm[:n].long()] if self.trainer.mode() == 2 else None
            self.trainer.run(n, ci=ci0, flags=self.flags,
                             reduce_row=comm.allreduce_ if R > 1 else None,
                             gid=gid_sorted, n_global=self.n_global)
        # 5. the step's host sync (overlapped by the K-loop): received counts -> union
        if R > 1:
            self._ready.synchronize()
            self.host_syncs += 1
            s = self._stage_host.numpy()
            c_l, own_l, over_l = (int(t) for t in s[0:3])
            c_r, own_r, over_r = (int(t) for t in s[4:7])
            if over_l or over_r:
                raise RuntimeError(f"rank {comm.rank}: boundary message over capacity "
                                   f"({self.mcap} rows); raise msg_capacity")
            n_next = int(s[9] - s[8]) + own_l + own_r
            n_u = n + c_l + c_r
            b.ensure(n_u, n)
            for k, (cnt, at) in enumerate(((c_l, n), (c_r, n + c_l))):
                _lib.call("spic_dist_unpack", _lib.ptr(self.recv[k]), cnt, at, _lib.ptr(b.x),
                          _lib.ptr(b.vp), b.cap, dv, _lib.ptr(b.w), _lib.ptr(b.gid), st)
            ci = self._bin(b, n_u, self.idx)
        else:
            n_u, n_next, ci = n, n, ci0
            self.idx.ci, self.idx.cap = ci0, self.idx0.cap
        p_all = b.view(n_u, self.uniform_w)
        # 6. scores on the union
        if self.trainer is not None:
            self.est.estimate_sorted(ci, n_u)
        elif isinstance(self.est, BlobEstimator):
            blob_sorted(ci, p_all, g, self.est.bandwidth, self.flags, self.bad_pid, self.h_cell)
        else:
            raise TypeError("unsupported estimator for the device step engine")
        rng.__exit__(None, None, None)
        # 7. pair kernel over the owned targets, epilogue into the next step's buffers
        rng = nvtx("collide")
        rng.__enter__()
        if self.U.shape[1] < n_u:
            self.U = torch.empty(dv, _round_up(int(n_u * 1.25) + 1024, 64), dtype=torch.float32,
                                 device=self.dev)
        U = self.U[:, :n_u]
        buf, nb = _lib.scratch("pairs", _lib.query("spic_landau_range_scratch_bytes", n_u, g.M,
                                                    dv, self.opt.landau_split, self.lo, self.hi))
        ev = None
        if self.time_collision:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        _lib.call("spic_landau_range", _lib.ptr(ci.xv), _lib.ptr(ci.sw), n_u, dv,
                  _lib.ptr(ci.cell_start), _lib.ptr(ci.sub_start) if self.S > 1 else None, g.M,
                  self.S, float(g.eta), self.gamma, float(self.uniform_w), self.opt.landau_split,
                  self.lo, self.hi, _lib.ptr(U), _lib.ptr(buf), nb, st)
        if ev is not None:
            ev[1].record()
            self.collision_events.append(ev)
        nx = self.nxt
        nx.ensure(n_next, 0)
        _lib.call("spic_dist_epilogue", _lib.ptr(U), n_u, _lib.ptr(ci.sw), _lib.ptr(ci.perm),
                  _lib.ptr(ci.cell_start), self.lo, self.hi, dv, float(self.nu * self.dt),
                  _lib.ptr(b.x), _lib.ptr(b.vp), b.cap, _lib.ptr(b.w), _lib.ptr(b.gid),
                  _lib.ptr(nx.x), _lib.ptr(nx.vp), nx.cap, _lib.ptr(nx.w), _lib.ptr(nx.gid),
                  _lib.ptr(d[3:9]), _lib.ptr(self.flags), _lib.ptr(self._epi), self._epi_n, st)
        comm.allreduce_(d[3:9])
        rng.__exit__(None, None, None)
        self.cur, self.nxt = nx, b
        self.n = n_next

    # ---- host reads -------------------------------------------------------------------------
    def step_host(self, row: int, x_host: torch.Tensor, v_host: torch.Tensor,
                  diag_host: torch.Tensor) -> int:
        """End-to-end step of this rank on HOST buffers (pinned float32 x (cap,), v planes
        (dv, cap), float64 diag (DIAG_W,), cap >= the rank's particle count): H2D of the rank's
        current particles, one decomposed step, D2H of its particles after the step (their
        count changes with migration) and of the step's diagnostics row. Returns the count."""
        n = self.n
        if x_host.shape[0] < n or v_host.shape[1] < n:
            raise ValueError("host buffers smaller than the rank's particle count")
        self.cur.x[:n].copy_(x_host[:n], non_blocking=True)
        self.cur.vp[:, :n].copy_(v_host[:, :n], non_blocking=True)
        self.step(row)
        n = self.n
        if x_host.shape[0] < n or v_host.shape[1] < n:
            raise ValueError("host buffers smaller than the rank's particle count")
        x_host[:n].copy_(self.cur.x[:n], non_blocking=True)
        v_host[:, :n].copy_(self.cur.vp[:, :n], non_blocking=True)
        diag_host.copy_(self.diag[row], non_blocking=True)
        return n

    def check(self) -> None:
        """The reference's exception for any flag raised on any rank (one allreduce)."""
        fl = self.flags.clone()
        self.comm.allreduce_(fl, op="max")
        f = fl.cpu().numpy()
        if f[_lib.FLAG_ISOLATED]:
            bad = int(self.bad_pid.item())
            # the blob kernel reports the union plane index; after the epilogue the union
            # planes are the `nxt` buffers; report the particle's global id
            idx = int(self.nxt.gid[bad & 0xFFFFFFFF].item()) if bad != _NO_PID else -1
            raise ValueError(f"isolated particle in velocity space (particle {idx})")
        raise_for_flags(fl, self.f)
        row = getattr(self, "_last_row", None)
        if row is not None:
            sw, L = float(self.diag[row, 8].item()), self.grid.L
            if abs(sw - L) > 1e-5 * L:  # a particle lost in the exchange (see module doc)
                raise ValueError("total particle weight drifted from L")

    def records(self, rows, steps, times) -> list:
        D = self.diag[list(rows)].cpu().numpy()
        out = []
        for r, step, t in zip(D, steps, times):
            out.append(DiagnosticsRecord(step=int(step), t=float(t), E_K=float(r[4]),
                                         E_E=float(r[0]), E_B=float(r[1]),
                                         E_total=float(r[4] + r[0] + r[1]),
                                         H_dot=float(r[3]) if self.nu > 0 else 0.0,
                                         P=np.array(r[5:5 + self.dv]), E_l2=float(r[2])))
        return out

    def gather_state(self):
        """(gid, x, v) of this rank's own particles (host copies)."""
        n = self.n
        return (self.cur.gid[:n].cpu().numpy().astype(np.int64),
                self.cur.x[:n].double().cpu().numpy(),
                self.cur.vp[:, :n].t().double().cpu().numpy())

    # bench helpers: the rank's own records of the last step (live-pair counts)
    @property
    def ci_own(self):
        return self.idx0.ci

    @property
    def n_own(self) -> int:
        return getattr(self, "_n0", self.n)

    @property
    def buf(self) -> _Buffers:
        return self.cur
