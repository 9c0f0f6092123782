"""Domain-decomposed step engine: one process per GPU, cell ranges per rank.

Per step on rank r (owned cells [lo, hi)), same kernels as engine.Simulation:

    push (own particles) -> migrate to the owners of the new cells (all-to-all)
    bin own particles -> deposit -> allreduce(rho, J) -> field step (replicated fields)
    SBTM: K x (partials over own particles -> allreduce(reduced row) -> finalize)
    halo: records of cells lo and hi-1 -> left / right neighbours (1-cell halo)
    bin own + halo -> scores (SBTM forward over own + halo; blob over own, then a second
    halo exchange of the boundary scores) -> Landau pair kernel with targets in [lo, hi)
    -> epilogue over the owned sorted range -> allreduce([H_dot, E_K, P])

The exchanges use torch.distributed (NCCL on the box) on device tensors; the variable
migration/halo sizes cost a few small host reads per step.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .collision import CellIndex, auto_sub_cells, build_cell_index, landau_sorted
from .config import DeviceOptions
from .parallel import CellPartition, Comm
from .pic import FIELD_NONE, FIELD_VML, FIELD_VPL, Grid, deposit_from_index, raise_for_flags
from .score import BlobEstimator, SbtmEstimator, blob_sorted
from .state import DiagnosticsRecord, FieldState, ParticleEnsemble, new_flags

DIAG_W = 9


class _Buffers:
    """Capacity-managed particle arrays of one rank (own particles first, then halo)."""

    def __init__(self, cap: int, dv: int, dev):
        self.cap, self.dv, self.dev = cap, dv, dev
        self.x = torch.empty(cap, dtype=torch.float32, device=dev)
        self.vp = torch.empty(dv, cap, dtype=torch.float32, device=dev)
        self.w = torch.empty(cap, dtype=torch.float32, device=dev)
        self.gid = torch.empty(cap, dtype=torch.int64, device=dev)

    def ensure(self, need: int, keep: int) -> None:
        if need <= self.cap:
            return
        cap = int(need * 1.25) + 1024
        nb = _Buffers(cap, self.dv, self.dev)
        nb.x[:keep].copy_(self.x[:keep])
        nb.vp[:, :keep].copy_(self.vp[:, :keep])
        nb.w[:keep].copy_(self.w[:keep])
        nb.gid[:keep].copy_(self.gid[:keep])
        self.__dict__.update(nb.__dict__)

    def view(self, n: int, uniform_w: float) -> ParticleEnsemble:
        # planes with leading dimension cap: pass a (dv, n) view; kernels get ldv = cap
        return ParticleEnsemble(self.x[:n], self.vp[:, :n], self.w[:n], uniform_w)


def _new_ci(n: int, M: int, S: int, dev) -> CellIndex:
    return CellIndex(torch.empty(n, dtype=torch.int32, device=dev),
                     torch.empty(M + 1, dtype=torch.int32, device=dev),
                     torch.empty(M * S + 1, dtype=torch.int32, device=dev), M, S,
                     torch.empty(n, 4, dtype=torch.float32, device=dev),
                     torch.zeros(n, 4, dtype=torch.float32, device=dev))


class DistSimulation:
    def __init__(self, x, v, w, gid, fields: FieldState, grid: Grid, *, dt: float, nu: float,
                 mode: str, gamma: float, estimator=None, comm: Comm | None = None,
                 partition: CellPartition | None = None, n_global: int | None = None,
                 options: DeviceOptions | None = None, max_rows: int = 1024):
        self.comm = comm or Comm()
        self.grid, self.f = grid, fields
        self.dt, self.nu, self.mode, self.gamma = float(dt), float(nu), mode, float(gamma)
        self.est = estimator
        self.opt = options or DeviceOptions()
        dev = fields.E1.device
        self.dev = dev
        dv = v.shape[1]
        self.dv = dv
        n = x.shape[0]
        self.part = partition or CellPartition.equal(grid.M, self.comm.size)
        self.lo, self.hi = self.part.owned(self.comm.rank)
        self.owner = torch.as_tensor(self.part.owner_table(), dtype=torch.int64, device=dev)
        self.n_global = n_global or n
        self.uniform_w = float(w[0]) if n and bool(torch.all(torch.as_tensor(w) == w[0])) else 0.0
        self.buf = _Buffers(max(1024, int(1.5 * n)), dv, dev)
        self.n = n
        self.buf.x[:n].copy_(torch.as_tensor(x, dtype=torch.float32))
        self.buf.vp[:, :n].copy_(torch.as_tensor(v, dtype=torch.float32).t())
        self.buf.w[:n].copy_(torch.as_tensor(w, dtype=torch.float32))
        self.buf.gid[:n].copy_(torch.as_tensor(gid, dtype=torch.int64))
        self.S = self.opt.sub_cells or auto_sub_cells(max(self.n_global, 1), grid.M)
        self.flags = new_flags(dev)
        self.bad_pid = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
        self.h_cell = torch.empty(grid.M, dtype=torch.float32, device=dev)
        self.diag = torch.zeros(max_rows, DIAG_W, dtype=torch.float64, device=dev)
        self.trainer = None
        if isinstance(estimator, SbtmEstimator):
            self.trainer = estimator.make_trainer()
        self._epi, self._epi_n = _lib.scratch("epilogue", 8 * 2 * 148 * 5 + 64)
        self.time_collision = False
        self.collision_events: list = []
        self.rho = torch.zeros(grid.M, dtype=torch.float64, device=dev)
        self.J = torch.zeros(dv, grid.M, dtype=torch.float64, device=dev)

    # ---- helpers ----------------------------------------------------------------------------
    def _bin(self, n: int) -> CellIndex:
        ci = _new_ci(max(n, 1), self.grid.M, self.S, self.dev)
        p = self.buf.view(n, self.uniform_w)
        buf, nb = _lib.scratch("bin", _lib.query("spic_bin_scratch_bytes", n, self.grid.M, self.S))
        _lib.call("spic_bin", _lib.ptr(p.x), _lib.ptr(self.buf.vp), self.buf.cap, _lib.ptr(p.w), n,
                  self.dv, float(self.grid.eta), self.grid.M, self.S, _lib.ptr(ci.perm),
                  _lib.ptr(ci.cell_start), _lib.ptr(ci.sub_start), _lib.ptr(ci.xv), _lib.ptr(ci.sw),
                  _lib.ptr(buf), nb, _lib.stream_handle())
        return ci

    def _migrate(self) -> None:
        comm, n, b = self.comm, self.n, self.buf
        if comm.size == 1:
            return
        cells = self.grid.cell_of(b.x[:n])
        dest = self.owner[cells.long()]
        order = torch.argsort(dest, stable=True)
        counts = torch.bincount(dest, minlength=comm.size)
        rows = torch.cat([b.x[:n, None], b.vp[:, :n].t(), b.w[:n, None]], dim=1)[order]
        gids = b.gid[:n][order]
        rrows = comm.alltoallv(rows, counts)
        rgid = comm.alltoallv(gids, counts)
        m = rrows.shape[0]
        b.ensure(m, 0)
        b.x[:m].copy_(rrows[:, 0])
        b.vp[:, :m].copy_(rrows[:, 1:1 + self.dv].t())
        b.w[:m].copy_(rrows[:, 1 + self.dv])
        b.gid[:m].copy_(rgid)
        self.n = m

    def _halo_rows(self, ci: CellIndex, cs: np.ndarray):
        lo, hi = self.lo, self.hi
        first = torch.cat([ci.xv[int(cs[lo]):int(cs[lo + 1])], ci.sw[int(cs[lo]):int(cs[lo + 1])]], 1)
        last = torch.cat([ci.xv[int(cs[hi - 1]):int(cs[hi])], ci.sw[int(cs[hi - 1]):int(cs[hi])]], 1)
        return first, last

    # ---- one step ---------------------------------------------------------------------------
    def step(self, row: int) -> None:
        g, f, b, comm = self.grid, self.f, self.buf, self.comm
        dv, st = self.dv, _lib.stream_handle()
        d = self.diag[row]
        d.zero_()
        # 1. push own particles
        _lib.call("spic_push", _lib.ptr(b.x), _lib.ptr(b.vp), b.cap, self.n, dv, _lib.ptr(f.E1),
                  _lib.ptr(f.E2), _lib.ptr(f.B3), g.M, float(g.eta), self.dt, _lib.ptr(self.flags), st)
        # 2. migrate to the owners of the new cells
        self._migrate()
        n = self.n
        p_own = self.buf.view(n, self.uniform_w)
        # 3. bin own particles, deposit, allreduce the grid moments, field step
        ci = self._bin(n)
        self.ci_own, self.n_own = ci, n  # own particles only (bench: live-pair count)
        deposit_from_index(ci, p_own, g, fields=FieldState(f.E1, f.E2, f.B3, self.rho, self.J,
                                                           f.rho_ion),
                           field_mode=FIELD_NONE, flags=self.flags)
        comm.allreduce_(self.rho)
        comm.allreduce_(self.J)
        f.rho.copy_(self.rho)
        f.J.copy_(self.J)
        fmode = FIELD_VML if self.mode == "VML" else FIELD_VPL
        _lib.call("spic_field_step", _lib.ptr(f.E1), _lib.ptr(f.E2), _lib.ptr(f.B3), _lib.ptr(f.J),
                  g.M, float(g.eta), self.dt, fmode, _lib.ptr(d[0:3]), _lib.ptr(self.flags), st)
        if not (self.nu > 0 and self.est is not None):
            buf, nb = _lib.scratch("moments", _lib.query("spic_moments_scratch_bytes", n))
            _lib.call("spic_moments", _lib.ptr(b.vp), b.cap, _lib.ptr(b.w), n, dv,
                      float(self.uniform_w), _lib.ptr(d[4:9]), _lib.ptr(self.flags), _lib.ptr(buf),
                      nb, st)
            comm.allreduce_(d[3:9])
            return
        # 4. SBTM training on own particles, gradient rows allreduced before every finalize
        if self.trainer is not None:
            gid_sorted = b.gid[:n][ci.perm.long()].to(torch.int32) \
                if self.trainer.mode() == 2 else None
            self.trainer.run(n, ci=ci, flags=self.flags,
                             reduce_row=comm.allreduce_ if comm.size > 1 else None,
                             gid=gid_sorted, n_global=self.n_global)
        # 5. halo exchange of the boundary cells
        cs = ci.cell_start.cpu().numpy()
        h = 0
        if comm.size > 1:
            first, last = self._halo_rows(ci, cs)
            from_left, from_right = comm.exchange_halo(first, last, self.part)
            hl, hr = self.part.halo_cells(comm.rank)
            halo = from_left if hl == hr else torch.cat([from_left, from_right], 0)
            h = halo.shape[0]
            b.ensure(n + h, n)
            if h:
                L = float(g.L)
                hx = halo[:, 0]
                b.x[n:n + h].copy_(torch.where(hx < 0, hx + L, hx))
                b.vp[:, n:n + h].copy_(halo[:, 1:1 + dv].t())
                b.w[n:n + h].copy_(halo[:, 7])
        # 6. bin own + halo, scores, pair kernel over own targets, epilogue
        ci2 = self._bin(n + h) if h else ci
        p_all = self.buf.view(n + h, self.uniform_w)
        if self.trainer is not None:
            self.est.estimate_sorted(ci2, n + h)
        elif isinstance(self.est, BlobEstimator):
            blob_sorted(ci2, p_all, g, self.est.bandwidth, self.flags, self.bad_pid, self.h_cell)
            if comm.size > 1:  # halo particles' scores come from their owners
                cs2 = ci2.cell_start.cpu().numpy()
                first, last = self._halo_rows(ci2, cs2)
                from_left, from_right = comm.exchange_halo(first, last, self.part)
                hl, hr = self.part.halo_cells(comm.rank)
                for cell, rows in ((hl, from_left), (hr, from_right)):
                    a, z = int(cs2[cell]), int(cs2[cell + 1])
                    if z > a and rows.shape[0] == z - a:
                        ci2.sw[a:z, :3].copy_(rows[:, 4:7])
                    if hl == hr:
                        break
        else:
            raise TypeError("unsupported estimator for the device step engine")
        ntot = n + h
        U = torch.empty(dv, max(ntot, 1), dtype=torch.float32, device=self.dev)
        buf, nb = _lib.scratch("pairs", _lib.query("spic_landau_scratch_bytes", ntot, g.M, dv,
                                                    self.opt.landau_split))
        ev = None
        if self.time_collision:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        _lib.call("spic_landau_range", _lib.ptr(ci2.xv), _lib.ptr(ci2.sw), ntot, dv,
                  _lib.ptr(ci2.cell_start), _lib.ptr(ci2.sub_start) if self.S > 1 else None, g.M,
                  self.S, float(g.eta), self.gamma, float(self.uniform_w), self.opt.landau_split,
                  self.lo, self.hi, _lib.ptr(U), _lib.ptr(buf), nb, st)
        if ev is not None:
            ev[1].record()
            self.collision_events.append(ev)
        cs2 = ci2.cell_start.cpu().numpy() if h else cs
        k0, k1 = int(cs2[self.lo]), int(cs2[self.hi])
        _lib.call("spic_collision_epilogue_range", _lib.ptr(U), _lib.ptr(ci2.sw), _lib.ptr(ci2.perm),
                  ntot, dv, k0, k1, float(self.nu * self.dt), _lib.ptr(b.vp), b.cap, None, ntot,
                  _lib.ptr(d[3:8]), _lib.ptr(self.flags), _lib.ptr(self._epi), self._epi_n, st)
        comm.allreduce_(d[3:8])

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
        self.buf.x[:n].copy_(x_host[:n], non_blocking=True)
        self.buf.vp[:, :n].copy_(v_host[:, :n], non_blocking=True)
        self.step(row)
        n = self.n
        if x_host.shape[0] < n or v_host.shape[1] < n:
            raise ValueError("host buffers smaller than the rank's particle count")
        x_host[:n].copy_(self.buf.x[:n], non_blocking=True)
        v_host[:, :n].copy_(self.buf.vp[:, :n], non_blocking=True)
        diag_host.copy_(self.diag[row], non_blocking=True)
        return n

    def check(self) -> None:
        fl = self.flags.clone()
        if self.comm.size > 1:
            import torch.distributed as dist

            dist.all_reduce(fl, op=dist.ReduceOp.MAX, group=self.comm.group)
        f = fl.cpu().numpy()
        if f[_lib.FLAG_ISOLATED]:
            idx = int(self.bad_pid.item()) & 0xFFFFFFFF
            raise ValueError(f"isolated particle in velocity space (particle {idx})")
        raise_for_flags(fl, self.f)

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
        return (self.buf.gid[:n].cpu().numpy(), self.buf.x[:n].double().cpu().numpy(),
                self.buf.vp[:, :n].t().double().cpu().numpy())
