"""The per-timestep hot path as one fixed sequence of sm_100a kernels (no host syncs).

Algorithm 1 of the reference (ref: run.py:81-118) re-ordered for the device without changing
results: the binning that the reference does before the score update is done right after the
position advance, so the deposit, the estimator and the collision all read the same
cell-sorted float4 records.

    push         spic_push            interpolate + Lorentz + advance + wrap (pid order)
    bin          spic_bin             (cell, sub-cell) counting sort + gather -> records
    deposit      spic_deposit_field   rho, J, field step, E_E/E_B/E_l2
    score        SBTM: K x (spic_ism_partials_ex + spic_sbtm_finalize_ex), spic_mlp_forward
                 blob: spic_blob
    collide      spic_landau (+ fold) + spic_collision_epilogue (v -= nu dt U, H_dot, E_K, P)
    (nu == 0)    spic_moments         E_K, P

Diagnostics land in a device table `diag[row]` = [E_E, E_B, E_l2, H_dot, E_K, P0, P1, P2, sw];
error conditions in `flags`. The host reads both only when asked (`records`, `check`).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from .collision import CellIndex, auto_sub_cells, build_cell_index, landau_sorted
from .config import DeviceOptions
from .pic import FIELD_VML, FIELD_VPL, Grid, deposit_from_index, raise_for_flags
from .score import BlobEstimator, SbtmEstimator, blob_sorted
from .state import DiagnosticsRecord, FieldState, ParticleEnsemble, new_flags

DIAG_W = 9


class _Nvtx:
    """Per-stage NVTX ranges (SURVEY §5 tracing; the reference's stage hook is run.py:83-105):
    named ranges "push", "bin", "deposit", "score", "collide" around each stage's launches,
    visible in nsys / ncu --nvtx timelines. Off unless SPIC_NVTX=1 (host-side markers only,
    nothing is added to the device stream or to a captured graph)."""

    def __call__(self, name: str):
        return torch.cuda.nvtx.range(name) if os.environ.get("SPIC_NVTX") == "1" else _NullCtx()


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


nvtx = _Nvtx()


class Simulation:
    def __init__(self, particles: ParticleEnsemble, fields: FieldState, grid: Grid, *, dt: float,
                 nu: float, mode: str, gamma: float, estimator=None,
                 options: DeviceOptions | None = None, max_rows: int = 1024):
        self.p, self.f, self.grid = particles, fields, grid
        self.dt, self.nu, self.mode, self.gamma = float(dt), float(nu), mode, float(gamma)
        self.est = estimator
        self.opt = options or DeviceOptions()
        n, dv, M = particles.n, particles.dv, grid.M
        dev = particles.x.device
        self.S = self.opt.sub_cells or auto_sub_cells(n, M)
        self.ci = CellIndex(torch.empty(n, dtype=torch.int32, device=dev),
                            torch.empty(M + 1, dtype=torch.int32, device=dev),
                            torch.empty(M * self.S + 1, dtype=torch.int32, device=dev), M, self.S,
                            torch.empty(n, 4, dtype=torch.float32, device=dev),
                            torch.zeros(n, 4, dtype=torch.float32, device=dev))
        self.U_sorted = torch.empty(dv, n, dtype=torch.float32, device=dev)
        self.flags = new_flags(dev)
        self.bad_pid = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
        self.h_cell = torch.empty(M, dtype=torch.float32, device=dev)
        self.diag = torch.zeros(max_rows, DIAG_W, dtype=torch.float64, device=dev)
        self.trainer = None
        if isinstance(estimator, SbtmEstimator):
            self.trainer = estimator.make_trainer()
        # optional CUDA-event brackets around the pair kernel (bench instrumentation)
        self.time_collision = False
        self.collision_events: list = []
        # epilogue scratch
        self._epi, self._epi_n = _lib.scratch("epilogue", 8 * 2 * 148 * 5 + 64)

    # ---- CUDA graph of one step --------------------------------------------------------------
    def capture(self, row: int = 0) -> None:
        """Capture one step (into diag[row]) as a CUDA graph; replay() then costs one launch.
        Call after at least one eager step (scratch buffers sized). Per-particle Hutchinson
        probes are drawn on the host per ISM step and cannot be captured."""
        if self.trainer is not None and self.trainer.mode() == 2:
            raise RuntimeError("per-particle Rademacher probes need the eager step")
        self._graph_row = row
        torch.cuda.synchronize()
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self.step(row, draw=False)
        torch.cuda.synchronize()

    def replay(self, row: int | None = None) -> None:
        """One captured step; its diagnostics row is copied to diag[row] if given."""
        if self.trainer is not None:
            self.trainer.draw_shared_probes()
        self._graph.replay()
        if self.trainer is not None and self.trainer.mode() == 1:
            self.trainer._z_free.record()
        if row is not None and row != self._graph_row:
            self.diag[row].copy_(self.diag[self._graph_row])

    # ---- one step ---------------------------------------------------------------------------
    def step(self, row: int, draw: bool = True, after_push=None) -> None:
        p, g, ci, f = self.p, self.grid, self.ci, self.f
        n, dv = p.n, p.dv
        st = _lib.stream_handle()
        with nvtx("push"):
            _lib.call("spic_push", _lib.ptr(p.x), _lib.ptr(p.vp), n, n, dv, _lib.ptr(f.E1),
                      _lib.ptr(f.E2), _lib.ptr(f.B3), g.M, float(g.eta), self.dt,
                      _lib.ptr(self.flags), st)
        if after_push is not None:  # the positions are final from here on (step_host)
            after_push()
        with nvtx("bin"):
            build_cell_index(p, g, self.S, out=ci)
        d = self.diag[row]
        d.zero_()
        fmode = FIELD_VML if self.mode == "VML" else FIELD_VPL
        with nvtx("deposit"):
            deposit_from_index(ci, p, g, fields=f, field_mode=fmode, dt=self.dt, diag_out=d[0:3],
                               flags=self.flags)
        if self.nu > 0 and self.est is not None:
            with nvtx("score"):
                if self.trainer is not None:
                    self.trainer.run(n, ci=ci, flags=self.flags, draw=draw)
                    self.est.estimate_sorted(ci, n)
                elif isinstance(self.est, BlobEstimator):
                    blob_sorted(ci, p, g, self.est.bandwidth, self.flags, self.bad_pid,
                                self.h_cell)
                else:
                    raise TypeError("unsupported estimator for the device step engine")
            collide = nvtx("collide")
            collide.__enter__()
            ev = None
            if self.time_collision:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            landau_sorted(ci, p, g, self.gamma, self.U_sorted, nsplit=self.opt.landau_split)
            if ev is not None:
                ev[1].record()
                self.collision_events.append(ev)
            _lib.call("spic_collision_epilogue", _lib.ptr(self.U_sorted), _lib.ptr(ci.sw),
                      _lib.ptr(ci.perm), n, dv, float(self.nu * self.dt), _lib.ptr(p.vp), n, None,
                      n, _lib.ptr(d[3:8]), _lib.ptr(self.flags), _lib.ptr(self._epi), self._epi_n,
                      st)
            collide.__exit__(None, None, None)
        else:
            buf, nb = _lib.scratch("moments", _lib.query("spic_moments_scratch_bytes", n))
            _lib.call("spic_moments", _lib.ptr(p.vp), n, _lib.ptr(p.w), n, dv, float(p.uniform_w),
                      _lib.ptr(d[4:9]), _lib.ptr(self.flags), _lib.ptr(buf), nb, st)

    def step_host(self, row: int, x_host: torch.Tensor, v_host: torch.Tensor,
                  diag_host: torch.Tensor, flags_host: torch.Tensor | None = None) -> None:
        """Public end-to-end step on HOST buffers (pinned float32 x (n,), v planes (dv, n),
        float64 diag (DIAG_W,)): H2D of the state, one device step, D2H of the updated state,
        of the step's diagnostics row and (if given, pinned int32 (8,)) of the error flags —
        all enqueued on (or joined into) the current stream; check_host(flags_host) after a sync raises the
        reference's exception for the step, as run() does once per step."""
        self.p.x.copy_(x_host, non_blocking=True)
        self.p.vp.copy_(v_host, non_blocking=True)
        # the push leaves the step's final positions: their D2H copy runs on a second stream
        # under the rest of the step (binning, deposit, score, collision only read x)
        main = torch.cuda.current_stream()
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream()
            self._ev_push, self._ev_xcopy = torch.cuda.Event(), torch.cuda.Event()

        def copy_x():
            self._ev_push.record(main)
            self._copy_stream.wait_event(self._ev_push)
            with torch.cuda.stream(self._copy_stream):
                x_host.copy_(self.p.x, non_blocking=True)
                self._ev_xcopy.record(self._copy_stream)

        self.step(row, after_push=copy_x)
        main.wait_event(self._ev_xcopy)  # a sync on the current stream covers the x copy
        v_host.copy_(self.p.vp, non_blocking=True)
        diag_host.copy_(self.diag[row], non_blocking=True)
        if flags_host is not None:
            flags_host.copy_(self.flags, non_blocking=True)

    # ---- host reads -------------------------------------------------------------------------
    def check(self) -> None:
        """Raise the reference's exception for any flagged condition (one D2H read)."""
        f = self.flags.cpu().numpy()
        if f[_lib.FLAG_ISOLATED]:
            idx = int(self.bad_pid.item()) & 0xFFFFFFFF
            raise ValueError(f"isolated particle in velocity space (particle {idx})")
        raise_for_flags(self.flags, self.f)

    def check_host(self, flags_host) -> None:
        """check() on a host copy of the flags (e.g. the one step_host() fills), no D2H read."""
        if flags_host[_lib.FLAG_ISOLATED]:
            self.check()
        raise_for_flags(flags_host, self.f)

    def lr_halvings(self) -> int:
        return int(self.flags[_lib.FLAG_LR_HALVINGS].item())

    def records(self, rows, steps, times) -> list:
        D = self.diag[list(rows)].cpu().numpy()
        dv = self.p.dv
        out = []
        for r, step, t in zip(D, steps, times):
            E_E, E_B, E_l2, H_dot, E_K = r[0], r[1], r[2], r[3], r[4]
            out.append(DiagnosticsRecord(step=int(step), t=float(t), E_K=float(E_K),
                                         E_E=float(E_E), E_B=float(E_B),
                                         E_total=float(E_K + E_E + E_B),
                                         H_dot=float(H_dot) if self.nu > 0 else 0.0,
                                         P=np.array(r[5:5 + dv]), E_l2=float(E_l2)))
        return out
