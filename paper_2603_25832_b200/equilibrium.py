"""Analytic t = 0 scores used to pretrain the SBTM network (ref: equilibrium.py:55-79).

grad_v log f0 for the presets, evaluated on device tensors (n, dv):
landau_damping: -v; two_stream: v1 from the equal N(+-c, 1) mixture, -v elsewhere;
weibel: -v / (beta/2) with v2 from the N(+-c, beta/2) mixture. The mixture score uses the
stable closed form (-u + c tanh(u c / var)) / var.
"""

from __future__ import annotations

import torch


def _mixture(u: torch.Tensor, c: float, var: float) -> torch.Tensor:
    return (-u + c * torch.tanh(u * (c / var))) / var


def analytic_initial_score(preset: str, v: torch.Tensor, *, c: float = 0.0,
                           beta: float = 1.0) -> torch.Tensor:
    if preset == "landau_damping":
        return -v
    if preset == "two_stream":
        s = -v.clone()
        s[:, 0] = _mixture(v[:, 0], c, 1.0)
        return s
    if preset == "weibel":
        var = beta / 2.0
        s = -v / var
        s[:, 1] = _mixture(v[:, 1], c, var)
        return s
    raise ValueError(f"unknown preset: {preset!r}")
