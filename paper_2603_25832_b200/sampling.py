"""Initial conditions — one-time host setup.

Same distributions and the same PCG64 draw order as the reference samplers
(ref: sampling.py:11-107), so a seeded run starts from bit-identical float64 arrays, which
the device path then rounds to float32 once. Extension samplers for BASELINE config 3
(anisotropic Weibel state, seeded B3 noise) are at the end.
"""

from __future__ import annotations

import numpy as np


def _cdf_residual(x, u, alpha, k, L):
    return (x + (alpha / k) * np.sin(k * x)) / L - u


def sample_positions(n: int, alpha: float, k: float, L: float, rng: np.random.Generator):
    """x with density ~ 1 + alpha cos(kx) on [0, L): inverse CDF by Newton iteration to
    |residual| <= 1e-12 (at most 100 sweeps), bisection for any stragglers."""
    if not abs(alpha) < 1:
        raise ValueError("need |alpha| < 1")
    u = rng.random(n)
    x = u * L
    sweeps = 0
    while sweeps < 100:
        res = _cdf_residual(x, u, alpha, k, L)
        if np.all(np.abs(res) <= 1e-12):
            break
        x = x - L * res / (1.0 + alpha * np.cos(k * x))
        sweeps += 1
    stragglers = np.abs(_cdf_residual(x, u, alpha, k, L)) > 1e-12
    if stragglers.any():
        want = u[stragglers]
        a = np.zeros(want.size)
        b = np.full(want.size, L)
        for _ in range(200):
            c = 0.5 * (a + b)
            over = (c + (alpha / k) * np.sin(k * c)) / L > want
            a, b = np.where(over, a, c), np.where(over, c, b)
        x[stragglers] = 0.5 * (a + b)
    return np.clip(x, 0.0, np.nextafter(L, 0.0))


def _signed_offsets(rng, n, c):
    """Fair-coin +-c (one uniform draw per particle)."""
    return np.where(rng.random(n) < 0.5, c, -c)


def sample_velocities(n: int, preset: str, rng: np.random.Generator, *, dv: int, c: float = 0.0,
                      beta: float = 1.0):
    """Per-preset velocity laws, components drawn in a fixed order:
    landau_damping N(0,1)^dv; two_stream v1 = +-c + N(0,1), rest N(0,1);
    weibel v1 ~ N(0, beta/2), v2 = +-c + N(0, beta/2), rest N(0, beta/2)."""
    out = np.empty((n, dv))
    if preset == "landau_damping":
        for comp in range(dv):
            out[:, comp] = rng.normal(size=n)
    elif preset == "two_stream":
        out[:, 0] = _signed_offsets(rng, n, c) + rng.normal(size=n)
        for comp in range(1, dv):
            out[:, comp] = rng.normal(size=n)
    elif preset == "weibel":
        sd = np.sqrt(beta / 2.0)
        out[:, 0] = sd * rng.normal(size=n)
        out[:, 1] = _signed_offsets(rng, n, c) + sd * rng.normal(size=n)
        for comp in range(2, dv):
            out[:, comp] = sd * rng.normal(size=n)
    else:
        raise ValueError(f"unknown preset: {preset!r}")
    return out


def sample_arrays(config, rng: np.random.Generator):
    """(x, v, w) for a SimConfig: positions first, then velocities, equal weights L/n.
    'custom' samples like landau_damping; weibel is spatially uniform (alpha ignored)."""
    family = "landau_damping" if config.preset == "custom" else config.preset
    alpha = 0.0 if config.preset == "weibel" else config.alpha
    x = sample_positions(config.n, alpha, config.k, config.L, rng)
    v = sample_velocities(config.n, family, rng, dv=config.dv, c=config.c, beta=config.beta)
    return x, v, np.full(config.n, config.L / config.n)


# ---- extensions (BASELINE config 3) ---------------------------------------------

def anisotropic_ensemble(n: int, L: float, temps, rng: np.random.Generator, *, dv: int = 3):
    """x ~ U[0, L), v_k ~ N(0, T_k): a bi-Maxwellian (e.g. T_x = 0.01, T_y = T_z = 0.04)."""
    x = np.minimum(rng.uniform(0.0, L, n), np.nextafter(L, 0.0))
    v = np.column_stack([np.sqrt(temps[i]) * rng.normal(size=n) for i in range(dv)])
    return x, v, np.full(n, L / n)


def seeded_b3_noise(M: int, amplitude: float, rng: np.random.Generator) -> np.ndarray:
    """B3 at the cell centres = amplitude x N(0, 1) (seeded magnetic noise)."""
    return amplitude * rng.normal(size=M)
