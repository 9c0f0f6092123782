"""Initial conditions (one-time host setup).

Restates the reference samplers (ref: sampling.py:11-107) with the identical PCG64 draw
order, so a seeded run starts from bit-identical float64 ensembles; the product then rounds
them to float32 once on upload. The extension sampler `anisotropic_ensemble` provides the
BASELINE config-3 Weibel initial state (bi-Maxwellian + seeded B3 noise), which
the reference presets cannot express.
"""

from __future__ import annotations

import numpy as np


def sample_positions(n: int, alpha: float, k: float, L: float, rng: np.random.Generator):
    """Inverse CDF of F(x) = (x + (alpha/k) sin kx)/L: Newton to 1e-12, bisection fallback."""
    if not abs(alpha) < 1:
        raise ValueError("need |alpha| < 1")
    u = rng.random(n)

    def resid(x):
        return (x + (alpha / k) * np.sin(k * x)) / L - u

    x = L * u
    for _ in range(100):
        r = resid(x)
        if np.all(np.abs(r) <= 1e-12):
            break
        x = x - r * L / (1.0 + alpha * np.cos(k * x))
    bad = np.abs(resid(x)) > 1e-12
    if np.any(bad):
        target = u[bad]
        lo, hi = np.zeros(target.size), np.full(target.size, L)
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            above = (mid + (alpha / k) * np.sin(k * mid)) / L > target
            lo, hi = np.where(above, lo, mid), np.where(above, mid, hi)
        x[bad] = 0.5 * (lo + hi)
    return np.clip(x, 0.0, np.nextafter(L, 0.0))


def sample_velocities(n: int, preset: str, rng: np.random.Generator, *, dv: int, c: float = 0.0,
                      beta: float = 1.0):
    v = np.empty((n, dv))
    if preset == "landau_damping":
        for i in range(dv):
            v[:, i] = rng.normal(size=n)
        return v
    if preset == "two_stream":
        v[:, 0] = np.where(rng.random(n) < 0.5, c, -c) + rng.normal(size=n)
        for i in range(1, dv):
            v[:, i] = rng.normal(size=n)
        return v
    if preset == "weibel":
        sd = np.sqrt(beta / 2.0)
        v[:, 0] = sd * rng.normal(size=n)
        v[:, 1] = np.where(rng.random(n) < 0.5, c, -c) + sd * rng.normal(size=n)
        for i in range(2, dv):
            v[:, i] = sd * rng.normal(size=n)
        return v
    raise ValueError(f"unknown preset: {preset!r}")


def sample_arrays(config, rng: np.random.Generator):
    """(x, v, w) float64 host arrays, positions first then velocities (ref: sampling.py:74-87)."""
    preset = "landau_damping" if config.preset == "custom" else config.preset
    alpha = 0.0 if config.preset == "weibel" else config.alpha
    x = sample_positions(config.n, alpha, config.k, config.L, rng)
    v = sample_velocities(config.n, preset, rng, dv=config.dv, c=config.c, beta=config.beta)
    return x, v, np.full(config.n, config.L / config.n)


def anisotropic_ensemble(n: int, L: float, temps, rng: np.random.Generator, *, dv: int = 3):
    """Extension (BASELINE config 3): x ~ U[0, L), v_k ~ N(0, T_k) (bi-Maxwellian)."""
    x = np.minimum(rng.uniform(0.0, L, n), np.nextafter(L, 0.0))
    v = np.empty((n, dv))
    for i in range(dv):
        v[:, i] = np.sqrt(temps[i]) * rng.normal(size=n)
    return x, v, np.full(n, L / n)


def seeded_b3_noise(M: int, amplitude: float, rng: np.random.Generator) -> np.ndarray:
    """Extension (BASELINE config 3): B3 at the cell centres = amplitude x N(0, 1) noise."""
    return amplitude * rng.normal(size=M)
