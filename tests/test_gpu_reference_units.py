"""The reference's unit tests of the hot-path operators (ref: pkg/tests/test_pic.py,
test_collision.py) restated against this package's device API, so the GPU suite checks the
same behaviours the reference checks, case by case.

Particle state is float32 on the device (grid quantities float64), so where the reference
asserts 1e-14-1e-15 on particle arithmetic the bound here is float32 rounding (stated per
test); grid-only operators (field steps, Poisson) keep float64 bounds.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F32 = 4e-7  # a few float32 ulps, relative


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_25832_b200 import _lib

    _lib.load()
    return _lib


def ens(x, v, w):
    from paper_2603_25832_b200.state import ParticleEnsemble

    return ParticleEnsemble.from_arrays(np.asarray(x, float), np.asarray(v, float),
                                        np.asarray(w, float))


def grid_of(L, M):
    from paper_2603_25832_b200.pic import Grid

    return Grid(M, L / M)


def npy(t):
    return t.double().cpu().numpy()


# ---------------------------------------------------------------------------------- Grid
def test_grid_centers_and_cell_of_clip(lib):
    for M in (1, 2, 7, 100):
        g = grid_of(4 * math.pi, M)
        c = g.centers
        assert c.shape == (M,) and c[-1] < g.L and c[0] == pytest.approx(g.eta / 2)
        if M > 1:
            assert np.all(np.diff(c) > 0)
    g = grid_of(10.0, 10)
    x = torch.tensor([np.nextafter(np.float32(10.0), np.float32(0.0))], dtype=torch.float32,
                     device="cuda")
    assert int(g.cell_of(x)[0]) == 9


# ------------------------------------------------------------------------------- Deposit
def test_deposit_particle_at_center_and_between_centers(lib):
    from paper_2603_25832_b200.pic import deposit

    g = grid_of(8.0, 8)
    rho, J = deposit(ens([g.centers[3]], [[0.5, 0.0]], [1.0]), g)
    exp = np.zeros(8)
    exp[3] = 1.0 / g.eta
    np.testing.assert_allclose(npy(rho), exp, atol=1e-6)
    np.testing.assert_allclose(npy(J)[0], 0.5 * exp, atol=1e-6)
    x = 0.5 * (g.centers[2] + g.centers[3])
    rho, _ = deposit(ens([x], [[0.0, 0.0]], [1.0]), g)
    r = npy(rho)
    assert r[2] == pytest.approx(0.5 / g.eta, rel=F32) and r[3] == pytest.approx(0.5 / g.eta, rel=F32)
    assert r.sum() * g.eta == pytest.approx(1.0, rel=F32)


def test_deposit_uniform_particles_give_unit_density(lib):
    from paper_2603_25832_b200.pic import deposit

    g = grid_of(10.0, 10)
    n = 10 * g.M
    x = (np.arange(n) + 0.5) * g.L / n
    rho, _ = deposit(ens(x, np.zeros((n, 2)), np.full(n, g.L / n)), g)
    np.testing.assert_allclose(npy(rho), 1.0, atol=1e-6)


def test_deposit_matches_brute_force_and_conserves(lib):
    """Cloud-in-cell onto the two nearest centres (periodic), by an explicit per-particle
    loop in float64 on the float32 inputs (the reference's brute_deposit construction)."""
    from paper_2603_25832_b200.pic import deposit

    rng = np.random.default_rng(0)
    g = grid_of(5.0, 7)
    n = 40
    x = rng.uniform(0, g.L, n).astype(np.float32).astype(np.float64)
    v = rng.normal(size=(n, 3)).astype(np.float32).astype(np.float64)
    w = np.full(n, g.L / n)
    rho, J = deposit(ens(x, v, w), g)
    rho_ref, J_ref = np.zeros(g.M), np.zeros((3, g.M))
    for xi, vi, wi in zip(x, v, w):
        s = xi / g.eta - 0.5
        j0 = math.floor(s)
        f = s - j0
        for j, wt in ((j0 % g.M, 1 - f), ((j0 + 1) % g.M, f)):
            rho_ref[j] += wi * wt / g.eta
            J_ref[:, j] += wi * wt * vi / g.eta
    np.testing.assert_allclose(npy(rho), rho_ref, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(npy(J), J_ref, rtol=1e-5, atol=1e-6)
    rng = np.random.default_rng(1)
    g = grid_of(4 * math.pi, 16)
    n = 5000
    x = rng.uniform(0, g.L, n).astype(np.float32).astype(np.float64)
    v = rng.normal(size=(n, 3)).astype(np.float32).astype(np.float64)
    w = np.full(n, g.L / n)
    rho, J = deposit(ens(x, v, w), g)
    # the CIC weights (1 - f) + f and the products w v are formed in float32 per particle, the
    # sums in float64: totals agree to float32 rounding of the terms
    wf = np.float64(np.float32(g.L / n))
    assert g.eta * npy(rho).sum() == pytest.approx(n * wf, rel=1e-6)
    for i in range(3):
        scale = float(wf * np.abs(v[:, i]).sum())
        assert g.eta * npy(J)[i].sum() == pytest.approx(float(wf * v[:, i].sum()), abs=1e-6 * scale)


# --------------------------------------------------------------------------- Interpolate
def test_interpolate_uniform_center_and_midpoint(lib):
    from paper_2603_25832_b200.pic import interpolate_fields
    from paper_2603_25832_b200.state import FieldState

    g = grid_of(6.0, 6)
    rng = np.random.default_rng(2)
    f = FieldState.zeros(g.M, 2)
    f.E1.fill_(3.25)
    Ep, _ = interpolate_fields(ens(rng.uniform(0, g.L, 100), np.zeros((100, 2)),
                                   np.full(100, g.L / 100)), f, g)
    np.testing.assert_allclose(npy(Ep)[:, 0], 3.25, rtol=F32)
    f.E1.copy_(torch.arange(6.0, dtype=torch.float64))
    Ep, _ = interpolate_fields(ens([g.centers[4]], [[0.0, 0.0]], [1.0]), f, g)
    assert float(Ep[0, 0]) == pytest.approx(4.0, abs=1e-5)  # x rounded to float32
    f.E1.copy_(torch.tensor([0.0, 2.0, 10.0, 4.0, 0.0, 0.0], dtype=torch.float64))
    Ep, _ = interpolate_fields(ens([0.5 * (g.centers[1] + g.centers[2])], [[0.0, 0.0]], [1.0]), f, g)
    assert float(Ep[0, 0]) == pytest.approx(6.0, abs=1e-5)


# -------------------------------------------------------------------------------- Push
def test_lorentz_push_cases(lib):
    from paper_2603_25832_b200.pic import lorentz_push

    p = ens([1.0], [[1.0, 2.0, 3.0]], [1.0])
    lorentz_push(p, np.zeros((1, 3)), np.zeros((1, 3)), 0.1)
    np.testing.assert_allclose(npy(p.v), [[1.0, 2.0, 3.0]])
    p = ens([0.0], [[1.0, 0.0, 0.0]], [1.0])  # (v x B)_2 = -v1 B3
    lorentz_push(p, np.zeros((1, 3)), np.array([[0.0, 0.0, 1.0]]), 0.1)
    np.testing.assert_allclose(npy(p.v), [[1.0, -0.1, 0.0]], atol=1e-7)
    p = ens([0.0], [[0.0, 2.0, 0.0]], [1.0])  # E + v x B = (1 + v2 B3, -v1 B3, 0)
    lorentz_push(p, np.array([[1.0, 0.0, 0.0]]), np.array([[0.0, 0.0, 0.5]]), 0.2)
    np.testing.assert_allclose(npy(p.v), [[0.4, 2.0, 0.0]], atol=1e-7)
    p = ens([0.0], [[1.0, 0.0]], [1.0])  # dv = 2 drops the third component
    lorentz_push(p, np.zeros((1, 2)), np.array([[0.0, 0.0, 1.0]]), 0.1)
    np.testing.assert_allclose(npy(p.v), [[1.0, -0.1]], atol=1e-7)


def test_advance_positions_cases(lib):
    from paper_2603_25832_b200.pic import advance_positions

    p = ens([2.0], [[0.0, 1.0]], [1.0])
    advance_positions(p, 0.1, 10.0)
    assert float(p.x[0]) == 2.0
    eps = 1e-3
    p = ens([10.0 - eps], [[2 * eps / 0.1, 0.0]], [1.0])
    advance_positions(p, 0.1, 10.0)
    assert float(p.x[0]) == pytest.approx(eps, abs=2e-6)  # float32 x near L: ulp(10) ~ 1e-6
    p = ens([1.0], [[2.0, 0.0]], [1.0])
    advance_positions(p, 0.05, 10.0)
    assert float(p.x[0]) == pytest.approx(1.1, rel=F32)


# ------------------------------------------------------------------------- Field steps
def test_maxwell_step_cases(lib):
    from paper_2603_25832_b200.pic import maxwell_step
    from paper_2603_25832_b200.state import FieldState

    def fs(M, E2=None, B3=None):
        f = FieldState.zeros(M, 3)
        if E2 is not None:
            f.E2.copy_(torch.as_tensor(E2, dtype=torch.float64))
        if B3 is not None:
            f.B3.copy_(torch.as_tensor(B3, dtype=torch.float64))
        return f

    J0 = lambda M: torch.zeros(3, M, dtype=torch.float64, device="cuda")  # noqa: E731
    g = grid_of(2 * math.pi, 32)
    f = fs(32, B3=np.full(32, 0.7))
    maxwell_step(f, J0(32), 0.1, g)
    assert np.allclose(npy(f.E1), 0.0) and np.allclose(npy(f.E2), 0.0)
    np.testing.assert_allclose(npy(f.B3), 0.7)
    g = grid_of(2 * math.pi, 16)
    f = fs(16)
    J = J0(16)
    J[0] = 1.0
    maxwell_step(f, J, 0.1, g)
    np.testing.assert_allclose(npy(f.E1), -0.1, atol=1e-15)
    g = grid_of(2 * math.pi, 64)  # single-mode Faraday
    k, dt = 3.0, 0.05
    f = fs(64, E2=np.sin(k * g.centers))
    maxwell_step(f, J0(64), dt, g)
    keff = math.sin(k * g.eta) / g.eta
    np.testing.assert_allclose(npy(f.B3), -dt * keff * np.cos(k * g.centers), atol=1e-14)
    g = grid_of(2 * math.pi, 128)  # dispersion factor of both updates
    dt = 0.01
    for k in (1.0, 4.0, 9.0):
        keff = math.sin(k * g.eta) / g.eta
        f = fs(128, E2=np.sin(k * g.centers))
        maxwell_step(f, J0(128), dt, g)
        np.testing.assert_allclose(npy(f.B3) / (-dt * k * np.cos(k * g.centers)), keff / k,
                                   atol=1e-10)
        f = fs(128, B3=np.cos(k * g.centers))
        maxwell_step(f, J0(128), dt, g)
        np.testing.assert_allclose(npy(f.E2) / (dt * k * np.sin(k * g.centers)), keff / k,
                                   atol=1e-10)
    g = grid_of(2 * math.pi, 64)  # the B3 update sees the fresh E2
    k, dt = 2.0, 0.1
    f = fs(64, B3=np.cos(k * g.centers))
    maxwell_step(f, J0(64), dt, g)
    keff = math.sin(k * g.eta) / g.eta
    np.testing.assert_allclose(npy(f.B3), np.cos(k * g.centers) * (1 - (dt * keff) ** 2),
                               atol=1e-13)
    g = grid_of(2 * math.pi, 32)  # mean B3 conserved
    rng = np.random.default_rng(4)
    f = fs(32, E2=rng.normal(size=32), B3=rng.normal(size=32))
    m0 = npy(f.B3).mean()
    for _ in range(10):
        maxwell_step(f, J0(32), 0.05, g)
    assert npy(f.B3).mean() == pytest.approx(m0, abs=1e-10)


def test_vpl_field_step_cases(lib):
    from paper_2603_25832_b200.pic import vpl_field_step
    from paper_2603_25832_b200.state import FieldState

    f = FieldState.zeros(8, 2)
    f.E1.fill_(1.5)
    vpl_field_step(f, torch.zeros(2, 8, dtype=torch.float64, device="cuda"), 0.1)
    np.testing.assert_allclose(npy(f.E1), 1.5)
    f = FieldState.zeros(8, 2)
    J = torch.zeros(2, 8, dtype=torch.float64, device="cuda")
    J[0] = 2.0
    vpl_field_step(f, J, 0.05)
    np.testing.assert_allclose(npy(f.E1), -0.1, atol=1e-15)
    rng = np.random.default_rng(6)
    f = FieldState.zeros(32, 2)
    f.E1.copy_(torch.as_tensor(rng.normal(size=32)))
    J = np.zeros((2, 32))
    J[0] = rng.normal(size=32)
    J[0] -= J[0].mean()
    m0 = npy(f.E1).mean()
    vpl_field_step(f, torch.as_tensor(J, device="cuda"), 0.1)
    assert npy(f.E1).mean() == pytest.approx(m0, abs=1e-15)


def test_poisson_cases(lib):
    from paper_2603_25832_b200.pic import poisson_solve

    dev = "cuda"
    g = grid_of(2 * math.pi, 32)
    E1 = poisson_solve(torch.full((32,), 0.8, dtype=torch.float64, device=dev), 0.8, g)
    np.testing.assert_allclose(npy(E1), 0.0, atol=1e-14)
    g = grid_of(4 * math.pi, 100)
    a, k = 0.1, 0.5
    rho = torch.as_tensor(1.0 + a * np.cos(k * g.centers), device=dev)
    np.testing.assert_allclose(npy(poisson_solve(rho, 1.0, g)), (a / k) * np.sin(k * g.centers),
                               atol=1e-13)
    with pytest.raises(ValueError, match="non-neutral plasma"):
        poisson_solve(torch.full((16,), 1.1, dtype=torch.float64, device=dev), 1.0,
                      grid_of(2 * math.pi, 16))
    alpha, k, L = 0.1, 0.5, 4 * math.pi
    g = grid_of(L, 100)
    E1 = npy(poisson_solve(torch.as_tensor(1.0 + alpha * np.cos(k * g.centers), device=dev), 1.0, g))
    E_E = 0.5 * g.eta * np.sum(E1 ** 2)
    assert E_E == pytest.approx(alpha ** 2 * L / (4 * k ** 2), rel=1e-12)


# ----------------------------------------------------------------------------- Binning
def test_cell_index_cases(lib):
    from paper_2603_25832_b200.collision import build_cell_index
    from paper_2603_25832_b200.pic import Grid

    g = Grid(8, 0.5)
    ci = build_cell_index(ens(np.full(20, 0.1), np.zeros((20, 2)), np.full(20, 0.2)), g)
    assert ci.bins[0].size == 20 and all(ci.bins[c].size == 0 for c in range(1, 8))
    ci = build_cell_index(ens([0.5], np.zeros((1, 2)), [1.0]), g)  # floor convention
    assert ci.bins[1].size == 1
    rng = np.random.default_rng(0)
    g = Grid(13, 4 * math.pi / 13)
    x = rng.uniform(0, g.L, 500).astype(np.float32).astype(np.float64)
    ci = build_cell_index(ens(x, rng.normal(size=(500, 2)), np.full(500, g.L / 500)), g)
    assert np.array_equal(np.sort(np.concatenate(ci.bins)), np.arange(500))
    for c, b in enumerate(ci.bins):
        assert np.all(np.floor(x[b] / g.eta).astype(int) == c)
    for M in (1, 2):  # tiny grids: the stencil holds each neighbour cell once
        g = Grid(M, 4 * math.pi / M)
        ci = build_cell_index(ens(np.linspace(0, g.L, 10, endpoint=False), np.zeros((10, 2)),
                                  np.full(10, g.L / 10)), g)
        nb = ci.neighbors(0)
        assert nb.size == np.unique(nb).size


# --------------------------------------------------------------------------- Collision
def test_collision_constant_scores_vanish_and_hand_example(lib):
    from paper_2603_25832_b200.collision import build_cell_index, collision_force
    from paper_2603_25832_b200.pic import Grid

    rng = np.random.default_rng(1)
    g = Grid(10, 4 * math.pi / 10)
    p = ens(rng.uniform(0, g.L, 200), rng.normal(size=(200, 3)), np.full(200, g.L / 200))
    U = collision_force(p, np.tile([0.3, -1.2, 0.7], (200, 1)), build_cell_index(p, g), g, -3.0)
    np.testing.assert_allclose(npy(U), 0.0, atol=1e-6)  # s_i - s_j = 0 exactly in float32
    g = Grid(4, 1.0)
    p = ens([0.5, 0.5], [[1.0, 0.0, 0.0], [0.0, 0.0, 0.0]], [1.0, 1.0])
    U = npy(collision_force(p, np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 0.0]]),
                            build_cell_index(p, g), g, -3.0))
    np.testing.assert_allclose(U[0], [0.0, 1.0 / g.eta, 0.0], atol=1e-6)
    np.testing.assert_allclose(U[1], -U[0], atol=1e-6)


def test_collision_push_cases(lib):
    from paper_2603_25832_b200.collision import collision_push

    p = ens(np.zeros(3), np.ones((3, 2)), np.ones(3))
    collision_push(p, torch.ones(3, 2, device="cuda"), 0.0, 0.1)
    np.testing.assert_allclose(npy(p.v), 1.0)
    collision_push(p, torch.zeros(3, 2, device="cuda"), 0.7, 0.1)
    np.testing.assert_allclose(npy(p.v), 1.0)
    p = ens(np.zeros(1), np.zeros((1, 3)), np.ones(1))
    collision_push(p, torch.tensor([[1.0, 2.0, 0.0]], device="cuda"), 0.4, 0.02)
    np.testing.assert_allclose(npy(p.v), [[-0.008, -0.016, 0.0]], atol=1e-9)
