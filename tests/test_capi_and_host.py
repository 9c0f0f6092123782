"""CPU tests: the C-ABI library builds, loads and exports every symbol the header declares;
host-side logic (config layering/validation, seeded sampling) matches the reference."""

import math
import os
import re
import shutil

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scorepic_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|int64_t|long long)\s+(spic_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for must in ("spic_bin", "spic_landau", "spic_collision_epilogue", "spic_blob",
                 "spic_mlp_forward", "spic_ism_partials_ex", "spic_sbtm_finalize_ex",
                 "spic_push", "spic_deposit_field", "spic_poisson", "spic_moments"):
        assert must in syms


def test_ctypes_table_matches_header():
    from paper_2603_25832_b200 import _lib

    assert sorted(_lib.SIGNATURES) == header_symbols()


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
def test_library_builds_loads_and_exports_all_symbols():
    import ctypes

    from paper_2603_25832_b200 import _lib, build

    path = build.build()
    lib = ctypes.CDLL(path)
    for name in header_symbols():
        assert hasattr(lib, name), name
    # argument-free / pure-host entry points can run without a GPU
    assert lib.spic_version() >= 1
    assert lib.spic_num_sms() == 148
    _lib.load()
    assert _lib.query("spic_mlp_num_params", 128, 3) == 128 * 4 + 128 + 3 * 128 + 3
    assert _lib.query("spic_bin_scratch_bytes", 1 << 20, 128, 32) > 0
    assert _lib.query("spic_landau_scratch_bytes", 1 << 20, 128, 3, 0) > 0


def test_sampling_reproduces_reference_initial_ensembles(golden):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.sampling import sample_arrays

    g = golden("run.npz")
    cfgs = {
        "sbtm": dict(preset="landau_damping", n=4096, M=16, dt=0.05, t_final=0.25, nu=0.1, K=3,
                     hidden=16, lr=1e-3, weight_decay=0.0, divergence="exact",
                     pretrain_budget=40, pretrain_batch=512, alpha=0.1, seed=3),
        "blob": dict(preset="two_stream", n=4096, M=16, dt=0.05, t_final=0.25, nu=0.05,
                     estimator="blob", bandwidth="silverman", alpha=0.01, seed=4),
        "vml": dict(preset="weibel", n=4096, M=16, dt=0.05, t_final=0.25, nu=0.0,
                    estimator="none", seed=5),
    }
    for tag, ov in cfgs.items():
        cfg = build_config(overrides=ov)
        x, v, w = sample_arrays(cfg, np.random.default_rng(cfg.seed))
        assert np.array_equal(x, g[f"{tag}_x0"]), tag
        assert np.array_equal(v, g[f"{tag}_v0"]), tag


def test_config_layering_and_errors():
    from paper_2603_25832_b200.config import build_config, parse_config_text

    cfg = build_config(file_values=parse_config_text("preset = two_stream\nn = 100 # c\nM=8"),
                       overrides=dict(nu=0.1, n=None))
    assert cfg.preset == "two_stream" and cfg.n == 100 and cfg.M == 8 and cfg.nu == 0.1
    assert cfg.L == pytest.approx(10 * math.pi) and cfg.gamma == -3.0
    with pytest.raises(ValueError, match="unknown config key"):
        parse_config_text("bogus = 1")
    with pytest.raises(ValueError, match="expected 'key = value'"):
        parse_config_text("n 100")
    with pytest.raises(ValueError, match="weibel requires VML"):
        build_config(overrides=dict(preset="weibel", mode="VPL"))
    with pytest.raises(ValueError, match="collisions require an estimator"):
        build_config(overrides=dict(nu=0.1, estimator="none"))
    with pytest.raises(ValueError, match="wavenumber k"):
        build_config(overrides=dict(k=0.3))
    with pytest.raises(ValueError, match="gamma must equal"):
        build_config(overrides=dict(gamma=-2.0))


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
def test_capi_rejects_invalid_arguments_before_any_launch():
    """The boundary's error behaviour (include/scorepic_b200.h status codes): invalid sizes,
    unsupported key ranges and short scratch buffers return SPIC_ERR_* before any device
    work, so these calls are safe without a GPU."""
    from paper_2603_25832_b200 import _lib

    L = _lib.load()
    ERR_ARG, ERR_SCRATCH, ERR_UNSUP = -1, -2, -3
    null = None
    # binning: dv, M, n out of range; M * S beyond the 15-bit key; scratch too small
    assert L.spic_bin(null, null, 0, null, 10, 4, 0.1, 8, 1, null, null, null, null, null, null,
                      0, null) == ERR_ARG
    assert L.spic_bin(null, null, 0, null, 10, 3, 0.1, 0, 1, null, null, null, null, null, null,
                      0, null) == ERR_ARG
    assert L.spic_bin(null, null, 0, null, -1, 3, 0.1, 8, 1, null, null, null, null, null, null,
                      0, null) == ERR_ARG
    assert L.spic_bin(null, null, 0, null, 10, 3, 0.1, 1024, 64, null, null, null, null, null,
                      null, 0, null) == ERR_UNSUP
    need = L.spic_bin_scratch_bytes(1 << 20, 128, 32)
    assert L.spic_bin(null, null, 0, null, 1 << 20, 3, 0.1, 128, 32, null, null, null, null,
                      null, null, need - 1, null) == ERR_SCRATCH
    # pair kernel: cell range out of order, dv, scratch
    assert L.spic_landau_range(null, null, 100, 3, null, null, 8, 1, 0.1, -3.0, 0.1, 0, 5, 3,
                               null, null, 1 << 30, null) == ERR_ARG
    assert L.spic_landau_range(null, null, 100, 4, null, null, 8, 1, 0.1, -3.0, 0.1, 0, 0, 8,
                               null, null, 1 << 30, null) == ERR_ARG
    assert L.spic_landau(null, null, 1 << 20, 3, null, null, 128, 32, 0.1, -3.0, 0.1, 0, null,
                         null, 0, null) == ERR_SCRATCH
    # push: eta, M
    assert L.spic_push(null, null, 0, 10, 3, null, null, null, 8, 0.0, 0.05, null, null) == ERR_ARG
    assert L.spic_push(null, null, 0, 10, 3, null, null, null, 0, 0.1, 0.05, null, null) == ERR_ARG
    # decomposition messages: cell bounds outside [0, M], negative row counts
    import ctypes

    int4 = ctypes.c_int32 * 4
    bad, ok = int4(0, 9, 0, 0), int4(0, 2, 0, 0)
    assert L.spic_dist_pack(null, null, 0, 3, null, 0.1, null, null, null, 8,
                            ctypes.cast(bad, ctypes.c_void_p), ctypes.cast(ok, ctypes.c_void_p),
                            16, null, null) == ERR_ARG
    assert L.spic_dist_unpack(null, -1, 0, null, null, 0, 3, null, null, null) == ERR_ARG
