"""scorepic_b200 — B200-native (sm_100a) per-timestep hot path of the scorepic collisional
particle-in-cell solver (Vlasov–Maxwell/Poisson–Landau with score-based collisions).

The reference's Python API names are kept (Grid, ParticleEnsemble, FieldState,
build_cell_index, collision_force, SbtmEstimator, BlobEstimator, run, ...); the compute is
the C-ABI library `lib/libscorepic_b200.so` (declared in include/scorepic_b200.h), built
with `python -m paper_2603_25832_b200.build`. There is no CPU fallback.
"""

__version__ = "0.1.0"

from .config import DeviceOptions, SimConfig, build_config, parse_config_text, preset_defaults  # noqa: F401,E402
