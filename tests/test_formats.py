"""Byte-level parity of the on-disk formats against files the reference's
own writers produced (tests/golden/make_formats.py -> tests/golden/formats.npz):
diagnostics.csv (17 significant digits, ref: diagnostics.py:42-53), the VMLS snapshot and
its JSON sidecar (diagnostics.py:72-90), the SBTM checkpoint (score.py:631-657) and
manifest.json (config.py:202-217; `code_version` is the implementation's own). CPU only:
the writers take host copies of the device state, so CPU tensors stand in for it here."""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def fx(golden):
    return golden("formats.npz")


def test_diagnostics_csv_bytes(fx, tmp_path):
    from paper_2603_25832_b200.diagnostics import read_diagnostics_csv, write_diagnostics_csv
    from paper_2603_25832_b200.state import DiagnosticsRecord

    recs = [DiagnosticsRecord(step=int(r[0]), t=float(r[1]), E_K=float(r[2]), E_E=float(r[3]),
                              E_B=float(r[4]), E_total=float(r[5]), H_dot=float(r[6]),
                              P=np.array(r[7:10]), E_l2=float(r[10])) for r in fx["records"]]
    path = tmp_path / "diagnostics.csv"
    write_diagnostics_csv(recs, str(path))
    assert path.read_bytes() == fx["csv"].tobytes()
    cols = read_diagnostics_csv(str(path))
    np.testing.assert_array_equal(cols["E_total"], fx["records"][:, 5])


def test_snapshot_and_sidecar_bytes(fx, tmp_path):
    from paper_2603_25832_b200.config import build_config
    from paper_2603_25832_b200.diagnostics import read_snapshot, write_snapshot
    from paper_2603_25832_b200.state import FieldState, ParticleEnsemble

    cpu = torch.device("cpu")
    p = ParticleEnsemble.from_arrays(fx["x"], fx["v"], fx["w"], device=cpu)
    f = FieldState.from_arrays(fx["E1"], fx["E2"], fx["B3"], device=cpu)
    cfg = build_config(overrides=dict(preset="weibel", n=4096, M=16, dt=0.05, t_final=0.25,
                                      seed=11))
    path = tmp_path / "snap.bin"
    write_snapshot(p, f, 3, 0.15, str(path), config=cfg)
    assert path.read_bytes() == fx["snap"].tobytes()
    assert (tmp_path / "snap.bin.json").read_bytes() == fx["snap_json"].tobytes()
    (x, v, w), (E1, E2, B3), meta = read_snapshot(str(path))
    np.testing.assert_array_equal(v, fx["v"])
    assert meta["step"] == 3


def test_sbtm_checkpoint_bytes(fx, tmp_path):
    from paper_2603_25832_b200.score import MlpScoreNet, load_checkpoint, save_checkpoint

    cpu = torch.device("cpu")
    net = MlpScoreNet(fx["W2"].shape[0], fx["W1"].shape[0], cpu)
    net.set_params([fx["W1"], fx["b1"], fx["W2"], fx["b2"]])
    path = tmp_path / "net.sbtm"
    save_checkpoint(net, str(path))
    assert path.read_bytes() == fx["ckpt"].tobytes()
    back = load_checkpoint(str(path), cpu)
    np.testing.assert_array_equal(back.params64.numpy(), net.params64.numpy())


def test_manifest_matches_reference(fx, tmp_path):
    from paper_2603_25832_b200.config import build_config, write_manifest

    cfg = build_config(overrides=dict(preset="weibel", n=4096, M=16, dt=0.05, t_final=0.25,
                                      seed=11))
    path = write_manifest(cfg, str(tmp_path), ["a warning"])
    got = json.loads(open(path, encoding="utf-8").read())
    ref = json.loads(fx["manifest"].tobytes().decode("utf-8"))
    got.pop("code_version")
    ref.pop("code_version")
    assert got == ref
