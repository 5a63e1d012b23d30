"""The CLI front end (paper_1904_13342_b200/cli.py) against the reference's
cli.hpp contract: exit codes 0 / 1 (usage) / 2 (data or processing error,
"error: <what>" on stderr), host-only subcommands on CPU; the device
subcommands end to end on the GPU with byte-identical outputs run to run
(acceptance.cpp:486-548) and equal to the in-memory API."""
import json
import os

import numpy as np
import pytest

from paper_1904_13342_b200 import cli
from paper_1904_13342_b200 import io as tio

GEO_FDK = {"type": "cone3d", "volume_shape": [64, 64, 64], "volume_spacing": [0.85] * 3,
           "detector_shape": [96, 96], "detector_spacing": [1.0, 1.0], "n_projections": 248,
           "angular_range_deg": 200.0, "sid": 750.0, "sdd": 1200.0}
GEO_PAR = {"type": "parallel2d", "volume_shape": [64, 64], "volume_spacing": [1.0, 1.0],
           "detector_shape": [93], "detector_spacing": [1.0], "n_projections": 30,
           "angular_range_deg": 180.0}


def _j(p, obj):
    p.write_text(json.dumps(obj))
    return str(p)


def test_usage_errors_exit_1(capsys):
    assert cli.run([]) == 1
    assert cli.run(["nope"]) == 1
    assert cli.run(["project", "--geometry", "g.json"]) == 1  # missing required options
    assert cli.run(["reconstruct", "fbp", "--filter", "shepp"]) == 1


def test_data_errors_exit_2(tmp_path, capsys):
    assert cli.run(["trajectory", "--geometry", str(tmp_path / "none.json"),
                    "--out", str(tmp_path / "t.json")]) == 2
    assert "error: cannot open" in capsys.readouterr().err
    assert cli.run(["reconstruct", "fdk", "--geometry", "g.json"]) == 2
    assert "need --config or all of --geometry, --sino, --out" in capsys.readouterr().err
    g = _j(tmp_path / "par.json", GEO_PAR)
    assert cli.run(["reconstruct", "fdk", "--geometry", g, "--sino", "s.json", "--out", "o.json"]) == 2
    assert "fdk expects a cone3d geometry" in capsys.readouterr().err
    assert cli.run(["phantom", "--out", str(tmp_path / "p.json")]) == 2
    assert "pass exactly one of --geometry or --size" in capsys.readouterr().err


def test_trajectory_on_host(tmp_path):
    g = _j(tmp_path / "cone.json", GEO_FDK)
    assert cli.run(["trajectory", "--geometry", g, "--out", str(tmp_path / "t.json")]) == 0
    t = json.load(open(tmp_path / "t.json"))
    assert t["type"] == "cone3d" and len(t["projection_matrices"]) == 248


def test_profile_and_pgm_on_host(tmp_path, tg):
    vol = tg.VolumeSpec.centered([4, 3, 5], [1.0, 1.0, 1.0])
    data = np.arange(60, dtype=np.float32).reshape(5, 3, 4)
    tio.write_image(str(tmp_path / "v.json"), tg.Image(vol, data))
    assert cli.run(["profile", "--image", str(tmp_path / "v.json"), "--out",
                    str(tmp_path / "p.csv")]) == 0
    h, rows = tio.read_csv(str(tmp_path / "p.csv"))
    assert h == ["position_mm", "value"] and [r[1] for r in rows] == list(data[2, 1].astype(float))
    assert cli.run(["export-pgm", "--image", str(tmp_path / "v.json"), "--out",
                    str(tmp_path / "v.pgm")]) == 0
    b = (tmp_path / "v.pgm").read_bytes()
    assert b.startswith(b"P5\n4 3\n255\n") and len(b) == len(b"P5\n4 3\n255\n") + 12


@pytest.mark.gpu
def test_shell_pipeline_fdk_byte_identical(tmp_path, tg):
    g = _j(tmp_path / "g.json", GEO_FDK)
    outs = []
    for r in range(2):
        d = tmp_path / f"run{r}"
        d.mkdir()
        assert cli.run(["phantom", "--geometry", g, "--out", str(d / "ph.json")]) == 0
        assert cli.run(["project", "--geometry", g, "--image", str(d / "ph.json"),
                        "--out", str(d / "sino.json"), "--noise-rel", "0.01"]) == 0
        assert cli.run(["reconstruct", "fdk", "--geometry", g, "--sino", str(d / "sino.json"),
                        "--out", str(d / "rec.json")]) == 0
        assert cli.run(["export-pgm", "--image", str(d / "rec.json"), "--lo", "0",
                        "--hi", "0.05", "--out", str(d / "rec.pgm")]) == 0
        outs.append({n: (d / n).read_bytes() for n in
                     ("ph.raw", "sino.raw", "rec.raw", "rec.pgm", "rec.json")})
    assert outs[0] == outs[1]
    # the same as the in-memory API
    geo = tio.load_geometry(g)
    ph = tg.shepp_logan_3d(geo.volume, device="cuda:0")
    sino = tg.add_gaussian_noise(tg.forward_project(ph, geo), 0.01, 1337)
    rec = tg.fdk_reconstruct(sino, geo)
    assert rec.data.cpu().numpy().tobytes() == outs[0]["rec.raw"]


@pytest.mark.gpu
def test_config_runs(tmp_path, tg):
    _j(tmp_path / "geo.json", GEO_FDK)
    cfg = _j(tmp_path / "fdk.json", {
        "geometry": "geo.json", "phantom": "shepp-logan", "noise_relative_std": 0.0, "seed": 1337,
        "outputs": {"image": "out/rec.json", "phantom_image": "out/ph.json",
                    "sinogram": "out/sino.json", "profile_csv": "out/prof.csv",
                    "phantom_profile_csv": "out/php.csv"}})
    assert cli.run(["reconstruct", "fdk", "--config", cfg]) == 0
    rec = tio.read_image(str(tmp_path / "out" / "rec.json"))
    ph = tio.read_image(str(tmp_path / "out" / "ph.json"))
    # acceptance.cpp:244-265: the shipped short-scan FDK config reconstructs the
    # phantom with RMSE < 0.08 (reference measured 0.00601)
    rmse = float(np.sqrt(np.mean((rec.data.astype(np.float64) - ph.data) ** 2)))
    assert rmse < 0.08
    _j(tmp_path / "par.json", GEO_PAR)
    tv = _j(tmp_path / "tv.json", {
        "geometry": "par.json", "phantom": "shepp-logan", "noise_relative_std": 0.02,
        "learning_rate": 1.5e-4, "iterations": 40, "tv_lambda": 3.0, "seed": 1337,
        "outputs": {"image": "tv/rec.json", "fbp_image": "tv/fbp.json", "loss_csv": "tv/loss.csv",
                    "sinogram": "tv/sino.json", "profile_csv": "tv/p.csv"}})
    assert cli.run(["reconstruct", "iterative", "--config", tv]) == 0
    h, rows = tio.read_csv(str(tmp_path / "tv" / "loss.csv"))
    assert h == ["iteration", "loss"] and len(rows) == 41 and rows[-1][1] < rows[0][1]


GEO_LEARN = {"type": "parallel2d", "volume_shape": [45, 45], "volume_spacing": [1.0, 1.0],
             "detector_shape": [64], "detector_spacing": [1.0], "n_projections": 60,
             "angular_range_deg": 180.0}


def test_learn_filter_rejects_non_parallel(tmp_path, capsys):
    _j(tmp_path / "cone.json", GEO_FDK)
    cfg = _j(tmp_path / "lf.json", {"geometry": "cone.json", "iterations": 1})
    assert cli.run(["learn-filter", "--config", cfg]) == 2
    assert "learn-filter expects a parallel2d geometry" in capsys.readouterr().err


@pytest.mark.gpu
def test_learn_filter_config(tmp_path, tg):
    """configs/learn_filter.json (noise 0.3, lr 1.5e-5, window 64), 60 of its
    5000 steps: every output role written, the loss and the distance to
    Ram-Lak fall, and the run is byte-identical when repeated"""
    _j(tmp_path / "lfg.json", GEO_LEARN)
    outs = {"filter_csv": "o/learned.csv", "ramp_csv": "o/ramp.csv", "ramlak_csv": "o/ramlak.csv",
            "loss_csv": "o/loss.csv", "distance_csv": "o/dist.csv", "image": "o/rec.json",
            "profile_csv": "o/prof.csv"}
    cfg = _j(tmp_path / "lf.json", {
        "geometry": "lfg.json", "phantom": "shepp-logan", "noise_relative_std": 0.3,
        "learning_rate": 1.5e-5, "iterations": 60, "seed": 1337, "filter_window": 64,
        "outputs": outs})
    assert cli.run(["learn-filter", "--config", cfg]) == 0
    h, rows = tio.read_csv(str(tmp_path / "o" / "loss.csv"))
    assert h == ["iteration", "loss"] and len(rows) == 61 and rows[-1][1] < rows[0][1]
    h, rows = tio.read_csv(str(tmp_path / "o" / "dist.csv"))
    assert h == ["iteration", "distance"] and rows[0][1] == 1.0 and rows[-1][1] < 1.0
    assert len(tio.read_filter_csv(str(tmp_path / "o" / "learned.csv"))) == 64
    first = {k: (tmp_path / v).read_bytes() for k, v in outs.items() if not v.endswith(".json")}
    assert cli.run(["learn-filter", "--config", cfg]) == 0
    assert first == {k: (tmp_path / v).read_bytes() for k, v in outs.items()
                     if not v.endswith(".json")}
