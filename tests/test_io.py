"""CPU: the file formats around the path (paper_1904_13342_b200/io.py),
restating the reference's own io tests (tests/test_io.cpp) — sidecar +
f32le payload, validation messages, geometry files incl. calibrated
projection matrices, trajectories, experiment configs, CSV round trips,
slices, profiles, PGM windows."""
import json
import math
import os

import numpy as np
import pytest

from paper_1904_13342_b200 import io as tio


def test_raw_roundtrip(tmp_path, tg):
    arr = tio.RawArray([3, 2], [0.5, 2.0], [-1.0, 3.0], np.arange(6, dtype=np.float32) * 0.25)
    tio.write_raw(str(tmp_path / "a.json"), arr)
    back = tio.read_raw(str(tmp_path / "a.json"))
    assert back.shape == arr.shape and back.spacing == arr.spacing and back.origin == arr.origin
    assert np.array_equal(back.data, arr.data)
    j = json.load(open(tmp_path / "a.json"))
    assert j["dtype"] == "f32le" and j["data"] == "a.raw"


def test_raw_payload_is_little_endian_f32(tmp_path, tg):
    # test_io.cpp:53-73: {1.5, -2.0} -> 00 00 C0 3F 00 00 00 C0
    tio.write_raw(str(tmp_path / "e.json"), tio.RawArray([2], [1.0], [0.0], np.array([1.5, -2.0])))
    assert (tmp_path / "e.raw").read_bytes() == bytes([0, 0, 0xC0, 0x3F, 0, 0, 0, 0xC0])


def test_raw_validation_messages(tmp_path, tg):
    with pytest.raises(tg.Error, match="cannot open"):
        tio.read_raw(str(tmp_path / "nope.json"))
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(tg.Error, match="malformed JSON"):
        tio.read_raw(str(tmp_path / "bad.json"))
    (tmp_path / "keys.json").write_text('{"shape": [2]}')
    with pytest.raises(tg.Error, match="misses required keys"):
        tio.read_raw(str(tmp_path / "keys.json"))
    (tmp_path / "dt.json").write_text('{"shape": [2], "dtype": "f64le", "data": "dt.raw"}')
    with pytest.raises(tg.Error, match="unsupported dtype"):
        tio.read_raw(str(tmp_path / "dt.json"))
    tio.write_raw(str(tmp_path / "trunc.json"), tio.RawArray([4], [1.0], [0.0], np.arange(4.0)))
    os.truncate(tmp_path / "trunc.raw", 12)
    with pytest.raises(tg.Error, match="payload size does not match"):
        tio.read_raw(str(tmp_path / "trunc.json"))


def test_image_roundtrip_keeps_grid(tmp_path, tg):
    vol = tg.VolumeSpec([4, 3, 2], [0.5, 1.0, 2.0], [-1.0, 0.0, 5.0])
    data = np.random.default_rng(1).uniform(-1, 1, (2, 3, 4)).astype(np.float32)
    tio.write_image(str(tmp_path / "img.json"), tg.Image(vol, data))
    back = tio.read_image(str(tmp_path / "img.json"))
    assert back.spec.shape == vol.shape and back.spec.spacing == vol.spacing
    assert back.spec.origin == vol.origin and np.array_equal(back.data, data)
    tio.write_raw(str(tmp_path / "vec.json"), tio.RawArray([5], [1.0], [0.0], np.zeros(5)))
    with pytest.raises(tg.Error, match="expected a 2D or 3D image"):
        tio.read_image(str(tmp_path / "vec.json"))


def test_sinograms_bind_to_geometry(tmp_path, tg):
    vol = tg.VolumeSpec.centered([16, 16], [1.0, 1.0])
    geo = tg.make_parallel(vol, tg.Detector1D.centered(23, 1.0), 6, math.pi)
    data = np.random.default_rng(2).uniform(0, 1, (6, 23)).astype(np.float32)
    tio.write_sinogram(str(tmp_path / "s.json"), tg.Sinogram.planar(6, geo.detector, data=data))
    back = tio.read_sinogram(str(tmp_path / "s.json"), geo)
    assert back.n_projections == 6 and np.array_equal(back.data, data)
    other = tg.make_parallel(vol, tg.Detector1D.centered(25, 1.0), 6, math.pi)
    with pytest.raises(tg.Error, match="does not match the geometry"):
        tio.read_sinogram(str(tmp_path / "s.json"), other)


def test_cone_sinograms_carry_both_pitches(tmp_path, tg):
    det = tg.Detector2D.centered(12, 10, 1.5, 2.0)
    geo = tg.make_cone(tg.VolumeSpec.centered([8, 8, 8], [1.0] * 3), det, 5, 2 * math.pi, 50., 100.)
    data = np.random.default_rng(3).uniform(0, 1, (5, 10, 12)).astype(np.float32)
    tio.write_sinogram(str(tmp_path / "c.json"), tg.Sinogram.cone_beam(5, det, data=data))
    arr = tio.read_raw(str(tmp_path / "c.json"))
    assert arr.shape == [12, 10, 5] and arr.spacing[0] == 1.5 and arr.spacing[1] == 2.0
    back = tio.read_sinogram(str(tmp_path / "c.json"), geo)
    assert back.is_cone() and np.array_equal(back.data, data)


def _write(p, obj):
    p.write_text(obj if isinstance(obj, str) else json.dumps(obj))
    return str(p)


def test_geometry_files_all_three_types(tmp_path, tg):
    par = tio.load_geometry(_write(tmp_path / "par.json", {
        "type": "parallel2d", "volume_shape": [16, 16], "volume_spacing": [1.0, 1.0],
        "detector_shape": [23], "detector_spacing": [1.0], "n_projections": 12,
        "angular_range_deg": 180.0}))
    assert isinstance(par, tg.ParallelGeometry) and par.n_projections == 12
    assert par.angular_range == pytest.approx(math.pi)
    fan = tio.load_geometry(_write(tmp_path / "fan.json", {
        "type": "fan2d", "volume_shape": [16, 16], "volume_spacing": [1.0, 1.0],
        "detector_shape": [23], "detector_spacing": [1.0], "n_projections": 12,
        "angular_range_deg": 360.0, "sid": 40.0, "sdd": 80.0}))
    assert isinstance(fan, tg.FanGeometry) and fan.sid == 40.0 and fan.sdd == 80.0
    cone = tio.load_geometry(_write(tmp_path / "cone.json", {
        "type": "cone3d", "volume_shape": [8, 8, 8], "volume_spacing": [1.0, 1.0, 1.0],
        "detector_shape": [12, 10], "detector_spacing": [1.5, 2.0], "n_projections": 6,
        "angular_range_deg": 360.0, "sid": 50.0, "sdd": 100.0}))
    assert isinstance(cone, tg.ConeGeometry)
    assert cone.detector.n_u == 12 and cone.detector.n_v == 10 and len(cone.matrices) == 6


def test_geometry_validation_messages(tmp_path, tg):
    base = {"volume_shape": [8, 8], "volume_spacing": [1.0, 1.0], "detector_shape": [11],
            "detector_spacing": [1.0], "n_projections": 4, "angular_range_deg": 180.0}
    with pytest.raises(tg.Error, match="geometry misses key"):
        tio.load_geometry(_write(tmp_path / "nokey.json", {"type": "parallel2d"}))
    with pytest.raises(tg.Error, match="unknown geometry type"):
        tio.load_geometry(_write(tmp_path / "unk.json", dict(base, type="spiral")))
    with pytest.raises(tg.Error, match="fan2d needs sid and sdd"):
        tio.load_geometry(_write(tmp_path / "fansdd.json", dict(base, type="fan2d",
                                                                 angular_range_deg=360.0)))
    with pytest.raises(tg.Error, match="parallel2d expects a 2D volume"):
        tio.load_geometry(_write(tmp_path / "rank.json", dict(
            base, type="parallel2d", volume_shape=[8, 8, 8], volume_spacing=[1.0] * 3)))


def test_cone_explicit_projection_matrices(tmp_path, tg):
    vol = tg.VolumeSpec.centered([8, 8, 8], [1.0] * 3)
    circ = tg.make_cone(vol, tg.Detector2D.centered(12, 10, 1.0, 1.0), 4, math.pi, 50.0, 100.0)
    j = {"type": "cone3d", "volume_shape": [8, 8, 8], "volume_spacing": [1.0] * 3,
         "detector_shape": [12, 10], "detector_spacing": [1.0, 1.0], "n_projections": 4,
         "angular_range_deg": 180.0, "sid": 50.0, "sdd": 100.0,
         "projection_matrices": [list(map(float, m)) for m in np.asarray(circ.matrices).reshape(-1, 12)]}
    geo = tio.load_geometry(_write(tmp_path / "mat.json", j))
    assert np.array_equal(np.asarray(geo.matrices), np.asarray(circ.matrices))
    j["projection_matrices"] = [[0.0] * 12]
    with pytest.raises(tg.Error, match="must equal n_projections"):
        tio.load_geometry(_write(tmp_path / "badcount.json", j))
    # a calibrated (scaled, perturbed) matrix set is normalised on load (set_matrices)
    m = np.asarray(circ.matrices).reshape(-1, 12) * 3.0
    m[:, 2] += 1e-3
    j["projection_matrices"] = m.tolist()
    cal = tio.load_geometry(_write(tmp_path / "cal.json", j))
    ref = tg.make_cone_from_matrices(vol, tg.Detector2D.centered(12, 10, 1.0, 1.0), math.pi,
                                     50.0, 100.0, m)
    assert np.array_equal(np.asarray(cal.matrices), np.asarray(ref.matrices))
    assert not cal.circular


def test_trajectory_files(tmp_path, tg):
    par = tg.make_parallel(tg.VolumeSpec.centered([8, 8], [1.0, 1.0]),
                           tg.Detector1D.centered(11, 1.0), 5, math.pi)
    tio.write_trajectory(str(tmp_path / "par.json"), par)
    jp = json.load(open(tmp_path / "par.json"))
    assert jp["type"] == "parallel2d" and len(jp["angles_rad"]) == 5 and len(jp["rays"]) == 5
    assert jp["angles_rad"][0] == par.angles[0]
    cone = tg.make_cone(tg.VolumeSpec.centered([8, 8, 8], [1.0] * 3),
                        tg.Detector2D.centered(12, 10, 1.0, 1.0), 3, math.pi, 50.0, 100.0)
    tio.write_trajectory(str(tmp_path / "cone.json"), cone)
    jc = json.load(open(tmp_path / "cone.json"))
    assert jc["type"] == "cone3d" and len(jc["projection_matrices"]) == 3
    assert len(jc["projection_matrices"][0]) == 12


def test_experiment_config_resolves_paths(tmp_path, tg):
    (tmp_path / "sub").mkdir()
    _write(tmp_path / "sub" / "geo.json", {
        "type": "parallel2d", "volume_shape": [16, 16], "volume_spacing": [1.0, 1.0],
        "detector_shape": [23], "detector_spacing": [1.0], "n_projections": 12,
        "angular_range_deg": 180.0})
    p = _write(tmp_path / "sub" / "exp.json", {
        "geometry": "geo.json", "phantom": "disk", "noise_relative_std": 0.02,
        "learning_rate": 5e-4, "iterations": 25, "tv_lambda": 1.5, "seed": 99,
        "filter_window": 64, "outputs": {"image": "out/rec.json", "loss": "out/loss.csv"}})
    e = tio.load_experiment_config(p)
    assert isinstance(e.geometry, tg.ParallelGeometry)
    assert (e.cfg.phantom, e.cfg.noise_relative_std, e.cfg.learning_rate, e.cfg.iterations,
            e.cfg.tv_lambda, e.cfg.seed, e.cfg.filter_window) == ("disk", 0.02, 5e-4, 25, 1.5, 99, 64)
    assert e.outputs["image"] == os.path.join(str(tmp_path / "sub"), "out/rec.json")


def test_reference_shipped_configs_parse(tg):
    ref = "/root/reference/proj/configs"
    if not os.path.isdir(ref):
        pytest.skip("reference configs not mounted")
    for name in ("fdk_short_scan.json", "iterative_tv.json", "learn_filter.json"):
        e = tio.load_experiment_config(os.path.join(ref, name))
        assert e.cfg.iterations >= 0


def test_csv_roundtrips_doubles_exactly(tmp_path, tg):
    tio.write_csv(str(tmp_path / "x.csv"), ["a", "b"], [[math.pi, 1.0 / 3.0], [2.0, 1e-300]])
    h, rows = tio.read_csv(str(tmp_path / "x.csv"))
    assert h == ["a", "b"] and rows[0] == [math.pi, 1.0 / 3.0] and rows[1][1] == 1e-300
    tio.write_filter_csv(str(tmp_path / "w.csv"), [0.5, -0.25, 1e-20])
    assert tio.read_filter_csv(str(tmp_path / "w.csv")) == [0.5, -0.25, 1e-20]
    (tmp_path / "bad.csv").write_text("a,b,c\n1,2,3\n")
    with pytest.raises(tg.Error, match=r"filter CSV rows must be \(bin_index, weight\)"):
        tio.read_filter_csv(str(tmp_path / "bad.csv"))


def test_slices_profiles_pgm(tmp_path, tg):
    vol = tg.VolumeSpec([3, 4, 5], [1.0, 2.0, 3.0], [0.0, 10.0, 20.0])
    z, y, x = np.meshgrid(np.arange(5), np.arange(4), np.arange(3), indexing="ij")
    img = tg.Image(vol, (x + 10.0 * y + 100.0 * z).astype(np.float32))
    ax = tio.extract_slice(img, 2, 3)
    assert ax.spec.shape == [3, 4] and ax.spec.spacing == [1.0, 2.0]
    assert ax.data[1, 2] == 2.0 + 10.0 + 300.0
    sag = tio.extract_slice(img, 0, 2)
    assert sag.spec.shape == [4, 5] and sag.spec.spacing == [2.0, 3.0]
    assert sag.spec.origin == [10.0, 20.0] and sag.data[4, 1] == 2.0 + 10.0 + 400.0
    with pytest.raises(tg.Error, match="axis out of range"):
        tio.extract_slice(img, 3, 0)
    with pytest.raises(tg.Error, match="slice index out of range"):
        tio.extract_slice(img, 2, 5)
    im2 = tg.Image(tg.VolumeSpec.centered([3, 2], [2.0, 1.0]),
                   np.array([[1, 2, 3], [10, 11, 12]], np.float32))
    px = tio.line_profile(im2, 0, 1)
    assert px[0][0] == -2.0 and px[2] == (2.0, 12.0)
    with pytest.raises(tg.Error, match="profile index out of range"):
        tio.line_profile(im2, 0, 2)
    tio.write_profile_csv(str(tmp_path / "p.csv"), [(-1.0, 2.0), (0.0, 3.5)])
    h, rows = tio.read_csv(str(tmp_path / "p.csv"))
    assert h == ["position_mm", "value"] and rows[1] == [0.0, 3.5]
    # PGM window: floor((v - lo) * 255 / (hi - lo)), clamped, rows top-down in -y
    pg = tg.Image(tg.VolumeSpec.centered([2, 2], [1.0, 1.0]),
                  np.array([[0.0, 0.5], [1.0, 3.0]], np.float32))
    tio.export_pgm(str(tmp_path / "x.pgm"), pg, 0.0, 2.0)
    b = (tmp_path / "x.pgm").read_bytes()
    hdr = b"P5\n2 2\n255\n"
    assert b[:len(hdr)] == hdr and list(b[len(hdr):]) == [127, 255, 0, 63]
    with pytest.raises(tg.Error, match="window must satisfy lo < hi"):
        tio.export_pgm(str(tmp_path / "y.pgm"), pg, 1.0, 1.0)
