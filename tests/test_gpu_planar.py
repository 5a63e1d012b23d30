"""GPU parity of the 2D operators K4-K7 (projector.hpp:171-260) and of the
phantom rasteriser against the CPU oracle / the reference's known answers."""
import math

import numpy as np
import pytest
import torch

from _helpers import assert_close, planar_pair, rand

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

CASES = {
    "parallel_c1": dict(shape=[256, 256], sp=[1.0, 1.0], nb=365, db=1.0, n=360, rng=math.pi),
    "fan_c2": dict(shape=[128, 128], sp=[2.0, 2.0], nb=256, db=3.2, n=90, rng=2 * math.pi, sid=750.0,
                   sdd=1200.0),
    "parallel_odd": dict(shape=[33, 17], sp=[1.3, 0.7], nb=29, db=0.9, n=7, rng=2 * math.pi),
    "fan_near": dict(shape=[5, 5], sp=[48.0, 48.0], nb=31, db=8.0, n=3, rng=math.pi, sid=64.0,
                     sdd=128.0),
}


def _fp(tg, geo, img):
    return tg.forward_project(tg.Image(geo.volume, torch.from_numpy(img).to(DEV)), geo).data.cpu().numpy()


def _bp(tg, geo, s):
    sino = tg.Sinogram.planar(geo.n_projections, geo.detector, data=torch.from_numpy(s).to(DEV))
    return tg.back_project(sino, geo).data.cpu().numpy()


@pytest.mark.parametrize("case", list(CASES))
def test_planar_forward_parity(tg, O, case):
    geo, og = planar_pair(tg, O, **CASES[case])
    img = rand(og.img_shape_yx, 11)
    out, ref = _fp(tg, geo, img), O.planar_forward(og, img)
    assert_close(out, ref, what=f"FP {case}")
    assert np.array_equal(out == 0.0, ref == 0.0)


@pytest.mark.parametrize("case", list(CASES))
def test_planar_backproject_parity(tg, O, case):
    geo, og = planar_pair(tg, O, **CASES[case])
    s = rand(og.sino_shape, 12, -1, 1)
    assert_close(_bp(tg, geo, s), O.planar_backproject(og, s), what=f"BP {case}")


def test_uniform_box(tg):
    """test_projector.cpp:34-45: axis-aligned rays through 15x15 ones = 15"""
    vol = tg.VolumeSpec.centered([15, 15], [1.0, 1.0])
    geo = tg.make_parallel(vol, tg.Detector1D.centered(15, 1.0), 1, math.pi)
    out = _fp(tg, geo, np.ones((15, 15), np.float32))
    assert np.allclose(out, 15.0, atol=1e-5)


def test_parallel_bp_counts_views(tg):
    """test_projector.cpp:134-142"""
    vol = tg.VolumeSpec.centered([9, 9], [1.0, 1.0])
    geo = tg.make_parallel(vol, tg.Detector1D.centered(15, 1.0), 12, 2 * math.pi)
    img = _bp(tg, geo, np.ones((12, 15), np.float32))
    assert img[4, 4] == 12.0
    assert np.allclose(img, 12.0, atol=1e-5)


def test_fan_bp_weights_and_behind_source(tg):
    """test_projector.cpp:144-166"""
    vol = tg.VolumeSpec.centered([5, 5], [16.0, 16.0])
    geo = tg.make_fan(vol, tg.Detector1D.centered(31, 8.0), 1, math.pi, 64.0, 128.0)
    img = _bp(tg, geo, np.ones((1, 31), np.float32))
    assert img[2, 0] == pytest.approx(4.0, abs=1e-5)
    assert img[2, 2] == pytest.approx(1.0, abs=1e-6)
    assert img[2, 4] == pytest.approx(4.0 / 9.0, abs=1e-6)
    assert img[3, 2] == pytest.approx(1.0, abs=1e-6)
    vol = tg.VolumeSpec.centered([5, 5], [48.0, 48.0])
    geo = tg.make_fan(vol, tg.Detector1D.centered(31, 8.0), 1, math.pi, 64.0, 128.0)
    img = _bp(tg, geo, np.ones((1, 31), np.float32))
    assert img[2, 0] == 0.0
    assert img[2, 1] == pytest.approx(16.0, abs=1e-4)


def test_disk_chords_and_mass(tg):
    """test_projector.cpp:47-70"""
    vol = tg.VolumeSpec.centered([256, 256], [1.0, 1.0])
    R = 80.0
    disk = tg.disk_phantom(vol, R, 1.0, device=DEV)
    geo = tg.make_parallel(vol, tg.Detector1D.centered(255, 1.0), 4, math.pi)
    s = tg.forward_project(disk, geo).data.cpu().numpy()
    for i in range(4):
        checked = good = 0
        for j in range(255):
            sj = geo.detector.origin + j * geo.detector.spacing
            if abs(sj) > 0.9 * R:
                continue
            checked += 1
            good += abs(s[i, j] - 2 * math.sqrt(R * R - sj * sj)) <= 1.0
        assert good >= checked * 9 // 10
        assert s[i].sum() * geo.detector.spacing == pytest.approx(math.pi * R * R, rel=0.01)


def test_phantoms_bit_exact(tg, O):
    v3 = tg.VolumeSpec.centered([67, 45, 33], [0.5, 0.7, 0.9])
    ov3 = O.make_volume(v3.shape, v3.spacing)
    assert np.array_equal(tg.shepp_logan_3d(v3, device=DEV).data.cpu().numpy(), O.shepp_logan_3d(ov3))
    v2 = tg.VolumeSpec.centered([129, 77], [0.4, 1.1])
    ov2 = O.make_volume(v2.shape, v2.spacing)
    assert np.array_equal(tg.shepp_logan_2d(v2, device=DEV).data.cpu().numpy(), O.shepp_logan_2d(ov2))
