"""GPU edge cases of the cone path against the oracle: more views than one
constant-bank chunk (K1 chunking), degenerate detectors (one column / one
row: the TMA re-pitch path), a one-slice volume, a single view, and an
accumulate pass on top of existing data."""
import math

import numpy as np
import pytest
import torch

from _helpers import assert_close, cone_pair, rand

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _bp(tg, geo, sino_np, **kw):
    s = tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=torch.from_numpy(sino_np).to(DEV))
    return tg.back_project(s, geo, **kw).data.cpu().numpy()


def _fp(tg, geo, vol_np):
    return tg.forward_project(tg.Image(geo.volume, torch.from_numpy(vol_np).to(DEV)), geo).data.cpu().numpy()


EDGES = {
    # 700 views > one 640-view constant-bank chunk of K1
    "many_views": dict(vshape=[24, 20, 18], vsp=[1.0] * 3, nu=32, nv=28, du=1.2, dv=1.2, n=700,
                       rng=2 * math.pi, sid=150.0, sdd=300.0),
    "one_column": dict(vshape=[16, 16, 12], vsp=[1.0] * 3, nu=1, nv=40, du=2.0, dv=1.0, n=12,
                       rng=2 * math.pi, sid=80.0, sdd=160.0),
    "one_row": dict(vshape=[16, 16, 12], vsp=[1.0] * 3, nu=41, nv=1, du=1.0, dv=3.0, n=12,
                    rng=2 * math.pi, sid=80.0, sdd=160.0),
    "one_slice": dict(vshape=[40, 36, 1], vsp=[1.0] * 3, nu=50, nv=9, du=1.0, dv=1.0, n=20,
                      rng=2 * math.pi, sid=100.0, sdd=200.0),
    "one_view": dict(vshape=[20, 20, 20], vsp=[1.0] * 3, nu=30, nv=30, du=1.0, dv=1.0, n=1,
                     rng=math.pi, sid=100.0, sdd=200.0),
}


@pytest.mark.parametrize("case", list(EDGES))
def test_edge_backproject(tg, O, case):
    geo, og = cone_pair(tg, O, **EDGES[case])
    s = rand(og.sino_shape, 3, -1.0, 1.0)
    assert_close(_bp(tg, geo, s), O.cone_backproject(og, s), what=f"BP {case}")


@pytest.mark.parametrize("case", list(EDGES))
def test_edge_forward(tg, O, case):
    geo, og = cone_pair(tg, O, **EDGES[case])
    v = rand(og.vol_shape_zyx, 4)
    out, ref = _fp(tg, geo, v), O.cone_forward(og, v)
    assert_close(out, ref, what=f"FP {case}")
    assert np.array_equal(out == 0.0, ref == 0.0)


def test_accumulate_adds_to_existing(tg, O):
    geo, og = cone_pair(tg, O, **EDGES["many_views"])
    s = rand(og.sino_shape, 5, -1.0, 1.0)
    base = torch.from_numpy(rand(og.vol_shape_zyx, 6)).to(DEV)
    out = base.clone()
    sino = torch.from_numpy(s).to(DEV)
    from paper_1904_13342_b200 import _native as N
    N.check(N.lib().tg_cone_backproject(geo._plan(0), sino.data_ptr(), out.data_ptr(), 0.5, 1,
                                        torch.cuda.current_stream().cuda_stream))
    want = base.cpu().numpy().astype(np.float64) + 0.5 * O.cone_backproject(og, s).astype(np.float64)
    assert_close(out.cpu().numpy(), want, what="accumulate")


def test_k2_single_layout_fallback_is_bitwise_equal(tg, O):
    """When the x- and y-fastest quad volumes do not both fit, K2 falls back
    to the x-fastest copy alone: same samples, same arithmetic, same bits."""
    import gc
    vol = tg.VolumeSpec.centered([96, 88, 80], [1.0] * 3)
    det = tg.Detector2D.centered(120, 100, 1.2, 1.2)
    ph = tg.shepp_logan_3d(vol, device=DEV)
    geo_a = tg.make_cone(vol, det, 40, 2 * math.pi, 300.0, 600.0)
    tg.set_cone_knob(geo_a, "k2_impl", 0)  # the quad-volume K2
    want = tg.forward_project(ph, geo_a).data.clone()
    one = 100 * 92 * 84 * 16  # one quad layout, bytes
    torch.cuda.synchronize()
    free, _ = torch.cuda.mem_get_info()
    total = torch.cuda.get_device_properties(0).total_memory
    # leave room for one layout (+ margins) but not two
    hog = torch.empty(int(free - total // 20 - int(1.5 * one) - (256 << 20)), dtype=torch.uint8,
                      device=DEV)
    try:
        geo_b = tg.make_cone(vol, det, 40, 2 * math.pi, 300.0, 600.0)  # fresh plan
        tg.set_cone_knob(geo_b, "k2_impl", 0)
        got = tg.forward_project(ph, geo_b).data.clone()
    finally:
        del hog
        gc.collect()
        torch.cuda.empty_cache()
    assert torch.equal(got, want)
