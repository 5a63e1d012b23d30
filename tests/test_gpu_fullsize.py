"""Parity at BASELINE config c4 (512^3, 496 x [1248 x 960]),
where the full CPU oracle would take minutes: compare bounded samples of
the full-size GPU outputs with the oracle (z-slices for K1, views for K2,
rows for K3) and check size-independent properties (linearity, slab ==
full volume, run-to-run determinism, exact zeros for missed rays)."""
import math
import os

import numpy as np
import pytest
import torch

from _helpers import FILTER_REL_RMSE, assert_close

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def c4(tg, O):
    vol = tg.VolumeSpec.centered([512] * 3, [0.5] * 3)
    det = tg.Detector2D.centered(1248, 960, 0.64, 0.64)
    geo = tg.make_cone(vol, det, 496, 220 * math.pi / 180, 750.0, 1200.0)
    O.set_threads(os.cpu_count() or 1)
    return geo


def _oracle_slab(O, geo, z0, nz):
    sp = geo.volume.spacing
    origin = list(geo.volume.origin)
    origin[2] = origin[2] + z0 * sp[2]
    ov = O.make_volume([512, 512, nz], sp, origin)
    od = O.det2_centered(1248, 960, 0.64, 0.64)
    return O.cone_from_matrices(ov, od, geo.angular_range, geo.sid, geo.sdd, geo.matrices)


def _bump(seed=0):
    u = torch.arange(1248, device=DEV, dtype=torch.float64)
    v = torch.arange(960, device=DEV, dtype=torch.float64)
    i = torch.arange(496, device=DEV, dtype=torch.float64)
    base = torch.clamp(1 - ((u[None] - 623.5) / 400) ** 2 - ((v[:, None] - 479.5) / 300) ** 2, min=0)
    return (base[None] * (1 + 0.1 * torch.sin(0.01 * i + seed))[:, None, None]).float().contiguous()


def test_c4_fdk_slices_vs_oracle(tg, O, c4):
    """K3 + K1 at full size; oracle back-projection of the identical filtered
    array on 64 z-slices: 16 groups of 4 spread from the top to the bottom of
    the volume (every K1 z-tile position and both tile halves are visited)"""
    raw = _bump()
    filt = tg.fdk_prefilter(raw, c4, True)
    vol = tg.back_project(tg.Sinogram.cone_beam(496, c4.detector, data=filt), c4).data
    f_np = filt.cpu().numpy()
    for z0 in np.linspace(0, 508, 16).astype(int):
        ref = O.cone_backproject(_oracle_slab(O, c4, int(z0), 4), f_np)
        assert_close(vol[z0:z0 + 4].cpu().numpy(), ref, what=f"c4 BP slices {z0}")


def test_c4_prefilter_rows_vs_oracle(tg, O, c4):
    raw = _bump()
    filt = tg.fdk_prefilter(raw, c4, True).cpu().numpy()
    views = [0, 62, 137, 186, 248, 310, 401, 495]
    s = raw[views].cpu().numpy()
    og = _oracle_slab(O, c4, 0, 1)
    w = O.apply_weights(s, O.cosine_weights_cone(og))
    pk = O.parker_weights_cone(O.make_cone(O.make_volume([512] * 3, [0.5] * 3),
                                           O.det2_centered(1248, 960, 0.64, 0.64), 496,
                                           220 * math.pi / 180, 750.0, 1200.0))[views]
    w = O.apply_weights(w, np.repeat(pk[:, None, :], 960, axis=1))
    ref = O.apply_filter(w, O.ramlak_weights(4096, 0.64))
    assert_close(filt[views], ref, rel_rmse=FILTER_REL_RMSE, what="c4 K3 rows")


def test_c4_forward_views_vs_oracle(tg, O, c4):
    """K2 at full size: eight views spread over the 220 deg scan against the
    oracle, exact zero pattern, through both K2 kernels (quad volume: the one
    the autotune keeps at c4; slab-staged), which give identical bits"""
    ph = tg.shepp_logan_3d(c4.volume, device=DEV).data
    views = [3, 65, 130, 190, 250, 301, 370, 490]
    og = O.cone_from_matrices(O.make_volume([512] * 3, [0.5] * 3),
                              O.det2_centered(1248, 960, 0.64, 0.64), c4.angular_range, c4.sid,
                              c4.sdd, c4.matrices[views])
    ref = O.cone_forward(og, ph.cpu().numpy())
    outs = {}
    for impl in (0, 1):
        tg.set_cone_knob(c4, "k2_impl", impl)
        outs[impl] = torch.stack([tg.cone_forward_views(c4, ph, v, 1)[0] for v in views]).cpu().numpy()
    tg.set_cone_knob(c4, "k2_impl", -1)
    out = outs[1]
    assert np.array_equal(outs[0], outs[1])
    assert_close(out, ref, what="c4 FP views")
    assert np.array_equal(out == 0.0, ref == 0.0)


def test_c4_linearity_determinism_slabs(tg, c4):
    p, q = _bump(0), _bump(1.3)
    bp = lambda s: tg.back_project(tg.Sinogram.cone_beam(496, c4.detector, data=s), c4).data
    a, b = bp(p), bp(q)
    c = bp(1.5 * p - 0.5 * q)
    assert float((c - (1.5 * a - 0.5 * b)).abs().max()) <= 1e-4 * float(c.abs().max())
    assert torch.equal(bp(p), a)  # run to run bitwise
    for z0, nz in [(0, 64), (192, 64), (448, 64)]:
        v0, nr = tg.cone_slab_rows(c4, z0, nz)
        slab = tg.cone_backproject_slab(c4, p[:, v0:v0 + nr].contiguous(), z0, nz, v0)
        assert torch.equal(slab, a[z0:z0 + nz])


def test_c4_calibrated_slices_vs_oracle(tg, O, c4):
    """the general (non-circular) K1 path at full c4 size: perturbed projection
    matrices (detector tilt / skew, out-of-plane terms; bench.py's
    k1_calibrated leg) through set_matrices, 12 z-slices in 3 groups against
    the oracle's back-projection with the same matrices"""
    m = np.asarray(c4.matrices).reshape(-1, 12).copy()
    rng = np.random.default_rng(11)
    m[:, [0, 1, 4, 5]] *= 1.0 + 2e-4 * rng.standard_normal((m.shape[0], 4))
    m[:, 2] += 2e-3 * rng.standard_normal(m.shape[0])
    m[:, 10] += 1e-5 * rng.standard_normal(m.shape[0])
    geo = tg.make_cone_from_matrices(c4.volume, c4.detector, c4.angular_range, c4.sid, c4.sdd, m)
    assert not geo.circular
    raw = _bump(0.7)
    vol = tg.back_project(tg.Sinogram.cone_beam(496, geo.detector, data=raw), geo).data
    r_np = raw.cpu().numpy()
    for z0 in (0, 254, 508):
        ref = O.cone_backproject(_oracle_slab(O, geo, z0, 4), r_np)
        assert_close(vol[z0:z0 + 4].cpu().numpy(), ref, what=f"c4 calibrated BP slices {z0}")
