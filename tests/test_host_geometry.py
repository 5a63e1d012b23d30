"""The product's host-side precompute (csrc/host_geometry.cpp through the C
ABI; no GPU needed) must be BIT-EXACT with the reference:
geometry, weight maps, filter weights, phantom tables, and the reference's
error text."""
import math

import numpy as np
import pytest


def test_make_cone_bitwise(tg, O):
    for shape, sp, nu, nv, du, dv, n, rng, sid, sdd in [
        ([64, 64, 64], [0.85] * 3, 96, 96, 1.0, 1.0, 248, 200 * math.pi / 180, 750.0, 1200.0),
        ([512, 512, 512], [0.5] * 3, 1248, 960, 0.64, 0.64, 496, 220 * math.pi / 180, 750.0, 1200.0),
        ([7, 9, 11], [1.3, 0.7, 2.1], 13, 5, 0.3, 0.9, 7, 2 * math.pi, 33.0, 91.0),
    ]:
        vol = tg.VolumeSpec.centered(shape, sp)
        det = tg.Detector2D.centered(nu, nv, du, dv)
        g = tg.make_cone(vol, det, n, rng, sid, sdd)
        og = O.make_cone(O.make_volume(shape, sp), O.det2_centered(nu, nv, du, dv), n, rng, sid, sdd)
        for a, b in [("matrices", "mats"), ("sources", "sources"), ("inv_blocks", "invs"),
                     ("angles", "angles")]:
            assert np.array_equal(getattr(g, a), getattr(og, b)), a
        assert g.circular


def test_set_matrices_bitwise(tg, O):
    vol = tg.VolumeSpec.centered([8, 8, 8], [1.0] * 3)
    det = tg.Detector2D.centered(8, 8, 1.0, 1.0)
    mats = tg.projection_matrices_circular(5, math.pi, 60.0, 100.0, det)
    t = 0.3
    R = np.array([[math.cos(t), 0, math.sin(t), 0], [0, 1, 0, 0], [-math.sin(t), 0, math.cos(t), 0],
                  [0, 0, 0, 1]])
    mats = np.stack([(m.reshape(3, 4) @ R).reshape(12) * 7.0 for m in mats])
    g = tg.make_cone_from_matrices(vol, det, math.pi, 60.0, 100.0, mats)
    og = O.cone_from_matrices(O.make_volume([8] * 3, [1.0] * 3), O.det2_centered(8, 8, 1.0, 1.0),
                              math.pi, 60.0, 100.0, mats)
    for a, b in [("matrices", "mats"), ("sources", "sources"), ("inv_blocks", "invs"),
                 ("angles", "angles")]:
        assert np.array_equal(getattr(g, a), getattr(og, b)), a
    assert not g.circular


@pytest.mark.parametrize("sid,sdd", [(0.0, 0.0), (80.0, 160.0)])
def test_planar_rays_bitwise(tg, O, sid, sdd):
    vol = tg.VolumeSpec.centered([16, 16], [1.0, 1.0])
    det = tg.Detector1D.centered(24, 1.0)
    g = tg.make_fan(vol, det, 360, 2 * math.pi, sid, sdd) if sdd else tg.make_parallel(vol, det, 360, math.pi)
    og = O.make_planar(O.make_volume([16, 16], [1.0, 1.0]), O.det1_centered(24, 1.0), 360,
                       2 * math.pi if sdd else math.pi, sid, sdd)
    assert np.array_equal(g.rays, og.rays) and np.array_equal(g.angles, og.angles)


def test_filter_weights_bitwise(tg, O):
    for P, ds in [(2, 1.0), (32, 1.0), (256, 0.7), (1024, 1.0), (4096, 0.64), (8192, 0.4)]:
        assert np.array_equal(tg.ramlak_weights(P, ds), O.ramlak_weights(P, ds))
        assert np.array_equal(tg.ramp_weights(P, ds), O.ramp_weights(P, ds))
    for n in [1, 5, 64, 65, 100, 365, 1248, 2048]:
        assert tg.filter_window(n) == O.filter_window(n)
    for m in range(-9, 10):
        assert tg.ramlak_spatial(m, 0.7) == O.ramlak_spatial(m, 0.7)


def test_weight_maps_bitwise(tg, O):
    vol = tg.VolumeSpec.centered([8, 8, 8], [1.0] * 3)
    det = tg.Detector2D.centered(101, 7, 2.0, 2.0)
    g = tg.make_cone(vol, det, 40, 210 * math.pi / 180, 200.0, 400.0)
    og = O.make_cone(O.make_volume([8] * 3, [1.0] * 3), O.det2_centered(101, 7, 2.0, 2.0), 40,
                     210 * math.pi / 180, 200.0, 400.0)
    cw = tg.cosine_weights(g)
    assert cw.shape == [101, 7]
    assert np.array_equal(cw.data, O.cosine_weights_cone(og).reshape(-1))
    pw = tg.parker_weights(g)
    assert pw.shape == [101, 7, 40]
    assert np.array_equal(pw.row_profile, O.parker_weights_cone(og))
    # the materialised map repeats the profile on every detector row
    full = pw.full().reshape(40, 7, 101)
    assert np.array_equal(full[:, 3], O.parker_weights_cone(og))
    v2 = tg.VolumeSpec.centered([8, 8], [1.0, 1.0])
    fan = tg.make_fan(v2, tg.Detector1D.centered(101, 2.0), 181,
                      math.pi + 2 * math.atan(101.0 / 400.0), 200.0, 400.0)
    ofan = O.make_planar(O.make_volume([8, 8], [1.0, 1.0]), O.det1_centered(101, 2.0), 181,
                         math.pi + 2 * math.atan(101.0 / 400.0), 200.0, 400.0)
    assert np.array_equal(tg.cosine_weights(fan).data, O.cosine_weights_fan(ofan))
    assert np.array_equal(tg.parker_weights(fan).data, O.parker_weights_fan(ofan).reshape(-1))


def test_phantom_tables_bitwise(tg, O):
    spec = tg.VolumeSpec.centered([100, 80, 60], [0.5, 0.7, 0.9])
    ov = O.make_volume(spec.shape, spec.spacing)
    assert np.array_equal(tg.head_phantom_ellipsoids(spec), O.head_ellipsoids(O.fov_half_extent(ov)))


def test_slab_rows_cover_slab(tg, O):
    """the row band of a z-slab contains every tap its voxels use (FP64 check
    of the projected slab corners against the oracle geometry)"""
    from paper_1904_13342_b200 import distributed as D
    vol = tg.VolumeSpec.centered([64, 64, 64], [0.85] * 3)
    det = tg.Detector2D.centered(96, 96, 1.0, 1.0)
    g = tg.make_cone(vol, det, 31, 2 * math.pi, 750.0, 1200.0)
    shards = D.slab_shards(g, 2)
    assert [s.nz for s in shards] == [32, 32]
    for sh in shards:
        zs = np.arange(sh.z0, sh.z0 + sh.nz)
        xs = vol.origin[0] + np.arange(64) * vol.spacing[0]
        Z = vol.origin[2] + zs * vol.spacing[2]
        X, Y, ZZ = np.meshgrid(xs, xs, Z, indexing="ij")
        for P in g.matrices:
            hy = P[4] * X + P[5] * Y + P[6] * ZZ + P[7]
            hz = P[8] * X + P[9] * Y + P[10] * ZZ + P[11]
            v = hy / hz
            lo, hi = np.floor(v.min()), np.floor(v.max()) + 1
            assert lo >= sh.v0 or lo < 0
            assert hi <= sh.v0 + sh.n_rows - 1 or hi > 95


@pytest.mark.parametrize("call,msg", [
    (lambda tg: tg.make_cone(tg.VolumeSpec.centered([4, 4, 4], [1.0] * 3),
                             tg.Detector2D.centered(8, 8, 1, 1), 3, math.pi, 20.0, 10.0),
     "cone beam requires 0 < SID < SDD"),
    (lambda tg: tg.make_cone(tg.VolumeSpec.centered([4, 4], [1.0] * 2),
                             tg.Detector2D.centered(8, 8, 1, 1), 3, math.pi, 10.0, 20.0),
     "cone beam geometry expects a 3D volume"),
    (lambda tg: tg.make_fan(tg.VolumeSpec.centered([4, 4], [1.0] * 2),
                            tg.Detector1D.centered(8, 1.0), 3, math.pi, 80.0, 50.0),
     "fan beam requires 0 < SID < SDD"),
    (lambda tg: tg.view_angles(0, math.pi), "need at least one projection"),
    (lambda tg: tg.view_angles(4, 2 * math.pi + 0.1), "angular range must lie in (0, 2*pi]"),
    (lambda tg: tg.make_cone_from_matrices(tg.VolumeSpec.centered([8] * 3, [1.0] * 3),
                                           tg.Detector2D.centered(8, 8, 1, 1), math.pi, 60.0, 100.0,
                                           [[0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1]]),
     "matrix block is not invertible"),
    (lambda tg: tg.make_cone_from_matrices(tg.VolumeSpec.centered([8] * 3, [1.0] * 3),
                                           tg.Detector2D.centered(8, 8, 1, 1), math.pi, 60.0, 100.0,
                                           [[1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]]),
     "projection matrix puts the iso-center at zero depth"),
    (lambda tg: tg.parker_weights(tg.make_cone(tg.VolumeSpec.centered([8] * 3, [1.0] * 3),
                                               tg.Detector2D.centered(101, 5, 2, 2), 50,
                                               170 * math.pi / 180, 200.0, 400.0)),
     "scan range is too short for redundancy weighting (need pi + fan angle)"),
    (lambda tg: tg.VolumeSpec.centered([0, 4], [1.0, 1.0]), "volume shape entries must be >= 1"),
    (lambda tg: tg.Detector2D.centered(4, 4, -1.0, 1.0), "detector spacing must be positive"),
])
def test_reference_error_text(tg, call, msg):
    with pytest.raises(tg.Error) as e:
        call(tg)
    assert str(e.value) == msg
