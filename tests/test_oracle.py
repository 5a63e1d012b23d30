"""Pinning the CPU oracle (test infrastructure) before it is trusted:

1. bitwise against the committed golden fixtures made by the reference itself
   (tests/golden/make_golden.py runs oracle/_ref);
2. bitwise against the compiled reference directly (oracle/_ref), when built;
3. against the known answers of the reference's own test suites
   (proj/tests/test_projector.cpp, test_geometry.cpp, test_filtering.cpp,
   test_pipelines.cpp, acceptance.cpp), re-expressed here.
"""
import math
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


# ---------------------------------------------------------------- golden ----

@pytest.mark.parametrize("name", ["cone_fdk_shortscan", "cone_odd"])
def test_oracle_matches_golden_cone(O, name):
    d = _load(name)
    vol = O.make_volume(list(d["vshape"]), list(d["vsp"]))
    nu, nv, du, dv = d["det"]
    det = O.det2_centered(int(nu), int(nv), du, dv)
    g = O.make_cone(vol, det, int(d["n"]), float(d["rng"]), float(d["sid"]), float(d["sdd"]))
    for k, gk in [("mats", "mats"), ("sources", "sources"), ("invs", "invs"), ("angles", "angles")]:
        assert np.array_equal(getattr(g, gk), d[k]), k
    ph = O.shepp_logan_3d(vol)
    assert np.array_equal(ph, d["phantom"])
    assert np.array_equal(O.cone_forward(g, ph), d["fp"])
    assert np.array_equal(O.cone_backproject(g, d["bp_in"]), d["bp"])
    assert np.array_equal(O.cosine_weights_cone(g), d["cosine"])
    if "parker" in d:
        assert np.array_equal(O.parker_weights_cone(g), d["parker"])
        assert np.array_equal(O.fdk_reconstruct(g, d["fp"], True), d["fdk"])
    assert np.array_equal(O.fdk_reconstruct(g, d["fp"], False), d["fdk_noparker"])


@pytest.mark.parametrize("name", ["parallel_fbp", "fan_full"])
def test_oracle_matches_golden_planar(O, name):
    d = _load(name)
    vol = O.make_volume(list(d["shape"]), list(d["sp"]))
    det = O.det1_centered(int(d["nb"]), float(d["db"]))
    g = O.make_planar(vol, det, int(d["n"]), float(d["rng"]), float(d["sid"]), float(d["sdd"]))
    assert np.array_equal(g.rays, d["rays"]) and np.array_equal(g.angles, d["angles"])
    ph = O.shepp_logan_2d(vol)
    assert np.array_equal(ph, d["phantom"])
    assert np.array_equal(O.planar_forward(g, ph), d["fp"])
    assert np.array_equal(O.planar_backproject(g, d["bp_in"]), d["bp"])
    if "fbp" in d:
        P = O.filter_window(int(d["nb"]))
        assert np.array_equal(O.fbp_reconstruct(g, d["fp"], O.ramlak_weights(P, float(d["db"]))),
                              d["fbp"])
        assert np.array_equal(O.fbp_reconstruct(g, d["fp"], O.ramp_weights(P, float(d["db"]))),
                              d["fbp_ramp"])
    if "cosine" in d:
        assert np.array_equal(O.cosine_weights_fan(g), d["cosine"])
    if "parker" in d:
        assert np.array_equal(O.parker_weights_fan(g).reshape(-1), d["parker"].reshape(-1))


def test_oracle_matches_golden_filters(O):
    d = _load("filters")
    for P, ds in [(32, 1.0), (256, 0.7), (1024, 1.0), (4096, 0.64)]:
        assert np.array_equal(O.ramlak_weights(P, ds), d[f"ramlak_{P}"])
        assert np.array_equal(O.ramp_weights(P, ds), d[f"ramp_{P}"])
    assert np.array_equal(O.apply_filter(d["rows"], O.ramlak_weights(256, 0.7)), d["rows_ramlak"])
    assert np.array_equal(O.apply_filter(d["rows64"], d["w_nonsym"]), d["rows64_nonsym"])


# ------------------------------------------------ the reference directly ----

needs_ref = pytest.mark.skipif(not os.path.exists(
    os.path.join(HERE, "..", "oracle", "_ref", "libtomograd_ref.so")),
    reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_bitwise_vs_reference_cone(O, seed):
    rng = np.random.default_rng(seed)
    shape = [int(v) for v in rng.integers(5, 19, 3)]
    sp = [float(v) for v in rng.uniform(0.6, 1.6, 3)]
    vol = O.make_volume(shape, sp)
    det = O.det2_centered(int(rng.integers(7, 31)), int(rng.integers(5, 25)), 1.3, 1.1)
    g = O.make_cone(vol, det, int(rng.integers(3, 17)), 2 * math.pi * float(rng.uniform(0.6, 1.0)),
                    90.0, 210.0)
    r = O.Ref.make_cone(vol, det, g.n_proj, g.range, g.sid, g.sdd)
    for k in ["mats", "sources", "invs", "angles"]:
        assert np.array_equal(getattr(g, k), getattr(r, k))
    for dt in [np.float32, np.float64]:
        v = rng.random(g.vol_shape_zyx).astype(dt)
        assert np.array_equal(O.cone_forward(g, v), O.Ref.cone_forward(r, v))
        s = rng.random(g.sino_shape).astype(dt)
        assert np.array_equal(O.cone_backproject(g, s), O.Ref.cone_backproject(r, s))
        assert np.array_equal(O.fdk_reconstruct(g, s, False), O.Ref.fdk_reconstruct(r, s, False))


@needs_ref
def test_oracle_bitwise_vs_reference_matrices(O):
    """make_cone_from_matrices: scaled and tilted matrices"""
    vol = O.make_volume([9, 8, 7], [1.0, 1.0, 1.0])
    det = O.det2_centered(16, 12, 1.0, 1.0)
    base = O.make_cone(vol, det, 5, math.pi, 60.0, 100.0).mats
    t = 0.2
    R = np.array([[1, 0, 0, 0], [0, math.cos(t), -math.sin(t), 0], [0, math.sin(t), math.cos(t), 0],
                  [0, 0, 0, 1]])
    mats = np.stack([(m.reshape(3, 4) @ R).reshape(12) * 7.0 for m in base])
    a = O.cone_from_matrices(vol, det, math.pi, 60.0, 100.0, mats)
    b = O.Ref.cone_from_matrices(vol, det, math.pi, 60.0, 100.0, mats)
    for k in ["mats", "sources", "invs", "angles"]:
        assert np.array_equal(getattr(a, k), getattr(b, k))
    v = np.random.default_rng(3).random(a.vol_shape_zyx).astype(np.float32)
    assert np.array_equal(O.cone_forward(a, v), O.Ref.cone_forward(b, v))


@needs_ref
@pytest.mark.parametrize("fan", [False, True])
def test_oracle_bitwise_vs_reference_planar(O, fan):
    vol = O.make_volume([23, 19], [1.1, 0.8])
    det = O.det1_centered(37, 0.9)
    sid, sdd = (70.0, 140.0) if fan else (0.0, 0.0)
    g = O.make_planar(vol, det, 17, 2 * math.pi, sid, sdd)
    r = O.Ref.planar_geometry(vol, det, 17, 2 * math.pi, sid, sdd)
    assert np.array_equal(g.rays, r.rays)
    img = np.random.default_rng(4).random(g.img_shape_yx)
    assert np.array_equal(O.planar_forward(g, img), O.Ref.planar_forward(r, img))
    s = np.random.default_rng(5).random(g.sino_shape).astype(np.float32)
    assert np.array_equal(O.planar_backproject(g, s), O.Ref.planar_backproject(r, s))


@needs_ref
def test_oracle_bitwise_vs_reference_weights(O):
    vol = O.make_volume([8, 8, 8], [1.0] * 3)
    det = O.det2_centered(101, 7, 2.0, 2.0)
    g = O.make_cone(vol, det, 40, 210 * math.pi / 180, 200.0, 400.0)
    r = O.Ref.make_cone(vol, det, 40, 210 * math.pi / 180, 200.0, 400.0)
    assert np.array_equal(O.cosine_weights_cone(g), O.Ref.cosine_weights_cone(r))
    assert np.array_equal(O.parker_weights_cone(g), O.Ref.parker_weights_cone(r))
    for P, ds in [(2, 1.0), (64, 0.5), (8192, 0.4)]:
        assert np.array_equal(O.ramlak_weights(P, ds), O.Ref.ramlak_weights(P, ds))


# ----------------------------------------- reference test-suite answers ----

def test_kat_uniform_box(O):
    """test_projector.cpp:34-45"""
    vol = O.make_volume([15, 15], [1.0, 1.0])
    g = O.make_planar(vol, O.det1_centered(15, 1.0), 1, math.pi)
    s = O.planar_forward(g, np.ones((15, 15)))
    assert np.allclose(s, 15.0, atol=1e-9)


def test_kat_cone_sphere_chords(O):
    """test_projector.cpp:88-104"""
    vol = O.make_volume([64, 64, 64], [1.0] * 3)
    R = 20.0
    sph = O.rasterize_ellipsoids(vol, [[0, 0, 0, R, R, R, 0.0, 1.0]])
    g = O.make_cone(vol, O.det2_centered(63, 63, 2.0, 2.0), 1, math.pi, 200.0, 400.0)
    s = O.cone_forward(g, sph)
    assert abs(s[0, 31, 31] - 2 * R) <= 1.0
    d = 9.98752338
    assert abs(s[0, 31, 41] - 2 * math.sqrt(R * R - d * d)) <= 1.0
    assert s[0, 0, 0] == 0.0


def test_kat_missed_rays_exact_zero(O):
    """test_projector.cpp:106-116"""
    vol = O.make_volume([64, 64], [1.0, 1.0])
    disk = O.rasterize_ellipses(vol, [[0, 0, 10.0, 10.0, 0.0, 1.0]])
    g = O.make_planar(vol, O.det1_centered(63, 1.0), 8, math.pi)
    s = O.planar_forward(g, disk)
    sb = g.det.origin + np.arange(63) * g.det.spacing
    assert np.all(s[:, np.abs(sb) >= 12.0] == 0.0)


def test_kat_backprojection_weights(O):
    """test_projector.cpp:134-178: parallel counts views; fan 1/U^2; cone 1/w^2"""
    vol = O.make_volume([9, 9], [1.0, 1.0])
    g = O.make_planar(vol, O.det1_centered(15, 1.0), 12, 2 * math.pi)
    img = O.planar_backproject(g, np.ones((12, 15)))
    assert img[4, 4] == 12.0 and np.allclose(img, 12.0, atol=1e-12)
    vol = O.make_volume([5, 5], [16.0, 16.0])
    g = O.make_planar(vol, O.det1_centered(31, 8.0), 1, math.pi, 64.0, 128.0)
    img = O.planar_backproject(g, np.ones((1, 31)))
    assert img[2, 0] == pytest.approx(4.0, abs=1e-12)
    assert img[2, 2] == pytest.approx(1.0, abs=1e-12)
    assert img[2, 4] == pytest.approx(4.0 / 9.0, abs=1e-12)
    vol = O.make_volume([5, 5, 5], [16.0] * 3)
    g = O.make_cone(vol, O.det2_centered(31, 31, 8.0, 8.0), 1, math.pi, 64.0, 128.0)
    img = O.cone_backproject(g, np.ones((1, 31, 31)))
    assert img[2, 2, 0] == pytest.approx(4.0, abs=1e-12)
    assert img[2, 2, 2] == pytest.approx(1.0, abs=1e-12)
    assert img[2, 2, 4] == pytest.approx(4.0 / 9.0, abs=1e-12)


def test_kat_adjointness(O):
    """test_projector.cpp:198-212"""
    vol = O.make_volume([32, 32], [1.0, 1.0])
    g = O.make_planar(vol, O.det1_centered(47, 1.0), 12, math.pi)
    rng = np.random.default_rng(7)
    f = rng.random((32, 32))
    p = rng.random((12, 47))
    lhs = float(np.sum(O.planar_forward(g, f) * p))
    rhs = float(np.sum(f * O.planar_backproject(g, p)))
    assert lhs / rhs == pytest.approx(1.0, abs=0.05)


def test_kat_geometry(O):
    """test_geometry.cpp:63-115: magnification, sources"""
    det = O.det2_centered(4, 4, 2.0, 2.0)
    P = np.zeros(12)
    O.lib().or_cone_projection_matrix(0.0, 100.0, 200.0, O.C.byref(det), O._ptr(P))
    P = P.reshape(3, 4)
    h = P @ np.array([0.0, 10.0, 0.0, 1.0])
    assert det.origin_u + (h[0] / h[2]) * det.spacing_u == pytest.approx(20.0)
    vol = O.make_volume([8, 8, 8], [1.0] * 3)
    g = O.make_cone(vol, O.det2_centered(16, 16, 1.0, 1.0), 6, 200 * math.pi / 180, 75.0, 120.0)
    for i in range(6):
        t = g.angles[i]
        assert g.sources[i, 0] == pytest.approx(-75.0 * math.cos(t), abs=1e-9)
        assert g.sources[i, 1] == pytest.approx(-75.0 * math.sin(t), abs=1e-9)


def test_kat_filters(O):
    """test_filtering.cpp:25-86"""
    assert O.ramlak_spatial(0, 1.0) == 0.25
    assert O.ramlak_spatial(2, 1.0) == 0.0
    assert O.ramlak_spatial(3, 1.0) == pytest.approx(-1.0 / (9 * math.pi ** 2))
    assert O.filter_window(100) == 256 and O.filter_window(64) == 128 and O.filter_window(65) == 256
    nb, j0, ds = 100, 40, 0.7
    row = np.zeros((1, nb))
    row[0, j0] = 1.0
    P = O.filter_window(nb)
    out = O.apply_filter(row, O.ramlak_weights(P, ds))[0]
    for j in range(nb):
        off = (j + P - j0) % P
        assert out[j] == pytest.approx(ds * O.ramlak_spatial(min(off, P - off), ds), abs=1e-9)


def test_kat_parker_conjugates(O):
    """test_filtering.cpp:163-190: conjugate rays sum to one"""
    rng_ = 200 * math.pi / 180
    delta = 0.5 * (rng_ - math.pi)
    for gi in range(-9, 10, 3):
        gamma = 0.1 * gi * delta
        for bi in range(0, 401, 7):
            beta = rng_ * bi / 400
            w = O.parker_weight(beta, gamma, delta, rng_)
            assert 0.0 <= w <= 1.0
            fwd = beta + math.pi + 2 * gamma
            if fwd <= rng_:
                assert w + O.parker_weight(fwd, -gamma, delta, rng_) == pytest.approx(1.0, abs=1e-6)


def test_kat_fdk_sphere_amplitude(O):
    """test_pipelines.cpp:86-103 style: a unit sphere reconstructs near 1"""
    vol = O.make_volume([40, 40, 40], [1.0] * 3)
    sph = O.rasterize_ellipsoids(vol, [[0, 0, 0, 12.0, 12.0, 12.0, 0.0, 1.0]])
    det = O.det2_centered(64, 64, 1.6, 1.6)
    g = O.make_cone(vol, det, 90, 2 * math.pi, 300.0, 480.0)
    rec = O.fdk_reconstruct(g, O.cone_forward(g, sph), False)
    assert rec[20, 20, 20] == pytest.approx(1.0, abs=0.05)
