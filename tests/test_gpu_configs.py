"""Parity at the BASELINE configs themselves, through the C ABI:

* bit-exact per-ray sample counts n = ceil((t1-t0)/step) and hit/miss
  (projector.hpp:83-107,117,138) from the device's own FP64 ray setup (the
  code K2 / K5 / K7 run) against the oracle's, at full c1, c2, c3 and on c4
  views, plus the exact c4 total;
* full-size c2 (fan 512^2, 360 x 1024: K5 / K4) and c3 (cone 256^3,
  248 x [400 x 600]: K2, K1, Parker FDK) against the oracle;
* sampled c5 (1024^3, 720 x [2048 x 1536]): two K2 views through the
  4-row-band cone_fp_kernel<64> the plan selects there, four K1 z-slices;
* K2 through both band heights (knob k2_tu 32 / 64) and without the
  y-fastest quad copy (k2_dual 0): bitwise identical outputs, parity;
* standalone apply_weights (filtering.hpp:136-154): bitwise, including the
  reference's two roundings (cosine, then Parker; pipelines.hpp:76-77).

Tolerance (tests/_helpers.py): relRMSE <= 1e-5 and
max|d| <= 1e-4 max|ref| per fp32 operator; bitwise for counts and weights."""
import json
import math
import os

import numpy as np
import pytest
import torch

from _helpers import assert_close, cone_pair, planar_pair, rand

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

C1 = dict(shape=[256, 256], sp=[1.0, 1.0], nb=365, db=1.0, n=360, rng=math.pi)
C2 = dict(shape=[512, 512], sp=[0.5, 0.5], nb=1024, db=0.8, n=360, rng=2 * math.pi, sid=750.0,
          sdd=1200.0)
C3 = dict(vshape=[256] * 3, vsp=[0.5] * 3, nu=400, nv=600, du=1.0, dv=1.0, n=248,
          rng=200 * math.pi / 180, sid=750.0, sdd=1200.0)


@pytest.fixture(scope="module", autouse=True)
def _threads(O):
    O.set_threads(os.cpu_count() or 1)


# ---- per-ray sample counts (row a7) -------------------------------------------


@pytest.mark.parametrize("case,total", [("c1", 47_610_000), ("c2", 192_400_000)])
def test_planar_ray_samples_bitwise(tg, O, case, total):
    geo, og = planar_pair(tg, O, **(C1 if case == "c1" else C2))
    dev = tg.ray_sample_counts(geo).cpu().numpy().astype(np.uint64)
    ref = O.planar_ray_samples(og)
    assert np.array_equal(dev, ref)
    # SURVEY §8a row a8 quotes the sums to 4 significant digits
    assert abs(int(ref.sum()) - total) <= 0.0005 * total


def test_cone_ray_samples_bitwise_c3(tg, O):
    geo, og = cone_pair(tg, O, C3["vshape"], C3["vsp"], C3["nu"], C3["nv"], C3["du"], C3["dv"],
                        C3["n"], C3["rng"], C3["sid"], C3["sdd"])
    dev = tg.ray_sample_counts(geo).cpu().numpy().astype(np.uint64)
    ref = O.cone_ray_samples(og)
    assert np.array_equal(dev, ref)
    assert int(ref.sum()) == pytest.approx(5.448906e9, rel=1e-6)
    # hit / miss: SURVEY §8a row a14 (1.44e7 of 5.95e7 rays hit at c3)
    assert int((ref > 0).sum()) == pytest.approx(1.44e7, rel=0.01)


@pytest.fixture(scope="module")
def c4(tg):
    vol = tg.VolumeSpec.centered([512] * 3, [0.5] * 3)
    det = tg.Detector2D.centered(1248, 960, 0.64, 0.64)
    return tg.make_cone(vol, det, 496, 220 * math.pi / 180, 750.0, 1200.0)


def test_cone_ray_samples_c4(tg, O, c4):
    """four c4 views bitwise against the oracle; the device total over all 496
    views equals the Σn bench.py divides by (profiles/c4_samples.json)"""
    views = [0, 137, 301, 495]
    og = O.cone_from_matrices(O.make_volume([512] * 3, [0.5] * 3),
                              O.det2_centered(1248, 960, 0.64, 0.64), c4.angular_range, c4.sid,
                              c4.sdd, c4.matrices[views])
    ref = O.cone_ray_samples(og)
    dev = np.stack([tg.ray_sample_counts(c4, v, 1)[0].cpu().numpy() for v in views])
    assert np.array_equal(dev.astype(np.uint64), ref)
    total = 0
    for v0 in range(0, 496, 62):
        total += int(tg.ray_sample_counts(c4, v0, 62).sum())
    with open(os.path.join(ROOT, "profiles", "c4_samples.json")) as f:
        assert total == int(json.load(f)["samples"]) == 217_954_916_998


# ---- full-size c2 / c3 ------------------------------------------------------------


def test_c2_fan_full(tg, O):
    geo, og = planar_pair(tg, O, **C2)
    ph = tg.shepp_logan_2d(geo.volume, device=DEV).data
    ph_np = ph.cpu().numpy()
    fp = tg.forward_project(tg.Image(geo.volume, ph), geo).data.cpu().numpy()
    ref = O.planar_forward(og, ph_np)
    assert_close(fp, ref, what="c2 fan FP (K5)")
    assert np.array_equal(fp == 0.0, ref == 0.0)
    s = rand(og.sino_shape, 21, -1, 1)
    bp = tg.back_project(tg.Sinogram.planar(geo.n_projections, geo.detector,
                                            data=torch.from_numpy(s).to(DEV)), geo).data
    assert_close(bp.cpu().numpy(), O.planar_backproject(og, s), what="c2 fan BP (K4)")


def test_c1_parallel_fbp_full(tg, O):
    geo, og = planar_pair(tg, O, **C1)
    ph = tg.shepp_logan_2d(geo.volume, device=DEV)
    sino = tg.forward_project(ph, geo)
    s_np = sino.data.cpu().numpy()
    rec = tg.fbp_reconstruct(sino, geo).data.cpu().numpy()
    P = tg.filter_window(geo.detector.n_bins)
    ref = O.fbp_reconstruct(og, s_np, O.ramlak_weights(P, geo.detector.spacing))
    assert_close(rec, ref, what="c1 FBP (K3 + K6)")


@pytest.fixture(scope="module")
def c3(tg, O):
    geo, og = cone_pair(tg, O, C3["vshape"], C3["vsp"], C3["nu"], C3["nv"], C3["du"], C3["dv"],
                        C3["n"], C3["rng"], C3["sid"], C3["sdd"])
    ph = tg.shepp_logan_3d(geo.volume, device=DEV).data
    sino = tg.forward_project(tg.Image(geo.volume, ph), geo).data
    return geo, og, ph, sino


def test_c3_forward_full(tg, O, c3):
    geo, og, ph, sino = c3
    ref = O.cone_forward(og, ph.cpu().numpy())
    out = sino.cpu().numpy()
    assert_close(out, ref, what="c3 cone FP (K2)")
    assert np.array_equal(out == 0.0, ref == 0.0)


def test_c3_backproject_full(tg, O, c3):
    geo, og, _, sino = c3
    s = sino.cpu().numpy()
    out = tg.back_project(tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=sino), geo)
    assert_close(out.data.cpu().numpy(), O.cone_backproject(og, s), what="c3 cone BP (K1)")


@pytest.mark.parametrize("parker", [True, False])
def test_c3_fdk_full(tg, O, c3, parker):
    geo, og, _, sino = c3
    s = sino.cpu().numpy()
    rec = tg.fdk_reconstruct(tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=sino),
                             geo, use_parker=parker).data.cpu().numpy()
    assert_close(rec, O.fdk_reconstruct(og, s, parker), what=f"c3 FDK parker={parker}")


# ---- K2 variants (band height, quad layouts) --------------------------------------

K2_CASES = {
    "shipped": dict(vshape=[64, 64, 64], vsp=[0.85] * 3, nu=96, nv=96, du=1.0, dv=1.0, n=248,
                    rng=200 * math.pi / 180, sid=750.0, sdd=1200.0),
    "odd": dict(vshape=[37, 29, 23], vsp=[1.1, 0.9, 1.3], nu=45, nv=33, du=1.7, dv=1.5, n=30,
                rng=2 * math.pi, sid=120.0, sdd=250.0),
    "wide": dict(vshape=[40, 48, 36], vsp=[1.0] * 3, nu=128, nv=20, du=0.8, dv=2.5, n=17,
                 rng=math.pi, sid=200.0, sdd=330.0),
}


@pytest.mark.parametrize("case", list(K2_CASES))
def test_k2_variants_bitwise(tg, O, case):
    """The slab-staged K2 (k2_impl 1, shared-memory boxes) and the quad-volume
    K2 (k2_impl 0) through both of its band heights (cone_fp_kernel<64> /
    <32>) and without its y-fastest copy (k2_dual 0) give the same bits: the
    sample positions and summation order are the same, only the tap source and
    the ray-to-CTA assignment differ."""
    c = K2_CASES[case]
    geo, og = cone_pair(tg, O, **c)
    v = rand(og.vol_shape_zyx, 5)
    img = tg.Image(geo.volume, torch.from_numpy(v).to(DEV))
    outs = {}
    tg.set_cone_knob(geo, "k2_impl", 0)
    for tu, dual in [(32, 1), (64, 1), (64, 0), (32, 0)]:
        tg.set_cone_knob(geo, "k2_tu", tu)
        tg.set_cone_knob(geo, "k2_dual", dual)
        outs[(0, tu, dual)] = tg.forward_project(img, geo).data.cpu().numpy()
    tg.set_cone_knob(geo, "k2_tu", 32)
    tg.set_cone_knob(geo, "k2_dual", 1)
    tg.set_cone_knob(geo, "k2_impl", 1)
    outs[(1,)] = tg.forward_project(img, geo).data.cpu().numpy()
    ref = O.cone_forward(og, v)
    assert_close(outs[(1,)], ref, what=f"K2 slab {case}")
    assert_close(outs[(0, 64, 1)], ref, what=f"K2<64> {case}")
    for k, o in outs.items():
        assert np.array_equal(o, outs[(1,)]), k


def test_k2_slab_fallback_paths_bitwise(tg, O, monkeypatch):
    """The slab-staged K2's fallbacks give the same bits as its shared-memory
    path: (1) boxes forced too small (every slab gathers from global memory),
    (2) z-dominant rays (calibrated matrices with x and z swapped: no x/y
    dominant axis, the CTA marches in one global pass)."""
    c = K2_CASES["shipped"]
    geo, og = cone_pair(tg, O, **c)
    v = rand(og.vol_shape_zyx, 9)
    img = tg.Image(geo.volume, torch.from_numpy(v).to(DEV))
    want = tg.forward_project(img, geo).data.cpu().numpy()
    monkeypatch.setenv("TG_K2_HZ", "4")
    geo_s, _ = cone_pair(tg, O, **c)  # fresh plan: boxes sized at its first forward
    got = tg.forward_project(img, geo_s).data.cpu().numpy()
    monkeypatch.delenv("TG_K2_HZ")
    assert np.array_equal(got, want)
    # z-dominant: permute the x and z columns of every projection matrix
    vol = tg.VolumeSpec.centered([40, 40, 40], [1.0] * 3)
    det = tg.Detector2D.centered(64, 64, 1.2, 1.2)
    base = tg.make_cone(vol, det, 24, 2 * math.pi, 200.0, 400.0)
    m = base.matrices.reshape(-1, 3, 4).copy()
    m[:, :, [0, 2]] = m[:, :, [2, 0]]
    mats = m.reshape(base.matrices.shape)
    from _helpers import cone_pair_from_matrices
    geo_z, og_z = cone_pair_from_matrices(tg, O, vol, det, 2 * math.pi, 200.0, 400.0, mats)
    vz = rand(og_z.vol_shape_zyx, 10)
    imz = tg.Image(geo_z.volume, torch.from_numpy(vz).to(DEV))
    tg.set_cone_knob(geo_z, "k2_impl", 1)
    slab = tg.forward_project(imz, geo_z).data.cpu().numpy()
    tg.set_cone_knob(geo_z, "k2_impl", 0)
    quad = tg.forward_project(imz, geo_z).data.cpu().numpy()
    assert np.array_equal(slab, quad)
    assert_close(slab, O.cone_forward(og_z, vz), what="K2 z-dominant")


# ---- c5 sampled -------------------------------------------------------------------


@pytest.fixture(scope="module")
def c5(tg):
    vol = tg.VolumeSpec.centered([1024] * 3, [0.25] * 3)
    det = tg.Detector2D.centered(2048, 1536, 0.4, 0.4)
    return tg.make_cone(vol, det, 720, 2 * math.pi, 750.0, 1200.0)


def test_c5_forward_views(tg, O, c5):
    """K2 at c5 (slab-staged; its 72-wide boxes where the plan's sizing picks
    them): two views of the 1024^3 Shepp-Logan against the oracle, exact zero
    pattern"""
    ph = tg.shepp_logan_3d(c5.volume, device=DEV).data
    views = [5, 410]
    out = torch.stack([tg.cone_forward_views(c5, ph, v, 1)[0] for v in views]).cpu().numpy()
    og = O.cone_from_matrices(O.make_volume([1024] * 3, [0.25] * 3),
                              O.det2_centered(2048, 1536, 0.4, 0.4), c5.angular_range, c5.sid,
                              c5.sdd, c5.matrices[views])
    ref = O.cone_forward(og, ph.cpu().numpy())
    assert_close(out, ref, what="c5 FP views")
    assert np.array_equal(out == 0.0, ref == 0.0)
    # the counts K2 marched at c5 match the oracle's too
    dev = np.stack([tg.ray_sample_counts(c5, v, 1)[0].cpu().numpy() for v in views])
    assert np.array_equal(dev.astype(np.uint64), O.cone_ray_samples(og))


def test_c5_backproject_slices(tg, O, c5):
    """K1 at c5 on 32-slice slabs (bitwise equal to the full volume's slices)
    from their detector row bands; two slices of each slab against the
    oracle on the same (zero-embedded) projections"""
    nu, nv, npj = 2048, 1536, 720
    for z0, picks in [(0, (0, 31)), (512, (3, 20))]:
        v0, nr = tg.cone_slab_rows(c5, z0, 32)
        band = torch.from_numpy(rand((npj, nr, nu), 100 + z0, -1, 1)).to(DEV)
        slab = tg.cone_backproject_slab(c5, band, z0, 32, v0).cpu().numpy()
        sino = np.zeros((npj, nv, nu), np.float32)  # lazily zero pages: only the band is touched
        sino[:, v0:v0 + nr] = band.cpu().numpy()
        for k in picks:
            z = z0 + k
            origin = list(c5.volume.origin)
            origin[2] += z * c5.volume.spacing[2]
            og = O.cone_from_matrices(O.make_volume([1024, 1024, 1], [0.25] * 3, origin),
                                      O.det2_centered(nu, nv, 0.4, 0.4), c5.angular_range,
                                      c5.sid, c5.sdd, c5.matrices)
            assert_close(slab[k:k + 1], O.cone_backproject(og, sino), what=f"c5 BP slice {z}")
        del sino


# ---- apply_weights (row a18) ------------------------------------------------------


def test_apply_weights_bitwise_two_roundings(tg, O):
    """filtering.hpp:136-154 on the device: out = T(double(x) w) for a full
    per-element map, a detector map broadcast over views (cosine) and the cone
    Parker row profile (tg_apply_row_weights); composed as the reference's FDK
    does (cosine, then Parker, each rounded to fp32: pipelines.hpp:76-77)"""
    c = dict(vshape=[40, 40, 30], vsp=[1.0] * 3, nu=77, nv=41, du=1.1, dv=1.3, n=33,
             rng=210 * math.pi / 180, sid=300.0, sdd=520.0)
    geo, og = cone_pair(tg, O, **c)
    p = rand(og.sino_shape, 9, -2, 3)
    sino = tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=torch.from_numpy(p).to(DEV))
    cw, pw = tg.cosine_weights(geo), tg.parker_weights(geo)
    a = tg.apply_weights(sino, cw)
    b = tg.apply_weights(a, pw)
    ref_a = O.apply_weights(p, O.cosine_weights_cone(og))
    ref_b = O.apply_weights(ref_a, np.repeat(O.parker_weights_cone(og)[:, None, :], 41, axis=1))
    assert np.array_equal(a.data.cpu().numpy(), ref_a)
    assert np.array_equal(b.data.cpu().numpy(), ref_b)
    # a full per-element map (the reference's materialised Parker map)
    full = tg.WeightMap(pw.shape, pw.full())
    assert np.array_equal(tg.apply_weights(a, full).data.cpu().numpy(), ref_b)
    # host input: same bits through the same kernel
    hb = tg.apply_weights(tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=ref_a), pw)
    assert np.array_equal(hb.data, ref_b)


def test_apply_weights_fan_bitwise(tg, O):
    geo, og = planar_pair(tg, O, shape=[64, 64], sp=[1.0, 1.0], nb=97, db=1.3, n=40,
                          rng=230 * math.pi / 180, sid=400.0, sdd=700.0)
    p = rand(og.sino_shape, 4, -1, 1)
    sino = tg.Sinogram.planar(geo.n_projections, geo.detector, data=torch.from_numpy(p).to(DEV))
    a = tg.apply_weights(sino, tg.cosine_weights(geo))
    b = tg.apply_weights(a, tg.parker_weights(geo))
    ref_a = O.apply_weights(p, O.cosine_weights_fan(og))
    ref_b = O.apply_weights(ref_a, O.parker_weights_fan(og))
    assert np.array_equal(a.data.cpu().numpy(), ref_a)
    assert np.array_equal(b.data.cpu().numpy(), ref_b)
