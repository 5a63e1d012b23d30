"""GPU parity of the cone-beam kernels (K1 back-projection, K2 forward
projection) against the CPU oracle, through the C ABI.

Tolerance (stated): relRMSE <= 1e-5 and max|d| <= 1e-4 max|ref|
per operator; exact zeros / bitwise where the reference is exact."""
import math

import numpy as np
import pytest
import torch

from _helpers import assert_close, cone_pair, cone_pair_from_matrices, rand

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _bp(tg, geo, sino_np, **kw):
    s = tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=torch.from_numpy(sino_np).to(DEV))
    return tg.back_project(s, geo, **kw).data.cpu().numpy()


def _fp(tg, geo, vol_np):
    img = tg.Image(geo.volume, torch.from_numpy(vol_np).to(DEV))
    return tg.forward_project(img, geo).data.cpu().numpy()


# shipped FDK geometry (configs/fdk_short_scan_geometry.json): 64^3 @0.85 mm,
# 96^2 detector @1 mm, 248 views over 200 deg, SID 750 / SDD 1200
SHIPPED = dict(vshape=[64, 64, 64], vsp=[0.85] * 3, nu=96, nv=96, du=1.0, dv=1.0, n=248,
               rng=200 * math.pi / 180, sid=750.0, sdd=1200.0)

CASES = {
    "shipped": SHIPPED,
    "odd": dict(vshape=[37, 29, 23], vsp=[1.1, 0.9, 1.3], nu=45, nv=33, du=1.7, dv=1.5, n=30,
                rng=2 * math.pi, sid=120.0, sdd=250.0),
    "wide": dict(vshape=[40, 48, 36], vsp=[1.0] * 3, nu=128, nv=20, du=0.8, dv=2.5, n=17,
                 rng=math.pi, sid=200.0, sdd=330.0),
    # voxels behind the source / outside the detector: slow + skip paths
    "near": dict(vshape=[32, 32, 16], vsp=[4.0] * 3, nu=24, nv=12, du=2.0, dv=2.0, n=9,
                 rng=2 * math.pi, sid=50.0, sdd=90.0),
}


@pytest.mark.parametrize("case", list(CASES))
def test_cone_backproject_parity(tg, O, case):
    geo, og = cone_pair(tg, O, **CASES[case])
    s = rand(og.sino_shape, 8, -1.0, 1.0)
    assert_close(_bp(tg, geo, s), O.cone_backproject(og, s), what=f"cone BP {case}")


@pytest.mark.parametrize("case", list(CASES))
def test_cone_forward_parity(tg, O, case):
    geo, og = cone_pair(tg, O, **CASES[case])
    v = rand(og.vol_shape_zyx, 7)
    out, ref = _fp(tg, geo, v), O.cone_forward(og, v)
    assert_close(out, ref, what=f"cone FP {case}")
    # rays that miss the clip box integrate to exactly zero (projector.hpp:137)
    assert np.array_equal(out == 0.0, ref == 0.0)


def test_cone_calibrated_matrices(tg, O):
    """general (non-circular) path: tilted trajectory, P[0][2], P[2][2] != 0"""
    vol = tg.VolumeSpec.centered([40, 36, 32], [1.0, 1.0, 1.0])
    det = tg.Detector2D.centered(80, 72, 1.0, 1.0)
    mats = tg.projection_matrices_circular(40, 2 * math.pi, 300.0, 500.0, det)
    tilt = 0.15
    R = np.array([[1, 0, 0, 0], [0, math.cos(tilt), -math.sin(tilt), 0],
                  [0, math.sin(tilt), math.cos(tilt), 0], [0, 0, 0, 1]])
    mats = np.stack([(m.reshape(3, 4) @ R).reshape(12) * 3.0 for m in mats])
    geo, og = cone_pair_from_matrices(tg, O, vol, det, 2 * math.pi, 300.0, 500.0, mats)
    assert not geo.circular
    s = rand(og.sino_shape, 8, -1.0, 1.0)
    assert_close(_bp(tg, geo, s), O.cone_backproject(og, s), what="BP calibrated")
    v = rand(og.vol_shape_zyx, 7)
    assert_close(_fp(tg, geo, v), O.cone_forward(og, v), what="FP calibrated")


def test_cone_sphere_chords(tg):
    """test_projector.cpp:88-104 known answers"""
    vol = tg.VolumeSpec.centered([64, 64, 64], [1.0, 1.0, 1.0])
    R = 20.0
    sphere = tg.rasterize(np.array([[0, 0, 0, R, R, R, 0.0, 1.0]]), vol, device=DEV)
    det = tg.Detector2D.centered(63, 63, 2.0, 2.0)
    geo = tg.make_cone(vol, det, 1, math.pi, 200.0, 400.0)
    s = tg.forward_project(sphere, geo).data.cpu().numpy()
    assert abs(s[0, 31, 31] - 2 * R) <= 1.0
    d = 9.98752338
    assert abs(s[0, 31, 41] - 2 * math.sqrt(R * R - d * d)) <= 1.0
    assert s[0, 0, 0] == 0.0


def test_cone_bp_inverse_square_depth(tg):
    """test_projector.cpp:168-178: uniform sinogram -> (SID / depth)^2"""
    vol = tg.VolumeSpec.centered([5, 5, 5], [16.0, 16.0, 16.0])
    det = tg.Detector2D.centered(31, 31, 8.0, 8.0)
    geo = tg.make_cone(vol, det, 1, math.pi, 64.0, 128.0)
    img = _bp(tg, geo, np.ones((1, 31, 31), np.float32))
    assert img[2, 2, 0] == pytest.approx(4.0, abs=1e-5)
    assert img[2, 2, 2] == pytest.approx(1.0, abs=1e-6)
    assert img[2, 2, 4] == pytest.approx(4.0 / 9.0, abs=1e-6)


def test_cone_linearity_and_determinism(tg, O):
    geo, og = cone_pair(tg, O, **CASES["odd"])
    p, q = rand(og.sino_shape, 31), rand(og.sino_shape, 32)
    bp, bq, bc = _bp(tg, geo, p), _bp(tg, geo, q), _bp(tg, geo, (1.5 * p - q).astype(np.float32))
    assert np.max(np.abs(bc - (1.5 * bp - bq))) <= 1e-4 * np.max(np.abs(bc))
    # run to run bitwise (one writer per voxel, no atomics)
    assert np.array_equal(_bp(tg, geo, p), bp)
    v = rand(og.vol_shape_zyx, 11)
    assert np.array_equal(_fp(tg, geo, v), _fp(tg, geo, v))


def test_cone_scale_and_accumulate(tg, O):
    geo, og = cone_pair(tg, O, **CASES["wide"])
    s = torch.from_numpy(rand(og.sino_shape, 5)).to(DEV)
    L = tg._native.lib()
    out = torch.ones(geo.volume.torch_shape, device=DEV)
    st = torch.cuda.current_stream().cuda_stream
    tg._native.check(L.tg_cone_backproject(geo._plan(0), s.data_ptr(), out.data_ptr(), 0.5, 1, st))
    ref = O.cone_backproject(og, s.cpu().numpy())
    assert_close(out.cpu().numpy(), 1.0 + 0.5 * ref, what="scale+accumulate")


@pytest.mark.parametrize("z0,nz", [(0, 32), (16, 16), (32, 32), (48, 16), (5, 21)])
def test_cone_slab_band(tg, O, z0, nz):
    """z-slab back-projection from only its detector row band equals the same
    z range of the full-volume result (bitwise when aligned to K1's 32-voxel z tile)."""
    geo, og = cone_pair(tg, O, **SHIPPED)
    s = rand(og.sino_shape, 3, -1.0, 1.0)
    full = _bp(tg, geo, s)
    v0, nr = tg.cone_slab_rows(geo, z0, nz)
    band = torch.from_numpy(np.ascontiguousarray(s[:, v0:v0 + nr, :])).to(DEV)
    slab = tg.cone_backproject_slab(geo, band, z0, nz, v0).cpu().numpy()
    if z0 % 32 == 0 and (nz % 32 == 0 or z0 + nz == 64):  # K1's z tile
        assert np.array_equal(slab, full[z0:z0 + nz])
    else:
        assert_close(slab, full[z0:z0 + nz], what="unaligned slab")


def test_cone_views_shard(tg, O):
    geo, og = cone_pair(tg, O, **CASES["wide"])
    v = torch.from_numpy(rand(og.vol_shape_zyx, 2)).to(DEV)
    full = tg.forward_project(tg.Image(geo.volume, v), geo).data
    part = tg.cone_forward_views(geo, v, 5, 7)
    assert torch.equal(part, full[5:12])


def test_cone_host_variants(tg, O):
    """the reference's by-value host semantics through the *_host entry points"""
    geo, og = cone_pair(tg, O, **CASES["odd"])
    v = rand(og.vol_shape_zyx, 4)
    img = tg.Image(geo.volume, v)
    s = tg.forward_project(img, geo).data
    assert isinstance(s, np.ndarray)
    assert_close(s, O.cone_forward(og, v), what="host FP")
    sino = rand(og.sino_shape, 6, -1, 1)
    out = tg.back_project(tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=sino), geo).data
    assert_close(out, O.cone_backproject(og, sino), what="host BP")


def test_shape_errors(tg):
    vol = tg.VolumeSpec.centered([4, 4, 4], [1.0, 1.0, 1.0])
    det = tg.Detector2D.centered(8, 8, 1.0, 1.0)
    geo = tg.make_cone(vol, det, 3, math.pi, 10.0, 20.0)
    planar = tg.Sinogram.planar(3, tg.Detector1D.centered(8, 1.0), device=DEV)
    with pytest.raises(tg.Error, match="^sinogram shape does not match the geometry$"):
        tg.back_project(planar, geo)
    wrong = tg.Image(tg.VolumeSpec.centered([4, 4, 4], [2.0, 2.0, 2.0]), device=DEV)
    with pytest.raises(tg.Error, match="^volume does not match the geometry's volume spec$"):
        tg.forward_project(wrong, geo)


def test_cone_host_phased_upload(tg, O):
    """slabs of >= 128 slices back-project from host buffers with the centre-out
    upload order (csrc/cone.cu phased_backproject): same result as the device
    path up to the chunked view accumulation, for the whole volume and for a
    slab from its row band (2D row-segment uploads)"""
    vol = tg.VolumeSpec.centered([40, 36, 160], [1.0, 1.0, 1.0])
    det = tg.Detector2D.centered(72, 230, 1.5, 1.5)
    geo = tg.make_cone(vol, det, 24, 2 * math.pi, 300.0, 600.0)
    sino = rand((24, 230, 72), 9, -1.0, 1.0)
    dev = _bp(tg, geo, sino)
    host = tg.back_project(tg.Sinogram.cone_beam(24, det, data=sino), geo).data
    assert_close(host, dev, 2e-7, 2e-6, "phased host BP vs device")
    z0, nz = 16, 128
    v0, nr = tg.cone_slab_rows(geo, z0, nz)
    band = np.ascontiguousarray(sino[:, v0:v0 + nr, :])
    slab = np.zeros((nz, 36, 40), np.float32)
    tg._native.check(tg._native.lib().tg_cone_backproject_slab_host(
        geo._plan(0), z0, nz, v0, nr, band.ctypes.data, slab.ctypes.data, 0, 0))
    # same K1 tiles as the device slab launch from the band (z0 = 16 is not
    # 32-aligned to the volume, so compare with that rather than the volume)
    want = tg.cone_backproject_slab(geo, torch.from_numpy(band).to(DEV), z0, nz, v0).cpu().numpy()
    assert_close(slab, want, 2e-7, 2e-6, "phased host slab vs device slab")
    assert_close(slab, dev[z0:z0 + nz], what="phased host slab vs device volume")


@pytest.mark.parametrize("z0,nz", [(0, 160), (32, 64), (96, 40)])
def test_cone_host_footprint_upload(tg, O, z0, nz):
    """the phased host back-projection ships each view's own detector footprint
    only (csrc/cone.cu phased_backproject): detector pixels outside the taps any
    voxel interpolates may hold anything (NaN here, on the host and left over in
    the device staging buffer from a previous call) without changing a bit of
    the result, and fewer bytes than the band cross PCIe; whole volume and
    z-slabs (the 64-slice slab is the N = 8 bench shard's shape)"""
    vol = tg.VolumeSpec.centered([40, 36, 160], [1.0, 1.0, 1.0])
    det = tg.Detector2D.centered(200, 260, 1.5, 1.5)
    geo = tg.make_cone(vol, det, 24, 2 * math.pi, 300.0, 600.0)
    sino = rand((24, 260, 200), 11, -1.0, 1.0)
    # pixels any voxel centre's bilinear taps touch (FP64), dilated by one
    M = np.asarray(geo.matrices, np.float64).reshape(-1, 3, 4)
    xs = vol.origin[0] + np.arange(40) * 1.0
    ys = vol.origin[1] + np.arange(36) * 1.0
    zs = vol.origin[2] + np.arange(z0, z0 + nz) * 1.0
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel(), np.ones(X.size)])
    used = np.zeros(sino.shape, bool)
    for i in range(24):
        h = M[i] @ pts
        u, v = np.floor(h[0] / h[2]).astype(np.int64), np.floor(h[1] / h[2]).astype(np.int64)
        for dv in range(-1, 3):
            for du in range(-1, 3):
                uu, vv = u + du, v + dv
                ok = (uu >= 0) & (uu < 200) & (vv >= 0) & (vv < 260)
                used[i, vv[ok], uu[ok]] = True
    assert used.mean() < 0.6
    v0, nr = tg.cone_slab_rows(geo, z0, nz)
    band = np.ascontiguousarray(sino[:, v0:v0 + nr, :])
    want = tg.cone_backproject_slab(geo, torch.from_numpy(band).to(DEV), z0, nz, v0).cpu().numpy()
    dirty = np.ascontiguousarray(np.where(used, sino, np.float32(np.nan))[:, v0:v0 + nr, :])
    L = tg._native.lib()
    plan = geo._plan(0)
    nan_vol = np.zeros((nz, 36, 40), np.float32)
    all_nan = np.full(band.shape, np.nan, np.float32)
    tg._native.check(L.tg_cone_backproject_slab_host(plan, z0, nz, v0, nr, all_nan.ctypes.data,
                                                     nan_vol.ctypes.data, 0, 0))
    assert np.isnan(nan_vol).any()
    out = np.zeros((nz, 36, 40), np.float32)
    tg._native.check(L.tg_cone_backproject_slab_host(plan, z0, nz, v0, nr, dirty.ctypes.data,
                                                     out.ctypes.data, 0, 0))
    assert np.isfinite(out).all()
    assert_close(out, want, 2e-7, 2e-6, "footprint-upload host slab BP vs device slab BP")
    shipped = int(L.tg_cone_last_h2d_bytes(plan))
    assert 0 < shipped < 0.7 * band.nbytes


def test_cone_many_views_bank_blocks(tg, O):
    """more views than one constant-bank block (640): K1 launches split at the
    aligned block boundary; the device path and the host pipeline (PDL-chained
    chunk launches whose chunks start inside a block and straddle its end)
    both match the oracle"""
    geo, og = cone_pair(tg, O, [20, 18, 40], [1.0] * 3, 28, 48, 1.5, 1.5, 700, 2 * math.pi,
                        150.0, 300.0)
    s = rand(og.sino_shape, 12, -1.0, 1.0)
    ref = O.cone_backproject(og, s)
    dev = _bp(tg, geo, s)
    assert_close(dev, ref, what="cone BP, 700 views (device)")
    host = tg.back_project(tg.Sinogram.cone_beam(700, geo.detector, data=s), geo).data
    assert_close(host, ref, what="cone BP, 700 views (host pipeline)")
    # five partial fp32 sums (view chunks / bank blocks) instead of two
    assert_close(host, dev, 1e-6, 2e-6, "host pipeline vs device, 700 views")
