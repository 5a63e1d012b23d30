"""GPU parity of K3 (row filter with fused FDK weights) and the FDK / FBP
pipelines against the CPU oracle.  K3 replaces the reference's complex-double
FFT with an fp32 shared-memory FFT; the stated tolerance is the same FP32
bar: relRMSE <= 1e-5, max|d| <= 1e-4 max|ref|."""
import math

import numpy as np
import pytest
import torch

from _helpers import assert_close, cone_pair, planar_pair, rand

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


# 1025 / 1248 / 1280: window 4096 with the pruned radix-16 first / last passes
# (row within 5 x 256 samples); 1281: window 4096, half-window pruning only
@pytest.mark.parametrize("n,spacing", [(100, 0.7), (400, 1.0), (1248, 0.64), (365, 1.0), (5, 2.0),
                                       (1025, 0.5), (1280, 0.64), (1281, 0.64)])
def test_ramlak_filter_parity(tg, O, n, spacing):
    rows = rand((7, n), 5, -1, 1)
    filt = tg.ramlak_filter(n, spacing)
    assert np.array_equal(filt.weights, O.ramlak_weights(filt.padded_n, spacing))
    s = tg.Sinogram.planar(7, tg.Detector1D.centered(n, spacing), data=torch.from_numpy(rows).to(DEV))
    out = tg.apply_filter(s, filt).data.cpu().numpy()
    assert_close(out, O.apply_filter(rows, filt.weights), what=f"ramlak {n}")


def test_filter_delta_response(tg, O):
    """test_filtering.cpp:71-86: delta -> spacing * kernel at the wrapped offset"""
    nb, j0, ds = 100, 40, 0.7
    row = np.zeros((1, nb), np.float32)
    row[0, j0] = 1.0
    filt = tg.ramlak_filter(nb, ds)
    s = tg.Sinogram.planar(1, tg.Detector1D.centered(nb, ds), data=torch.from_numpy(row).to(DEV))
    out = tg.apply_filter(s, filt).data.cpu().numpy()[0]
    for j in range(nb):
        off = (j + filt.padded_n - j0) % filt.padded_n
        m = min(off, filt.padded_n - off)
        assert out[j] == pytest.approx(ds * tg.ramlak_spatial(m, ds), abs=1e-6)


def test_filter_nonsymmetric_weights(tg, O):
    """test_filtering.cpp:100-127 setting: random (non-symmetric) weights —
    symmetrised at plan creation, Re(IFFT(W X)) = IFFT(W_s X) for real rows"""
    nb, P = 10, 32
    rng = np.random.default_rng(6)
    rows = rng.uniform(-1, 1, (2, nb)).astype(np.float32)
    w = rng.uniform(-1, 1, P) + 2.0
    filt = tg.Filter1D(nb, P, 1.0, w)
    s = tg.Sinogram.planar(2, tg.Detector1D.centered(nb, 1.0), data=torch.from_numpy(rows).to(DEV))
    out = tg.apply_filter(s, filt).data.cpu().numpy()
    assert_close(out, O.apply_filter(rows, w), what="non-symmetric filter")


def test_filter_errors(tg):
    s = tg.Sinogram.planar(1, tg.Detector1D.centered(16, 1.0), device=DEV)
    with pytest.raises(tg.Error, match="^filter was built for a different detector width$"):
        tg.apply_filter(s, tg.ramp_filter(17, 1.0))
    with pytest.raises(tg.Error, match="^filter spacing does not match the detector spacing$"):
        tg.apply_filter(s, tg.ramp_filter(16, 1.5))
    with pytest.raises(tg.Error, match="^filter window is smaller than the detector row$"):
        tg.apply_filter(s, tg.Filter1D(16, 8, 1.0, np.ones(8)))
    with pytest.raises(tg.Error, match="^filter window is inconsistent with its weight vector$"):
        tg.apply_filter(s, tg.Filter1D(16, 32, 1.0, np.ones(31)))


FDK_CASES = {
    "shipped": dict(vshape=[64, 64, 64], vsp=[0.85] * 3, nu=96, nv=96, du=1.0, dv=1.0, n=248,
                    rng=200 * math.pi / 180, sid=750.0, sdd=1200.0),
    "c3_small": dict(vshape=[48, 48, 40], vsp=[2.5] * 3, nu=100, nv=150, du=4.0, dv=4.0, n=62,
                     rng=200 * math.pi / 180, sid=750.0, sdd=1200.0),
}


@pytest.mark.parametrize("case", list(FDK_CASES))
@pytest.mark.parametrize("parker", [True, False])
def test_fdk_parity(tg, O, case, parker):
    geo, og = cone_pair(tg, O, **FDK_CASES[case])
    ph = O.shepp_logan_3d(og.vol)
    sino = O.cone_forward(og, ph)
    rec = tg.fdk_reconstruct(tg.Sinogram.cone_beam(geo.n_projections, geo.detector,
                                                   data=torch.from_numpy(sino).to(DEV)), geo,
                             use_parker=parker)
    assert_close(rec.data.cpu().numpy(), O.fdk_reconstruct(og, sino, parker), what=f"FDK {case}")


def test_fdk_prefilter_band_and_weights(tg, O):
    """K3 on a detector row band with cosine + Parker fused equals the
    reference's apply_weights x2 + apply_filter on those rows"""
    geo, og = cone_pair(tg, O, **FDK_CASES["c3_small"])
    s = rand(og.sino_shape, 9, 0, 1)
    v0, nr = 37, 41
    band = torch.from_numpy(np.ascontiguousarray(s[:, v0:v0 + nr])).to(DEV)
    out = tg.fdk_prefilter(band, geo, True, v0=v0).cpu().numpy()
    w = O.apply_weights(s, O.cosine_weights_cone(og))
    pk = O.parker_weights_cone(og)
    w = O.apply_weights(w, np.repeat(pk[:, None, :], og.det.n_v, axis=1))
    ref = O.apply_filter(w, O.ramlak_weights(O.filter_window(og.det.n_u), og.det.spacing_u))
    assert_close(out, ref[:, v0:v0 + nr], what="prefilter band")


def test_fdk_host_pipeline(tg, O):
    geo, og = cone_pair(tg, O, **FDK_CASES["c3_small"])
    sino = O.cone_forward(og, O.shepp_logan_3d(og.vol))
    out = tg.fdk_reconstruct(tg.Sinogram.cone_beam(geo.n_projections, geo.detector, data=sino), geo)
    assert isinstance(out.data, np.ndarray)
    assert_close(out.data, O.fdk_reconstruct(og, sino), what="host FDK")


def test_parker_range_error(tg):
    vol = tg.VolumeSpec.centered([8, 8, 8], [1.0] * 3)
    geo = tg.make_cone(vol, tg.Detector2D.centered(101, 4, 2.0, 2.0), 50, 170 * math.pi / 180,
                       200.0, 400.0)
    s = tg.Sinogram.cone_beam(50, geo.detector, device=DEV)
    with pytest.raises(tg.Error, match=r"^scan range is too short for redundancy weighting \(need pi \+ fan angle\)$"):
        tg.fdk_reconstruct(s, geo)


def test_fbp_parity(tg, O):
    """c1-like: parallel 128^2, 180 views, FBP (Ram-Lak) vs the oracle"""
    geo, og = planar_pair(tg, O, [128, 128], [1.0, 1.0], 183, 1.0, 180, math.pi)
    ph = O.shepp_logan_2d(og.vol)
    sino = O.planar_forward(og, ph)
    rec = tg.fbp_reconstruct(tg.Sinogram.planar(180, geo.detector, data=torch.from_numpy(sino).to(DEV)),
                             geo)
    ref = O.fbp_reconstruct(og, sino, O.ramlak_weights(O.filter_window(183), 1.0))
    assert_close(rec.data.cpu().numpy(), ref, what="FBP")


@pytest.mark.parametrize("parker", [True, False])
@pytest.mark.parametrize("nu", [64, 260])
def test_fdk_host_row_band(tg, O, parker, nu):
    """FDK from a host sinogram (tg_cone_fdk_host, the C++ drop-in's path)
    uploads and filters only the detector rows the volume projects onto:
    rows outside that band may hold anything (NaN here) and the result still
    matches the device FDK of the clean data and the oracle.  nu = 64 (window
    128) takes the view-chunk pipeline, nu = 260 (window 1024) the centre-out
    phased one with strided row-segment filtering"""
    geo, og = cone_pair(tg, O, [40, 36, 24], [1.0] * 3, nu, 140, 1.0, 1.0, 60,
                        220 * math.pi / 180, 300.0, 600.0)
    ph = O.shepp_logan_3d(og.vol)
    sino = O.cone_forward(og, ph)
    v0, nr = tg.cone_slab_rows(geo, 0, 24)
    assert v0 > 10 and v0 + nr < 130
    dirty = sino.copy()
    dirty[:, :v0] = np.nan
    dirty[:, v0 + nr:] = np.nan
    host = tg.fdk_reconstruct(tg.Sinogram.cone_beam(60, geo.detector, data=dirty), geo,
                              use_parker=parker).data
    dev = tg.fdk_reconstruct(tg.Sinogram.cone_beam(60, geo.detector,
                                                   data=torch.from_numpy(sino).to(DEV)), geo,
                             use_parker=parker).data.cpu().numpy()
    assert np.isfinite(host).all()
    # chunked K1 accumulation (8 view chunks) vs one launch: fp32 sum order
    assert_close(host, dev, 1e-6, 2e-6, "host FDK (row band) vs device FDK")
    assert_close(host, O.fdk_reconstruct(og, sino, parker), what="host FDK vs oracle")
