"""Shared test helpers: build the same geometry in the product (through the
C ABI) and in the CPU oracle, and compare results with the SURVEY §8c
metrics."""
import numpy as np

# FP32-lerp parity tolerance for every operator:
# relative RMSE and max |d| relative to max |ref|.
REL_RMSE = 1e-5
REL_MAX = 1e-4
# The standalone row filter (K3) on smooth projections: the Ram-Lak taps sum
# to zero, so the filtered row is a cancellation much smaller than its input
# and fp32 FFT rounding (~eps log2 P |x|) is amplified relative to |y|; the
# reference does this in complex double.  Stated bound for the filter output
# alone; FDK volumes (after the 1/w^2 sum over views) meet REL_RMSE.
FILTER_REL_RMSE = 5e-5


def cone_pair(tg, O, vshape, vsp, nu, nv, du, dv, n, rng, sid, sdd, origin=None):
    if origin is None:
        vol = tg.VolumeSpec.centered(vshape, vsp)
    else:
        vol = tg.VolumeSpec(list(vshape), list(vsp), list(origin))
    det = tg.Detector2D.centered(nu, nv, du, dv)
    geo = tg.make_cone(vol, det, n, rng, sid, sdd)
    ov = O.make_volume(vol.shape, vol.spacing, vol.origin)
    od = O.or_det2(det.n_u, det.n_v, det.spacing_u, det.spacing_v, det.origin_u, det.origin_v)
    og = O.make_cone(ov, od, n, rng, sid, sdd)
    assert np.array_equal(geo.matrices, og.mats)
    return geo, og


def cone_pair_from_matrices(tg, O, vol, det, rng, sid, sdd, mats):
    geo = tg.make_cone_from_matrices(vol, det, rng, sid, sdd, mats)
    ov = O.make_volume(vol.shape, vol.spacing, vol.origin)
    od = O.or_det2(det.n_u, det.n_v, det.spacing_u, det.spacing_v, det.origin_u, det.origin_v)
    og = O.cone_from_matrices(ov, od, rng, sid, sdd, mats)
    assert np.array_equal(geo.matrices, og.mats)
    return geo, og


def planar_pair(tg, O, shape, sp, nb, db, n, rng, sid=0.0, sdd=0.0):
    vol = tg.VolumeSpec.centered(shape, sp)
    det = tg.Detector1D.centered(nb, db)
    if sdd > 0:
        geo = tg.make_fan(vol, det, n, rng, sid, sdd)
    else:
        geo = tg.make_parallel(vol, det, n, rng)
    ov = O.make_volume(vol.shape, vol.spacing, vol.origin)
    og = O.make_planar(ov, O.or_det1(det.n_bins, det.spacing, det.origin), n, rng, sid, sdd)
    assert np.array_equal(geo.rays, og.rays)
    return geo, og


def assert_close(out, ref, rel_rmse=REL_RMSE, rel_max=REL_MAX, what=""):
    import oracle as O
    mx, rr = O.rel_errors(np.asarray(out), np.asarray(ref))
    assert rr <= rel_rmse and mx <= rel_max, f"{what}: relRMSE {rr:.3g} (<= {rel_rmse}), " \
                                             f"max|d|/max|ref| {mx:.3g} (<= {rel_max})"
    return mx, rr


def rand(shape, seed, lo=0.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape).astype(np.float32)
