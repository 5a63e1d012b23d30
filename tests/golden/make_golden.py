"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, the
reference's own headers compiled by oracle/Makefile), so the oracle and the
product stay pinned even where /root/reference is not mounted.

    python tests/golden/make_golden.py

Cases are small (the whole set is well under 2 MB) and use T = float storage
(double maths) like the GPU path, plus a few T = double cases.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

R = O.Ref


def cone_case(name, vshape, vsp, nu, nv, du, dv, n, rng, sid, sdd, seed):
    vol = O.make_volume(vshape, vsp)
    det = O.det2_centered(nu, nv, du, dv)
    g = R.make_cone(vol, det, n, rng, sid, sdd)
    ph = R.shepp_logan_3d(vol)
    sino = R.cone_forward(g, ph)
    rs = np.random.default_rng(seed).uniform(-1, 1, g.sino_shape).astype(np.float32)
    bp = R.cone_backproject(g, rs)
    out = dict(vshape=np.array(vshape), vsp=np.array(vsp, float), det=np.array([nu, nv, du, dv], float),
               n=n, rng=rng, sid=sid, sdd=sdd, mats=g.mats, sources=g.sources, invs=g.invs,
               angles=g.angles, phantom=ph, fp=sino, bp_in=rs, bp=bp,
               cosine=R.cosine_weights_cone(g))
    try:
        out["parker"] = R.parker_weights_cone(g)
        out["fdk"] = R.fdk_reconstruct(g, sino, True)
    except O.OracleError:
        pass
    out["fdk_noparker"] = R.fdk_reconstruct(g, sino, False)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def planar_case(name, shape, sp, nb, db, n, rng, sid, sdd, seed):
    vol = O.make_volume(shape, sp)
    det = O.det1_centered(nb, db)
    g = R.planar_geometry(vol, det, n, rng, sid, sdd)
    ph = R.shepp_logan_2d(vol)
    sino = R.planar_forward(g, ph)
    rs = np.random.default_rng(seed).uniform(-1, 1, g.sino_shape).astype(np.float32)
    out = dict(shape=np.array(shape), sp=np.array(sp, float), nb=nb, db=db, n=n, rng=rng, sid=sid,
               sdd=sdd, rays=g.rays, angles=g.angles, phantom=ph, fp=sino, bp_in=rs,
               bp=R.planar_backproject(g, rs))
    if sdd == 0.0:
        out["fbp"] = R.fbp_reconstruct(g, sino, True)
        out["fbp_ramp"] = R.fbp_reconstruct(g, sino, False)
    else:
        out["cosine"] = R.cosine_weights_fan(g)
        try:
            out["parker"] = R.parker_weights_fan(g)
        except O.OracleError:
            pass
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def filters():
    out = {}
    for P, ds in [(32, 1.0), (256, 0.7), (1024, 1.0), (4096, 0.64)]:
        out[f"ramlak_{P}"] = R.ramlak_weights(P, ds)
        out[f"ramp_{P}"] = R.ramp_weights(P, ds)
    rows = np.random.default_rng(5).uniform(-1, 1, (3, 100)).astype(np.float32)
    out["rows"] = rows
    out["rows_ramlak"] = R.apply_filter(rows, 0.7, R.ramlak_weights(256, 0.7))
    w = np.random.default_rng(6).uniform(-1, 1, 32) + 2.0
    rows64 = np.random.default_rng(7).uniform(-1, 1, (2, 10))
    out["rows64"] = rows64
    out["w_nonsym"] = w
    out["rows64_nonsym"] = R.apply_filter(rows64, 1.0, w)
    np.savez_compressed(os.path.join(HERE, "filters.npz"), **out)


def main():
    assert O.ref_available(), "needs oracle/_ref (make -C oracle with /root/reference mounted)"
    R.set_threads(os.cpu_count() or 1)
    cone_case("cone_fdk_shortscan", [32, 32, 24], [1.7, 1.7, 1.7], 48, 40, 2.0, 2.0, 62,
              200 * math.pi / 180, 750.0, 1200.0, 8)
    cone_case("cone_odd", [21, 17, 13], [1.1, 0.9, 1.3], 29, 23, 1.7, 1.5, 11, 2 * math.pi,
              120.0, 250.0, 9)
    planar_case("parallel_fbp", [64, 64], [1.0, 1.0], 91, 1.0, 45, math.pi, 0.0, 0.0, 10)
    planar_case("fan_full", [48, 40], [1.2, 1.0], 71, 1.6, 36, 2 * math.pi, 150.0, 300.0, 11)
    filters()


if __name__ == "__main__":
    main()
