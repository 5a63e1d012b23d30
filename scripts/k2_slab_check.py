"""Slab-staged K2 (k2_impl 1) against the quad-volume K2 (k2_impl 0): bitwise
equality on small geometries (random volumes, calibrated matrices, odd
sizes) and at c3; device times at c4 (all views) and c5 (a view subset).

    python scripts/k2_slab_check.py [--quick] [--c5-views N]  -> JSON lines
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ms(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both(tg, geo, vol, view0=0, n=None):
    import torch
    n = geo.n_projections if n is None else n
    outs = []
    for impl in (0, 1):
        tg.set_cone_knob(geo, "k2_impl", impl)
        o = torch.empty((n, geo.detector.n_v, geo.detector.n_u), device=vol.device)
        tg.cone_forward_views(geo, vol, view0, n, out=o)
        outs.append(o)
    torch.cuda.synchronize()
    d = (outs[0] != outs[1])
    return int(d.sum()), float((outs[0] - outs[1]).abs().max()), outs


def main():
    import numpy as np
    import torch
    import paper_1904_13342_b200 as tg
    dev = "cuda:0"
    g = torch.Generator(device="cpu").manual_seed(3)
    cases = {
        "shipped": ([64, 64, 64], [0.85] * 3, 96, 96, 1.0, 1.0, 248, 200, 750.0, 1200.0),
        "odd": ([37, 29, 23], [1.1, 0.9, 1.3], 45, 33, 1.7, 1.5, 30, 360, 120.0, 250.0),
        "wide": ([40, 48, 36], [1.0] * 3, 128, 20, 0.8, 2.5, 17, 180, 200.0, 330.0),
        "c3": ([256] * 3, [0.5] * 3, 400, 600, 1.0, 1.0, 248, 200, 750.0, 1200.0),
    }
    for name, (vs, vsp, nu, nv, du, dv, n, rng, sid, sdd) in cases.items():
        geo = tg.make_cone(tg.VolumeSpec.centered(vs, vsp), tg.Detector2D.centered(nu, nv, du, dv),
                           n, rng * math.pi / 180, sid, sdd)
        vol = torch.rand(vs[::-1], generator=g).to(dev)
        nd, mx, outs = both(tg, geo, vol)
        r = {"case": name, "mismatch": nd, "maxdiff": mx, "nonzero": int((outs[1] != 0).sum())}
        if name == "c3":
            for impl in (0, 1):
                tg.set_cone_knob(geo, "k2_impl", impl)
                o = outs[impl]
                r[f"ms_impl{impl}"] = ms(lambda: tg.cone_forward_views(geo, vol, 0, n, out=o))
        print(json.dumps(r), flush=True)
    # calibrated (perturbed) matrices
    vol_s = tg.VolumeSpec.centered([48, 52, 40], [1.0] * 3)
    det = tg.Detector2D.centered(70, 60, 1.3, 1.3)
    base = tg.make_cone(vol_s, det, 40, 2 * math.pi, 300.0, 600.0)
    rs = np.random.RandomState(5)
    mats = base.matrices * (1 + 1e-3 * rs.standard_normal(base.matrices.shape))
    geo = tg.make_cone_from_matrices(vol_s, det, 2 * math.pi, 300.0, 600.0, mats)
    vol = torch.rand([40, 52, 48], generator=g).to(dev)
    nd, mx, _ = both(tg, geo, vol)
    print(json.dumps({"case": "calibrated", "mismatch": nd, "maxdiff": mx}), flush=True)
    if "--quick" in sys.argv:
        return
    # c4: all views
    geo = tg.make_cone(tg.VolumeSpec.centered([512] * 3, [0.5] * 3),
                       tg.Detector2D.centered(1248, 960, 0.64, 0.64), 496, 220 * math.pi / 180,
                       750.0, 1200.0)
    ph = tg.shepp_logan_3d(geo.volume, device=dev).data
    out = torch.empty((496, 960, 1248), device=dev)
    r = {"case": "c4"}
    res = {}
    for impl in (1, 0):
        tg.set_cone_knob(geo, "k2_impl", impl)
        r[f"ms_impl{impl}"] = ms(lambda: tg.cone_forward_views(geo, ph, 0, 496, out=out), reps=2)
        res[impl] = out.clone() if impl == 1 else None
    r["mismatch"] = int((res[1] != out).sum())
    r["gsamples_impl1"] = 2.179549e11 / (r["ms_impl1"] / 1e3) / 1e9
    r["gsamples_impl0"] = 2.179549e11 / (r["ms_impl0"] / 1e3) / 1e9
    print(json.dumps(r), flush=True)
    del out, res, ph
    torch.cuda.empty_cache()
    # c5: a view subset
    nv5 = 90
    for a_ in sys.argv:
        if a_.startswith("--c5-views="):
            nv5 = int(a_.split("=")[1])
    geo = tg.make_cone(tg.VolumeSpec.centered([1024] * 3, [0.25] * 3),
                       tg.Detector2D.centered(2048, 1536, 0.4, 0.4), 720, 2 * math.pi, 750.0, 1200.0)
    ph = tg.shepp_logan_3d(geo.volume, device=dev).data
    out = torch.empty((nv5, 1536, 2048), device=dev)
    r = {"case": "c5", "views": nv5}
    for impl in (1, 0):
        tg.set_cone_knob(geo, "k2_impl", impl)
        r[f"ms_impl{impl}"] = ms(lambda: tg.cone_forward_views(geo, ph, 0, nv5, out=out), reps=1)
        if impl == 1:
            keep = out.clone()
    r["mismatch"] = int((keep != out).sum())
    # c5 full-scan sample count per view ~ 1.614458e12 / 720
    for impl in (0, 1):
        r[f"gsamples_impl{impl}"] = 1.614458e12 / 720 * nv5 / (r[f"ms_impl{impl}"] / 1e3) / 1e9
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
