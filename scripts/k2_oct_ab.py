"""[Experiment record: the TG_K2_OCT variant was removed after this
measurement, profiles/r2_k2_bank_model.txt.]
K2 quad kernel with the OCT layout (TG_K2_OCT=1: one 32-byte cell of the
8 taps per trilinear cell, one 256-bit gather per sample, FP32x2 lerps)
against the plain quad kernel, forced k2_impl 0, at c4 (all 496 views) and c5
(views 0-89), with a bitwise comparison; the slab kernel on the same views."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg


def run(cfg):
    if cfg == "c4":
        geo = tg.make_cone(tg.VolumeSpec.centered([512] * 3, [0.5] * 3),
                           tg.Detector2D.centered(1248, 960, 0.64, 0.64), 496,
                           220 * math.pi / 180, 750.0, 1200.0)
        v0, nv = 0, 496
    else:
        geo = tg.make_cone(tg.VolumeSpec.centered([1024] * 3, [0.25] * 3),
                           tg.Detector2D.centered(2048, 1536, 0.4, 0.4), 720, 2 * math.pi,
                           750.0, 1200.0)
        v0, nv = 0, 90
    ph = tg.shepp_logan_3d(geo.volume, device="cuda:0").data
    tg.set_cone_knob(geo, "k2_impl", 0)
    out = torch.empty((nv, geo.detector.n_v, geo.detector.n_u), device="cuda:0")
    res = {"cfg": cfg}
    ref = None
    for mix in ("0", "1", "0", "1"):
        os.environ["TG_K2_OCT"] = mix
        tg.cone_forward_views(geo, ph, v0, nv, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.cone_forward_views(geo, ph, v0, nv, out=out)
        b.record()
        torch.cuda.synchronize()
        res.setdefault(f"oct{mix}_ms", []).append(a.elapsed_time(b))
        if ref is None:
            ref = out.clone()
        else:
            res[f"oct{mix}_bitwise"] = bool(torch.equal(out, ref))
    tg.set_cone_knob(geo, "k2_impl", 1)
    tg.cone_forward_views(geo, ph, v0, nv, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tg.cone_forward_views(geo, ph, v0, nv, out=out)
    b.record()
    torch.cuda.synchronize()
    res["slab_ms"] = a.elapsed_time(b)
    res["slab_bitwise"] = bool(torch.equal(out, ref))
    tg.set_cone_knob(geo, "k2_impl", -1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or ["c4", "c5"]:
        run(c)
        torch.cuda.empty_cache()
