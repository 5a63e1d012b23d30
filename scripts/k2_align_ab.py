"""[Experiment record: the TG_K2_ALIGN variant was removed after this
measurement, profiles/r2_k2_align_ab.txt.]
K2 quad kernel: plane-aligned lane schedule (TG_K2_ALIGN=1: 5 CTAs/SM,
2: 4 CTAs/SM, 3: 6 CTAs/SM) against the lock-step kernel (TG_K2_ALIGN=0),
forced k2_impl 0 (quad volume), at c4 (all 496 views) and c5 (views 0-89),
with a bitwise comparison against the lock-step output."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg


def timed(geo, ph, v0, nv, out):
    tg.cone_forward_views(geo, ph, v0, nv, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tg.cone_forward_views(geo, ph, v0, nv, out=out)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def run(cfg, modes):
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
    os.environ["TG_K2_ALIGN"] = "0"
    res["align0_ms"] = [timed(geo, ph, v0, nv, out)]
    ref = out.clone()
    for rep in range(2):
        for m in modes:
            os.environ["TG_K2_ALIGN"] = m
            res.setdefault(f"align{m}_ms", []).append(timed(geo, ph, v0, nv, out))
            res[f"align{m}_bitwise"] = bool(torch.equal(out, ref))
    tg.set_cone_knob(geo, "k2_impl", 1)
    res["slab_ms"] = timed(geo, ph, v0, nv, out)
    res["slab_bitwise"] = bool(torch.equal(out, ref))
    tg.set_cone_knob(geo, "k2_impl", -1)
    os.environ.pop("TG_K2_ALIGN")
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    modes = os.environ.get("MODES", "0,1,2,3").split(",")
    for c in sys.argv[1:] or ["c4", "c5"]:
        run(c, modes)
        torch.cuda.empty_cache()
