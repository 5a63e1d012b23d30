"""Slab-staged K2 timing at c4 (views 100-123 near 45 deg, 0-23) and c5
(views 0-44, 90-134), forced k2_impl 1, plus a bitwise check against the
quad kernel on a few views.  One JSON line per config; used for A/B of
library builds (swap the .so between runs)."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg


def geo_of(cfg):
    if cfg == "c4":
        return tg.make_cone(tg.VolumeSpec.centered([512] * 3, [0.5] * 3),
                            tg.Detector2D.centered(1248, 960, 0.64, 0.64), 496,
                            220 * math.pi / 180, 750.0, 1200.0), [(100, 24), (0, 24)]
    return tg.make_cone(tg.VolumeSpec.centered([1024] * 3, [0.25] * 3),
                        tg.Detector2D.centered(2048, 1536, 0.4, 0.4), 720, 2 * math.pi,
                        750.0, 1200.0), [(0, 45), (90, 45)]


def main():
    for cfg in sys.argv[1:] or ["c4", "c5"]:
        geo, blocks = geo_of(cfg)
        ph = tg.shepp_logan_3d(geo.volume, device="cuda:0").data
        res = {"cfg": cfg}
        for v0, nv in blocks:
            out = torch.empty((nv, geo.detector.n_v, geo.detector.n_u), device="cuda:0")
            tg.set_cone_knob(geo, "k2_impl", 1)
            tg.cone_forward_views(geo, ph, v0, nv, out=out)
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                tg.cone_forward_views(geo, ph, v0, nv, out=out)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[f"v{v0}_ms"] = min(ts)
            sl = out[:4].clone()
            tg.set_cone_knob(geo, "k2_impl", 0)
            q = torch.empty_like(sl)
            tg.cone_forward_views(geo, ph, v0, 4, out=q)
            torch.cuda.synchronize()
            res[f"v{v0}_bitwise"] = bool(torch.equal(sl, q))
            del out
        tg.set_cone_knob(geo, "k2_impl", -1)
        print(json.dumps(res), flush=True)
        del ph
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
