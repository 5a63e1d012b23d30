"""Per view-chunk K2 device time, slab (k2_impl 1) vs quad (0), at c4 or c5."""
import math, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
if cfg == "c4":
    geo = tg.make_cone(tg.VolumeSpec.centered([512] * 3, [0.5] * 3),
                       tg.Detector2D.centered(1248, 960, 0.64, 0.64), 496, 220 * math.pi / 180, 750.0, 1200.0)
    chunk = 31
else:
    geo = tg.make_cone(tg.VolumeSpec.centered([1024] * 3, [0.25] * 3),
                       tg.Detector2D.centered(2048, 1536, 0.4, 0.4), 720, 2 * math.pi, 750.0, 1200.0)
    chunk = 45
ph = tg.shepp_logan_3d(geo.volume, device="cuda:0").data
out = torch.empty((chunk, geo.detector.n_v, geo.detector.n_u), device="cuda:0")
res = {}
for impl in (1, 0):
    tg.set_cone_knob(geo, "k2_impl", impl)
    tg.cone_forward_views(geo, ph, 0, chunk, out=out)
    ts = []
    for v0 in range(0, geo.n_projections, chunk):
        n = min(chunk, geo.n_projections - v0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.cone_forward_views(geo, ph, v0, n, out=out[:n])
        b.record()
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 2))
    res[impl] = ts
print(json.dumps({"cfg": cfg, "chunk": chunk, "slab": res[1], "quad": res[0],
                  "angle_deg": [round(v * geo.angular_range / geo.n_projections * 180 / math.pi, 1)
                                for v in range(0, geo.n_projections, chunk)]}))
