"""One config's K2 forward over a view subset (ncu target / quick timing).
    python scripts/k2_one.py c4|c5 VIEW0 NVIEWS [impl]"""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg
cfg, v0, nv = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
impl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
if cfg == "c4":
    geo = tg.make_cone(tg.VolumeSpec.centered([512] * 3, [0.5] * 3),
                       tg.Detector2D.centered(1248, 960, 0.64, 0.64), 496, 220 * math.pi / 180, 750.0, 1200.0)
else:
    geo = tg.make_cone(tg.VolumeSpec.centered([1024] * 3, [0.25] * 3),
                       tg.Detector2D.centered(2048, 1536, 0.4, 0.4), 720, 2 * math.pi, 750.0, 1200.0)
tg.set_cone_knob(geo, "k2_impl", impl)
ph = tg.shepp_logan_3d(geo.volume, device="cuda:0").data
out = torch.empty((nv, geo.detector.n_v, geo.detector.n_u), device="cuda:0")
for _ in range(2):
    tg.cone_forward_views(geo, ph, v0, nv, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
tg.cone_forward_views(geo, ph, v0, nv, out=out)
b.record()
torch.cuda.synchronize()
print(cfg, v0, nv, impl, "ms", a.elapsed_time(b))
