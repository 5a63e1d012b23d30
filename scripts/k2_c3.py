"""Config c3 cone forward projection (ncu target / quick timing): python scripts/k2_c3.py [impl]"""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg
impl = int(sys.argv[1]) if len(sys.argv) > 1 else -1
geo = tg.make_cone(tg.VolumeSpec.centered([256] * 3, [0.5] * 3), tg.Detector2D.centered(400, 600, 1.0, 1.0),
                   248, 200 * math.pi / 180, 750.0, 1200.0)
tg.set_cone_knob(geo, "k2_impl", impl)
ph = tg.shepp_logan_3d(geo.volume, device="cuda:0").data
out = torch.empty((248, 600, 400), device="cuda:0")
for _ in range(2):
    tg.cone_forward_views(geo, ph, 0, 248, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
tg.cone_forward_views(geo, ph, 0, 248, out=out)
b.record()
torch.cuda.synchronize()
print("c3", impl, "ms", a.elapsed_time(b))
