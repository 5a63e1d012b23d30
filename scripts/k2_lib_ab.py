"""K2 (forced implementation) at c4 (all views) or c5 (views 0-89) with
whatever libtomograd_b200.so is in place: CUDA-event time of 3 calls and a
saved / compared output, to A/B two builds of the library:
    python k2_lib_ab.py c4|c5 IMPL save|cmp FILE LABEL"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg

cfg, impl, mode, path, label = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
if cfg == "c4":
    geo = tg.make_cone(tg.VolumeSpec.centered([512] * 3, [0.5] * 3),
                       tg.Detector2D.centered(1248, 960, 0.64, 0.64), 496, 220 * math.pi / 180, 750.0, 1200.0)
    v0, nv = 0, 496
else:
    geo = tg.make_cone(tg.VolumeSpec.centered([1024] * 3, [0.25] * 3),
                       tg.Detector2D.centered(2048, 1536, 0.4, 0.4), 720, 2 * math.pi, 750.0, 1200.0)
    v0, nv = 0, 90
tg.set_cone_knob(geo, "k2_impl", impl)
ph = tg.shepp_logan_3d(geo.volume, device="cuda:0").data
out = torch.empty((nv, geo.detector.n_v, geo.detector.n_u), device="cuda:0")
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
res = {"cfg": cfg, "impl": impl, "label": label, "ms": ts}
# a digest instead of the (multi-GB) output: bitwise equal outputs give equal sums
h = out.view(torch.int32).to(torch.int64)
dig = [int(h.sum()), int((h * torch.arange(1, 8, device=h.device).repeat(h.numel() // 7 + 1)[:h.numel()].view_as(h)).sum())]
if mode == "save":
    json.dump(dig, open(path, "w"))
else:
    res["digest_equal"] = dig == json.load(open(path))
print(json.dumps(res), flush=True)
