import math, sys, torch
sys.path.insert(0, '.')
import paper_1904_13342_b200 as tg
geo = tg.make_cone(tg.VolumeSpec.centered([37, 29, 23], [1.1, 0.9, 1.3]), tg.Detector2D.centered(45, 33, 1.7, 1.5), 3, 2*math.pi, 120.0, 250.0)
vol = torch.rand([23, 29, 37]).cuda()
tg.set_cone_knob(geo, "k2_impl", 1)
o = tg.cone_forward_views(geo, vol, 0, 3)
torch.cuda.synchronize()
print("ok", float(o.sum()))
