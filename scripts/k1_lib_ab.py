"""K1 at c4 (circular, or calibrated matrices with 'cal') with whatever
libtomograd_b200.so is in place: CUDA-event time of 10 launches and an output
digest saved / compared, to A/B two builds of the library:
    python k1_lib_ab.py circ|cal save|cmp FILE LABEL"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_1904_13342_b200 as tg

kind, mode, path, label = sys.argv[1:5]
dev = torch.device("cuda", 0)
geo = bench.c4_geometry(tg)
if kind == "cal":
    m = np.asarray(geo.matrices).reshape(-1, 12).copy()
    rng = np.random.default_rng(11)
    m[:, [0, 1, 4, 5]] *= 1.0 + 2e-4 * rng.standard_normal((m.shape[0], 4))
    m[:, 2] += 2e-3 * rng.standard_normal(m.shape[0])
    m[:, 10] += 1e-5 * rng.standard_normal(m.shape[0])
    geo = tg.make_cone_from_matrices(geo.volume, geo.detector, geo.angular_range, geo.sid, geo.sdd, m)
sino = bench.bump_band(torch, 496, 0, 960, 1248, dev)
out = torch.empty((512, 512, 512), dtype=torch.float32, device=dev)
for _ in range(2):
    tg.cone_backproject_slab(geo, sino, 0, 512, 0, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    tg.cone_backproject_slab(geo, sino, 0, 512, 0, out=out)
b.record()
torch.cuda.synchronize()
h = out.view(torch.int32).to(torch.int64)
dig = [int(h.sum()), int((h[::3] * 7 + 1).sum())]
res = {"kind": kind, "label": label, "ms": a.elapsed_time(b) / 10}
if mode == "save":
    json.dump(dig, open(path, "w"))
else:
    res["digest_equal"] = dig == json.load(open(path))
print(json.dumps(res), flush=True)
