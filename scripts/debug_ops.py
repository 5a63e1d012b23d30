"""Run each operator once on cuda:0 (debug aid; CUDA_LAUNCH_BLOCKING=1)."""
import math, sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1904_13342_b200 as tg
which = sys.argv[1:] or ["phantom", "pfp", "pbp", "filter", "cfp", "cbp"]
vol3 = tg.VolumeSpec.centered([64, 64, 64], [0.85] * 3)
det = tg.Detector2D.centered(96, 96, 1.0, 1.0)
geo = tg.make_cone(vol3, det, 248, 200 * math.pi / 180, 750.0, 1200.0)
for w in which:
    try:
        if w == "phantom":
            x = tg.shepp_logan_3d(vol3, device="cuda:0"); torch.cuda.synchronize(); print(w, float(x.data.sum()))
        elif w == "pfp":
            v2 = tg.VolumeSpec.centered([64, 64], [1.0, 1.0]); g2 = tg.make_parallel(v2, tg.Detector1D.centered(91, 1.0), 30, math.pi)
            s = tg.forward_project(tg.shepp_logan_2d(v2, device="cuda:0"), g2); torch.cuda.synchronize(); print(w, float(s.data.sum()))
        elif w == "pbp":
            v2 = tg.VolumeSpec.centered([64, 64], [1.0, 1.0]); g2 = tg.make_parallel(v2, tg.Detector1D.centered(91, 1.0), 30, math.pi)
            s = tg.Sinogram.planar(30, g2.detector, data=torch.ones(30, 91, device="cuda:0"))
            x = tg.back_project(s, g2); torch.cuda.synchronize(); print(w, float(x.data.sum()))
        elif w == "filter":
            s = tg.Sinogram.planar(8, tg.Detector1D.centered(100, 1.0), data=torch.rand(8, 100, device="cuda:0"))
            x = tg.apply_filter(s, tg.ramlak_filter(100, 1.0)); torch.cuda.synchronize(); print(w, float(x.data.sum()))
        elif w == "cfp":
            s = tg.forward_project(tg.shepp_logan_3d(vol3, device="cuda:0"), geo); torch.cuda.synchronize(); print(w, float(s.data.sum()))
        elif w == "cbp":
            print("box", geo._plan(0) and None)
            s = tg.Sinogram.cone_beam(248, det, data=torch.ones(248, 96, 96, device="cuda:0"))
            x = tg.back_project(s, geo); torch.cuda.synchronize(); print(w, float(x.data.sum()))
    except Exception as e:
        print(w, "FAILED", type(e).__name__, str(e)[:300]); traceback.print_exc(limit=1)
        break
