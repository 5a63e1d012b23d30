"""Config c2 (fan 512^2, 360 x 1024 @0.8 mm, SID 750 / SDD 1200) forward and
back projection, a few launches each: the command ncu captures for K4 / K5
(and c1's K6 / K7 with --c1)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1904_13342_b200 as tg
    dev = "cuda:0"
    if "--c1" in sys.argv:
        v = tg.VolumeSpec.centered([256, 256], [1.0, 1.0])
        g = tg.make_parallel(v, tg.Detector1D.centered(365, 1.0), 360, math.pi)
    else:
        v = tg.VolumeSpec.centered([512, 512], [0.5, 0.5])
        g = tg.make_fan(v, tg.Detector1D.centered(1024, 0.8), 360, 2 * math.pi, 750.0, 1200.0)
    ph = tg.shepp_logan_2d(v, device=dev)
    for _ in range(3):
        s = tg.forward_project(ph, g)
        tg.back_project(s, g)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
