"""[Experiment record: the TG_K1_BOXU / TG_K1_LANEMAP / TG_K2_TU / TG_K2_WU /
TG_K2_DUAL knobs were removed from the library once the measurements in
DESIGN.md §5 picked the winners; TG_K1_K remains.]
Time K2 at config c5 (1024^3, 720 x [2048 x 1536]) under the current TG_K2_* env."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1904_13342_b200 as tg
    dev = torch.device("cuda", 0)
    vol = tg.VolumeSpec.centered([1024] * 3, [0.25] * 3)
    det = tg.Detector2D.centered(2048, 1536, 0.4, 0.4)
    geo = tg.make_cone(vol, det, 720, 2 * math.pi, 750.0, 1200.0)
    ph = tg.shepp_logan_3d(vol, device=dev).data
    nviews = int(os.environ.get("NV", "90"))
    out = torch.empty((nviews, 1536, 2048), dtype=torch.float32, device=dev)
    tg.cone_forward_views(geo, ph, 0, nviews, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tg.cone_forward_views(geo, ph, 0, nviews, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    samples = 1.614458e12 * nviews / 720  # approx (views are statistically alike)
    print(json.dumps({"tu": os.environ.get("TG_K2_TU", "32"), "views": nviews, "ms": ms,
                      "gsamples_approx": samples / (ms / 1e3) / 1e9,
                      "checksum": float(out.double().sum())}), flush=True)


if __name__ == "__main__":
    main()
