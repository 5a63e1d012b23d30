"""[Experiment record: the TG_K1_BOXU / TG_K1_LANEMAP / TG_K2_TU / TG_K2_WU /
TG_K2_DUAL knobs were removed from the library once the measurements in
DESIGN.md §5 picked the winners; TG_K1_K remains.]
K2 time per chunk of views (c4 or c5) under the current TG_K2_* env."""
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
    if os.environ.get("CFG", "c4") == "c5":
        vol = tg.VolumeSpec.centered([1024] * 3, [0.25] * 3)
        det = tg.Detector2D.centered(2048, 1536, 0.4, 0.4)
        geo = tg.make_cone(vol, det, 720, 2 * math.pi, 750.0, 1200.0)
        chunk = 45
    else:
        vol = tg.VolumeSpec.centered([512] * 3, [0.5] * 3)
        det = tg.Detector2D.centered(1248, 960, 0.64, 0.64)
        geo = tg.make_cone(vol, det, 496, 220 * math.pi / 180, 750.0, 1200.0)
        chunk = 31
    ph = tg.shepp_logan_3d(vol, device=dev).data
    out = torch.empty((chunk, det.n_v, det.n_u), dtype=torch.float32, device=dev)
    tg.cone_forward_views(geo, ph, 0, chunk, out=out)
    res = []
    for v0 in range(0, geo.n_projections, chunk):
        n = min(chunk, geo.n_projections - v0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.cone_forward_views(geo, ph, v0, n, out=out)
        b.record()
        torch.cuda.synchronize()
        res.append(round(a.elapsed_time(b), 1))
    print(json.dumps({"cfg": os.environ.get("CFG", "c4"), "dual": os.environ.get("TG_K2_DUAL", "1"),
                      "tu": os.environ.get("TG_K2_TU", "32"), "total": round(sum(res), 1),
                      "per_chunk_ms": res}), flush=True)


if __name__ == "__main__":
    main()
