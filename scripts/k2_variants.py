"""[Experiment record: the TG_K1_BOXU / TG_K1_LANEMAP / TG_K2_TU / TG_K2_WU /
TG_K2_DUAL knobs were removed from the library once the measurements in
DESIGN.md §5 picked the winners; TG_K1_K remains.]
Time K2 (cone forward projection) at c4 under the current TG_K2_* env (one
variant per process).  --sweep runs each variant in a subprocess."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import torch
    import bench
    import paper_1904_13342_b200 as tg
    dev = torch.device("cuda", 0)
    geo = bench.c4_geometry(tg)
    ph = tg.shepp_logan_3d(geo.volume, device=dev).data
    out = torch.empty((496, 960, 1248), dtype=torch.float32, device=dev)
    tg.cone_forward_views(geo, ph, 0, 496, out=out)
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.cone_forward_views(geo, ph, 0, 496, out=out)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    med = sorted(ms)[1]
    print(json.dumps({"octet": os.environ.get("TG_K2_OCTET", "1"), "ms": med,
                      "gsamples": 217954916998 / (med / 1e3) / 1e9,
                      "checksum": float(out.double().sum()),
                      "abs_checksum": float(out.double().abs().sum())}), flush=True)


def sweep():
    for v in ["0", "1"]:
        subprocess.run([sys.executable, os.path.abspath(__file__)],
                       env=dict(os.environ, TG_K2_OCTET=v), timeout=600)


if __name__ == "__main__":
    sweep() if "--sweep" in sys.argv else one()
