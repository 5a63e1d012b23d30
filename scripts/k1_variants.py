"""[Experiment record: the TG_K1_BOXU / TG_K1_LANEMAP / TG_K2_TU / TG_K2_WU /
TG_K2_DUAL knobs were removed from the library once the measurements in
DESIGN.md §5 picked the winners; TG_K1_K remains.]
Time K1 at c4 under the current TG_K1_* environment (one variant per
process; the plan reads the knobs at creation).  Prints one JSON line.

    TG_K1_BOXU=52 TG_K1_LANEMAP=1 python scripts/k1_variants.py
    python scripts/k1_variants.py --sweep      # every variant, one subprocess each
"""
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
    from paper_1904_13342_b200 import distributed as D
    dev = torch.device("cuda", 0)
    geo = bench.c4_geometry(tg)
    me = D.slab_shards(geo, 1)[0]
    raw = bench.bump_band(torch, bench.C4["views"], me.v0, me.n_rows, bench.C4["nu"], dev)
    band = tg.fdk_prefilter(raw, geo, True, v0=me.v0)
    slab = torch.empty((me.nz, 512, 512), dtype=torch.float32, device=dev)
    ref = None
    for _ in range(3):
        tg.cone_backproject_slab(geo, band, me.z0, me.nz, me.v0, out=slab, scale=1.0)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(8)]
    for a, b in evs:
        a.record()
        tg.cone_backproject_slab(geo, band, me.z0, me.nz, me.v0, out=slab, scale=1.0)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)
    med = ms[len(ms) // 2]
    plan = geo._plan(0)
    print(json.dumps({"boxu": os.environ.get("TG_K1_BOXU", "auto"),
                      "lanemap": os.environ.get("TG_K1_LANEMAP", "0"),
                      "k": os.environ.get("TG_K1_K", "32"),
                      "ms_med": med, "ms_min": ms[0],
                      "gups": 512 ** 3 * 496 / (med / 1e3) / 1e9,
                      "checksum": float(slab.double().sum())}), flush=True)


def sweep():
    for boxu in ["48", "44", "52", "56"]:
        for lm in ["0", "1", "2"]:
            env = dict(os.environ, TG_K1_BOXU=boxu, TG_K1_LANEMAP=lm)
            subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, timeout=300)


if __name__ == "__main__":
    sweep() if "--sweep" in sys.argv else one()
