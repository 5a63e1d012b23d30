"""K3 (FDK cosine x Parker pre-weights + Ram-Lak) on the c4 band, CUDA events,
plus a checksum of the output for bitwise A/B of library builds."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_1904_13342_b200 as tg
    from paper_1904_13342_b200 import distributed as D
    dev = torch.device("cuda", 0)
    geo = bench.c4_geometry(tg)
    me = D.slab_shards(geo, 1)[0]
    raw = bench.bump_band(torch, bench.C4["views"], me.v0, me.n_rows, bench.C4["nu"], dev)
    g = torch.Generator(device=dev).manual_seed(5)
    raw = raw * (1 + 0.001 * torch.randn(raw.shape, generator=g, device=dev))
    band = tg.fdk_prefilter(raw, geo, True, v0=me.v0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.fdk_prefilter(raw, geo, True, v0=me.v0, out=band)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"k3_ms_min": min(ts), "k3_ms": ts,
                      "bits": int(band.view(torch.int32).to(torch.int64).sum())}))


if __name__ == "__main__":
    main()
