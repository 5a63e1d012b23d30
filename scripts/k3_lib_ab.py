"""K3 on the c4 band with whatever libtomograd_b200.so is in place: time
(CUDA events, 5 calls) and save or compare the output.  Used to A/B two
builds of the library: python k3_lib_ab.py save|cmp <file> <label>."""
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
    mode, path, label = sys.argv[1], sys.argv[2], sys.argv[3]
    dev = torch.device("cuda", 0)
    geo = bench.c4_geometry(tg)
    me = D.slab_shards(geo, 1)[0]
    raw = bench.bump_band(torch, bench.C4["views"], me.v0, me.n_rows, bench.C4["nu"], dev)
    g = torch.Generator(device=dev).manual_seed(5)
    raw = raw * (1 + 0.001 * torch.randn(raw.shape, generator=g, device=dev))
    band = tg.fdk_prefilter(raw, geo, True, v0=me.v0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.fdk_prefilter(raw, geo, True, v0=me.v0, out=band)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res = {"label": label, "k3_ms_min": min(ts), "k3_ms": ts}
    if mode == "save":
        torch.save(band.cpu(), path)
    else:
        ref = torch.load(path)
        res["bitwise_vs_saved"] = bool(torch.equal(band.cpu(), ref))
        res["max_abs_diff"] = float((band.cpu() - ref).abs().max())
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
