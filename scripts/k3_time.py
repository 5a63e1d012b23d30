"""K3 (FDK cosine x Parker pre-weights + Ram-Lak) on the c4 band, CUDA events.
Arguments are values of an environment knob (TG_K3_X2 in the FP32x2
experiment recorded in profiles/r2_k3_variants.txt) set before each timing;
every run's output is compared bitwise with the first run's."""
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
    modes = sys.argv[1:] or ["0", "1", "2", "3", "4"]
    ref = None
    for m in modes:
        os.environ[os.environ.get("KNOB", "TG_K3_X2")] = m
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
        if ref is None:
            ref = band.clone()
        print(json.dumps({"TG_K3_X2": m, "k3_ms_min": min(ts), "k3_ms": ts,
                          "bitwise_vs_first": bool(torch.equal(band, ref)),
                          "max_abs_diff": float((band - ref).abs().max())}), flush=True)


if __name__ == "__main__":
    main()
