"""Time the reference's learn-filter experiment (configs/learn_filter.json:
45^2 parallel, 64 bins, 60 views, window 64, noise 0.3, lr 1.5e-5) through the
device graph, next to the reference's own CPU implementation (oracle/_ref,
all host threads, a bounded number of iterations; per-iteration cost scales
linearly).  Prints one JSON line.

    python scripts/learn_filter_bench.py [--iters 5000] [--ref-iters 200]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5000)
    ap.add_argument("--ref-iters", type=int, default=200)
    a = ap.parse_args()
    import torch
    import paper_1904_13342_b200 as tg
    dev = torch.device("cuda", 0)
    vol = tg.VolumeSpec.centered([45, 45], [1.0, 1.0])
    geo = tg.make_parallel(vol, tg.Detector1D.centered(64, 1.0), 60, math.pi)
    cfg = tg.ExperimentConfig(noise_relative_std=0.3, learning_rate=1.5e-5, iterations=20,
                              filter_window=64)
    tg.experiment_learn_filter(geo, cfg, device=dev)  # warm-up (plans, pools)
    cfg.iterations = a.iters
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = tg.experiment_learn_filter(geo, cfg, device=dev)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    out = {"workload": "learn_filter.json (45^2, 64 bins, 60 views, P=64, noise 0.3)",
           "iterations": a.iters, "device_s": dev_s, "device_ms_per_iter": 1e3 * dev_s / a.iters,
           "loss_first": r.loss_history[0], "loss_last": r.loss_history[-1],
           "distance_last": r.distance_history[-1]}
    import oracle as O
    if O.ref_available() and a.ref_iters > 0:
        ov = O.make_volume([45, 45], [1.0, 1.0])
        og = O.Ref.planar_geometry(ov, O.det1_centered(64, 1.0), 60, math.pi)
        O.Ref.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        l, d, w, _ = O.Ref.experiment_learn_filter(og, "shepp-logan", 0.3, 1337, 64, 1.5e-5,
                                                   a.ref_iters)
        ref_s = time.perf_counter() - t0
        n = min(a.ref_iters, a.iters)
        out.update({"reference_iterations": a.ref_iters, "reference_s": ref_s,
                    "reference_ms_per_iter": 1e3 * ref_s / a.ref_iters,
                    "reference_threads": O.Ref.num_threads(),
                    "loss_rel_dev_at_ref_iters": abs(r.loss_history[n] - l[n]) / l[n],
                    "speedup_per_iter": (ref_s / a.ref_iters) / (dev_s / a.iters)})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
