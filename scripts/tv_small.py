"""The reference's own iterative_tv config (configs/iterative_tv*.json: 128^2,
185 bins, 30 views / 180 deg, lr 1.5e-4, lambda 3, 1200 iterations): device
loop time vs the reference CPU (oracle/_ref, all host threads)."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import numpy as np
    import torch
    import paper_1904_13342_b200 as tg
    import oracle as O
    vol = tg.VolumeSpec.centered([128, 128], [1.0, 1.0])
    geo = tg.make_parallel(vol, tg.Detector1D.centered(185, 1.0), 30, math.pi)
    cfg = tg.ExperimentConfig(noise_relative_std=0.02, learning_rate=1.5e-4, iterations=1200,
                              tv_lambda=3.0)
    ph = tg.shepp_logan_2d(vol, device="cuda:0")
    sino = tg.add_gaussian_noise(tg.forward_project(ph, geo), 0.02, 1337)
    tg.tv_reconstruct(sino, geo, tg.ExperimentConfig(learning_rate=1.5e-4, iterations=5, tv_lambda=3.0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    img, hist = tg.tv_reconstruct(sino, geo, cfg)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    out = {"device_s": dev_s, "iterations": 1200, "device_ms_per_iter": 1e3 * dev_s / 1200,
           "final_loss": hist[-1]}
    if O.ref_available():
        O.Ref.set_threads(os.cpu_count() or 1)
        ov = O.make_volume([128, 128], [1.0, 1.0])
        og = O.Ref.planar_geometry(ov, O.det1_centered(185, 1.0), 30, math.pi)
        p = sino.data.cpu().numpy().astype(np.float64)
        n = 60
        t0 = time.perf_counter()
        _, h = O.Ref.tv_reconstruct_planar(og, p, n, 1.5e-4, 3.0)
        ref_s = (time.perf_counter() - t0) * 1200 / n
        out.update({"reference_cpu_s_est": ref_s, "reference_threads": os.cpu_count(),
                    "reference_sample_iterations": n})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
