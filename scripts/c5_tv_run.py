"""Config c5 end to end on one B200: Shepp-Logan 1024^3 @0.25 mm, 720 views of
2048 x 1536 @0.4 mm over 360 deg; FDK (no Parker, full scan) vs 20 TV-regularised
gradient steps warm-started from the FDK image.  Reports the loss history and the
RMSE against the phantom inside the FOV."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1904_13342_b200 as tg
    dev = torch.device("cuda", 0)
    vol = tg.VolumeSpec.centered([1024] * 3, [0.25] * 3)
    det = tg.Detector2D.centered(2048, 1536, 0.4, 0.4)
    geo = tg.make_cone(vol, det, 720, 2 * math.pi, 750.0, 1200.0)
    ph = tg.shepp_logan_3d(vol, device=dev)
    t0 = time.perf_counter()
    sino = tg.forward_project(ph, geo)
    torch.cuda.synchronize()
    t_fp = time.perf_counter() - t0
    t0 = time.perf_counter()
    fdk = tg.fdk_reconstruct(sino, geo, use_parker=False)
    torch.cuda.synchronize()
    t_fdk = time.perf_counter() - t0

    def rmse(x):
        d = (x.data - ph.data).double()
        return float(torch.sqrt((d * d).mean()))

    iters = int(os.environ.get("ITERS", "20"))
    cfg = tg.ExperimentConfig(learning_rate=float(os.environ.get("LR", "2e-7")), iterations=iters,
                              tv_lambda=0.05)
    t0 = time.perf_counter()
    rec, hist = tg.tv_reconstruct(sino, geo, cfg, init=fdk.data)
    torch.cuda.synchronize()
    t_tv = time.perf_counter() - t0
    print(json.dumps({"workload": "c5 1024^3, 720 x 2048 x 1536, full scan",
                      "fp_s": t_fp, "fdk_s": t_fdk, "fdk_rmse": rmse(fdk),
                      "tv_iterations": iters, "tv_s": t_tv, "tv_s_per_iter": t_tv / iters,
                      "tv_rmse": rmse(rec), "loss_history": hist}), flush=True)


if __name__ == "__main__":
    main()
