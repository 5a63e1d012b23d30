"""BASELINE configs c1-c3 on the device path and on the reference CPU
(oracle/_ref, all host threads): per-operator times at full size.

    python scripts/configs_bench.py [--no-cpu]      -> one JSON line

c1 parallel 256^2, 360 views / pi, 365 bins; c2 fan 512^2, 360 views / 2 pi,
1024 bins @0.8 mm, SID 750 / SDD 1200; c3 cone 256^3 @0.5 mm, 248 views / 200 deg,
[400 x 600] @1 mm, Parker + Ram-Lak FDK."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def dev_ms(fn, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def cpu_s(fn, reps=1):
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def main():
    import numpy as np
    import torch
    import paper_1904_13342_b200 as tg
    import oracle as O
    cpu = "--no-cpu" not in sys.argv and O.ref_available()
    if cpu:
        O.Ref.set_threads(os.cpu_count() or 1)
    out = {"cpu_threads": os.cpu_count() if cpu else None}
    dev = "cuda:0"

    # c1 parallel
    v1 = tg.VolumeSpec.centered([256, 256], [1.0, 1.0])
    g1 = tg.make_parallel(v1, tg.Detector1D.centered(365, 1.0), 360, math.pi)
    ph1 = tg.shepp_logan_2d(v1, device=dev)
    s1 = tg.forward_project(ph1, g1)
    r = {"fp_ms": dev_ms(lambda: tg.forward_project(ph1, g1)),
         "bp_ms": dev_ms(lambda: tg.back_project(s1, g1)),
         "fbp_ms": dev_ms(lambda: tg.fbp_reconstruct(s1, g1))}
    if cpu:
        ov = O.make_volume([256, 256], [1.0, 1.0])
        og = O.Ref.planar_geometry(ov, O.det1_centered(365, 1.0), 360, math.pi)
        img = ph1.data.cpu().numpy()
        sn = s1.data.cpu().numpy()
        r.update({"ref_fp_s": cpu_s(lambda: O.Ref.planar_forward(og, img)),
                  "ref_bp_s": cpu_s(lambda: O.Ref.planar_backproject(og, sn)),
                  "ref_fbp_s": cpu_s(lambda: O.Ref.fbp_reconstruct(og, sn))})
    r["fp_gsamples_s"] = 4.761e7 / (r["fp_ms"] / 1e3) / 1e9
    r["bp_gups"] = 256 * 256 * 360 / (r["bp_ms"] / 1e3) / 1e9
    out["c1_parallel_256"] = r

    # c2 fan
    v2 = tg.VolumeSpec.centered([512, 512], [0.5, 0.5])
    g2 = tg.make_fan(v2, tg.Detector1D.centered(1024, 0.8), 360, 2 * math.pi, 750.0, 1200.0)
    ph2 = tg.shepp_logan_2d(v2, device=dev)
    s2 = tg.forward_project(ph2, g2)
    r = {"fp_ms": dev_ms(lambda: tg.forward_project(ph2, g2)),
         "bp_ms": dev_ms(lambda: tg.back_project(s2, g2))}
    if cpu:
        ov = O.make_volume([512, 512], [0.5, 0.5])
        og = O.Ref.planar_geometry(ov, O.det1_centered(1024, 0.8), 360, 2 * math.pi, 750.0, 1200.0)
        img = ph2.data.cpu().numpy()
        sn = s2.data.cpu().numpy()
        r.update({"ref_fp_s": cpu_s(lambda: O.Ref.planar_forward(og, img)),
                  "ref_bp_s": cpu_s(lambda: O.Ref.planar_backproject(og, sn))})
    r["fp_gsamples_s"] = 1.924e8 / (r["fp_ms"] / 1e3) / 1e9
    r["bp_gups"] = 512 * 512 * 360 / (r["bp_ms"] / 1e3) / 1e9
    out["c2_fan_512"] = r

    # c3 cone FDK short scan
    v3 = tg.VolumeSpec.centered([256] * 3, [0.5] * 3)
    d3 = tg.Detector2D.centered(400, 600, 1.0, 1.0)
    g3 = tg.make_cone(v3, d3, 248, 200 * math.pi / 180, 750.0, 1200.0)
    ph3 = tg.shepp_logan_3d(v3, device=dev)
    s3 = tg.forward_project(ph3, g3)
    r = {"fp_ms": dev_ms(lambda: tg.forward_project(ph3, g3)),
         "bp_ms": dev_ms(lambda: tg.back_project(s3, g3)),
         "fdk_ms": dev_ms(lambda: tg.fdk_reconstruct(s3, g3))}
    r["fp_gsamples_s"] = 5.448906e9 / (r["fp_ms"] / 1e3) / 1e9
    r["bp_gups"] = 4.160750e9 / (r["bp_ms"] / 1e3) / 1e9
    if cpu:
        ov = O.make_volume([256] * 3, [0.5] * 3)
        od = O.det2_centered(400, 600, 1.0, 1.0)
        og = O.Ref.make_cone(ov, od, 248, 200 * math.pi / 180, 750.0, 1200.0)
        sn = s3.data.cpu().numpy()
        r["ref_fdk_s"] = cpu_s(lambda: O.Ref.fdk_reconstruct(og, sn))
        r["ref_bp_s"] = cpu_s(lambda: O.Ref.cone_backproject(og, sn))
    out["c3_cone_fdk_256"] = r
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
