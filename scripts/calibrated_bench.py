"""K1 / K2 at c4 with calibrated (non-circular) projection matrices — the
general per-voxel path: the circular c4 matrices with a
small detector tilt / skew and out-of-plane terms, normalised by
set_matrices (make_cone_from_matrices)."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import bench
    import paper_1904_13342_b200 as tg
    from paper_1904_13342_b200 import distributed as D
    dev = torch.device("cuda", 0)
    circ = bench.c4_geometry(tg)
    m = np.asarray(circ.matrices).reshape(-1, 12).copy()
    rng = np.random.default_rng(11)
    m[:, [0, 1, 4, 5]] *= 1.0 + 2e-4 * rng.standard_normal((m.shape[0], 4))
    m[:, 2] += 2e-3 * rng.standard_normal(m.shape[0])   # P[0][2] != 0
    m[:, 10] += 1e-5 * rng.standard_normal(m.shape[0])  # P[2][2] != 0
    geo = tg.make_cone_from_matrices(circ.volume, circ.detector, circ.angular_range, circ.sid,
                                     circ.sdd, m)
    assert not geo.circular
    sino = bench.bump_band(torch, 496, 0, 960, 1248, dev)
    out = torch.empty((512, 512, 512), dtype=torch.float32, device=dev)
    def bp():
        tg.cone_backproject_slab(geo, sino, 0, 512, 0, out=out)
    ph = tg.shepp_logan_3d(geo.volume, device=dev).data
    fp_out = torch.empty((496, 960, 1248), dtype=torch.float32, device=dev)
    def fp():
        tg.cone_forward_views(geo, ph, 0, 496, out=fp_out)
    res = {}
    for name, fn, units in (("bp", bp, 512 ** 3 * 496), ("fp", fp, 217954916998)):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        res[name] = {"ms": ms, "rate_g_per_s": units / (ms / 1e3) / 1e9}
    print(json.dumps({"workload": "c4 with calibrated (non-circular) matrices", **res}))


if __name__ == "__main__":
    main()
