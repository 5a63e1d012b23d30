"""Device time of the 2D operators at BASELINE c1 / c2 through the raw C ABI on
pre-allocated device buffers (no per-call allocation), 50 back-to-back calls
between CUDA events: K7 / K5 forward (pad + march) and K6 / K4 back-projection.
    python scripts/planar_times.py   -> one JSON line"""
import json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1904_13342_b200 as tg
from paper_1904_13342_b200 import _native as N

CFG = {
    "c1": dict(shape=256, sp=1.0, nb=365, db=1.0, n=360, rng=math.pi, sid=0.0, sdd=0.0,
               samples=4.761255e7),
    "c2": dict(shape=512, sp=0.5, nb=1024, db=0.8, n=360, rng=2 * math.pi, sid=750.0, sdd=1200.0,
               samples=1.924493e8),
}


def main():
    L = N.lib()
    out = {}
    st = torch.cuda.current_stream().cuda_stream
    for name, c in CFG.items():
        vol = tg.VolumeSpec.centered([c["shape"]] * 2, [c["sp"]] * 2)
        det = tg.Detector1D.centered(c["nb"], c["db"])
        geo = (tg.make_fan(vol, det, c["n"], c["rng"], c["sid"], c["sdd"]) if c["sdd"] > 0
               else tg.make_parallel(vol, det, c["n"], c["rng"]))
        img = tg.shepp_logan_2d(vol, device="cuda:0").data
        sino = torch.empty((c["n"], c["nb"]), device="cuda:0")
        rec = torch.empty_like(img)
        plan = geo._plan(0)
        fp = lambda: N.check(L.tg_planar_forward(plan, img.data_ptr(), sino.data_ptr(), st))
        bp = lambda: N.check(L.tg_planar_backproject(plan, sino.data_ptr(), rec.data_ptr(), 1.0, 0, st))
        r = {}
        for k, fn in (("fp", fp), ("bp", bp)):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(50):
                fn()
            b.record()
            torch.cuda.synchronize()
            r[k + "_us"] = 1e3 * a.elapsed_time(b) / 50
        r["fp_gsamples_s"] = c["samples"] / (r["fp_us"] * 1e-6) / 1e9
        r["bp_gups"] = c["shape"] ** 2 * c["n"] / (r["bp_us"] * 1e-6) / 1e9
        out[name] = r
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
