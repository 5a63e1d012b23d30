"""Time the c4 host-buffer back-projection (tg_cone_backproject_slab_host, the
bench's e2e leg) under the TG_E2E_* schedule knobs of csrc/cone.cu
phased_backproject (one variant per process).  Prints one JSON line each.

    python scripts/e2e_variants.py --sweep
"""
import json
import os
import subprocess
import sys
import time

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
    band = bench.bump_band(torch, bench.C4["views"], me.v0, me.n_rows, bench.C4["nu"], dev)
    h_band = torch.empty(band.shape, dtype=torch.float32, pin_memory=True)
    h_band.copy_(band.cpu())
    h_slab = torch.empty((me.nz, 512, 512), dtype=torch.float32, pin_memory=True)
    L = tg._native.lib()
    plan = geo._plan(0)
    if os.environ.get("E2E_FDK"):
        # the FDK from a full host sinogram (tg_cone_fdk_host, bench.py's fdk_e2e leg)
        h_sino = torch.zeros((bench.C4["views"], bench.C4["nv"], bench.C4["nu"]), dtype=torch.float32,
                             pin_memory=True)
        h_sino[:, me.v0:me.v0 + me.n_rows].copy_(band.cpu())
        h_vol = torch.empty((512, 512, 512), dtype=torch.float32, pin_memory=True)

        def step():
            tg._native.check(L.tg_cone_fdk_host(plan, h_sino.data_ptr(), h_vol.data_ptr(), 1))
    else:
        def step():
            tg._native.check(L.tg_cone_backproject_slab_host(plan, me.z0, me.nz, me.v0, me.n_rows,
                                                             h_band.data_ptr(), h_slab.data_ptr(), 0, 1))
    for _ in range(2):
        step()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * sorted(ts)[len(ts) // 2]
    print(json.dumps({k: os.environ.get(k, "default") for k in
                      ("TG_E2E_CENTRE_UNITS", "TG_E2E_RINGS", "TG_E2E_CHUNKS", "TG_E2E_GROUP",
                               "TG_E2E_NOPDL", "E2E_FDK", "TG_E2E_CHUNKS_LATE", "TG_E2E_LATE_FROM")} |
                     {"h2d_bytes": int(L.tg_cone_last_h2d_bytes(plan))} |
                     {"ms_med": ms, "ms_min": 1e3 * min(ts),
                      "gups": 512 ** 3 * 496 / (ms / 1e3) / 1e9}), flush=True)


def sweep():
    # round-1 sweep: centre {1,2,4} x rings {2,4,6,8} x chunks {4,8,16} -> 2/4/4 best
    # (45.9 ms vs 47.0 at 8 chunks, 50-55 ms at 16); then chunks {2,3,4} x rings {3,4,5}
    # footprint uploads (1.41 GB instead of 2.09): K1 rather than PCIe bounds the
    # pipeline, so re-sweep toward fewer phases / chunks and the copy group size
    # programmatic dependent launch between the chunked K1 launches: on / off,
    # and with it more chunks (whose launch tails PDL now hides)
    # (measured: 2/2/4 43.3 ms with PDL, 44.2 without; 8 chunks 45.7; 2/4/4 43.7;
    # 2/3/6 44.8; 1/2/4 44.8 — profiles/r1_e2e_pdl_sweep.jsonl)
    # round 2 (K1 36.5 ms after the 4-view producer): re-sweep around 2/2/4
    grid = [("2", "2", "4", "8", "pdl"), ("1", "2", "4", "8", "pdl"), ("2", "2", "3", "8", "pdl"),
            ("2", "2", "6", "8", "pdl"), ("2", "3", "4", "8", "pdl"), ("1", "3", "4", "8", "pdl"),
            ("2", "2", "4", "4", "pdl"), ("2", "2", "4", "16", "pdl"), ("1", "2", "3", "8", "pdl")]
    # measured: 2/2/4/8 40.92, 2/3/4/8 40.33, 2/2/4/16 40.64, 1/3/4/8 40.99, 2/2/3/8 41.25,
    # 2/2/6/8 42.76 ms (profiles/r2_e2e_sweep.jsonl)
    if "--fdk" in sys.argv:
        os.environ["E2E_FDK"] = "1"
        grid = [(c, r, ch, "8", "pdl") for c in ("1", "2") for r in ("2", "3", "4")
                for ch in ("3", "4", "6")]
        # measured (profiles/r2_e2e_fdk_sweep.jsonl): 1/4/3 46.05 ms, 2/3/4 46.46, 2/2/4 47.54
        if "--fdk2" in sys.argv:
            grid = [("1", r, ch, g, "pdl") for r, ch, g in (("4", "3", "8"), ("5", "3", "8"),
                    ("6", "3", "8"), ("5", "2", "8"), ("4", "2", "8"), ("5", "3", "16"),
                    ("8", "3", "8"), ("6", "2", "8"))]
    if "--grid2" in sys.argv:
        grid = [("2", "3", "4", "8", "pdl"), ("2", "3", "4", "16", "pdl"), ("2", "4", "4", "8", "pdl"),
                ("2", "4", "4", "16", "pdl"), ("3", "3", "4", "8", "pdl"), ("2", "3", "5", "8", "pdl"),
                ("2", "3", "4", "12", "pdl"), ("2", "5", "4", "8", "pdl")]
    if "--late" in sys.argv:
        # BP: fewer view chunks from the third phase on (TG_E2E_CHUNKS_LATE)
        grid = [("2", "3", "4", "8", "pdl"), ("2", "3", "4", "8", "late2"), ("2", "3", "4", "8", "late1"),
                ("2", "3", "4", "8", "late3"), ("2", "4", "4", "8", "late2"), ("2", "2", "4", "8", "late2"),
                ("2", "3", "6", "8", "late2"), ("2", "3", "4", "8", "pdl")]
    if "--late2" in sys.argv:
        grid = [("2", "3", "4", "8", "late2from1"), ("2", "3", "4", "8", "late2from2"),
                ("2", "3", "4", "8", "late2from3"), ("2", "4", "4", "8", "late2from1"),
                ("2", "4", "4", "8", "late1from3"), ("2", "3", "5", "8", "late2from1"),
                ("1", "3", "4", "8", "late2from1"), ("2", "3", "4", "8", "late2from2")]
    if "--fdklate" in sys.argv:
        os.environ["E2E_FDK"] = "1"
        grid = [("1", "5", "3", "8", "pdl"), ("1", "5", "3", "8", "late2from2"),
                ("1", "5", "3", "8", "late1from2"), ("1", "5", "3", "8", "late1from3"),
                ("1", "5", "4", "8", "late2from2"), ("1", "5", "4", "8", "late1from2"),
                ("1", "4", "3", "8", "late1from2"), ("1", "5", "3", "8", "pdl")]
    if "--grid1" in sys.argv:
        grid = [("2", "2", "4", "8", "pdl"), ("2", "2", "4", "8", "nopdl")]
    for c, r, ch, g, mode in grid:
        env = dict(os.environ, TG_E2E_CENTRE_UNITS=c, TG_E2E_RINGS=r, TG_E2E_CHUNKS=ch,
                   TG_E2E_GROUP=g)
        if mode == "nopdl":
            env["TG_E2E_NOPDL"] = "1"
        if mode.startswith("late"):
            late, _, frm = mode[4:].partition("from")
            env["TG_E2E_CHUNKS_LATE"] = late
            if frm:
                env["TG_E2E_LATE_FROM"] = frm
        subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, timeout=300)


if __name__ == "__main__":
    sweep() if "--sweep" in sys.argv else one()
