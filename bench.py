#!/usr/bin/env python
"""Benchmark of the B200 projector path on BASELINE config c4 (SURVEY
Appendix A): 512^3 volume @0.5 mm, 496 projections of [1248 x 960] @0.64 mm
over 220 deg, SID 750 / SDD 1200, FDK short scan (Parker + Ram-Lak, P = 4096).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one K1 cone back-projection (projector.hpp:283-313) of the
FDK-filtered projections of this rank's z-slab: the headline metric is BP
GUPS = voxel-updates / s over the whole job.  Under torchrun each rank owns a
32-aligned z-slab and only the detector row band it projects onto (no
data-path collective: SURVEY §8e); per-GPU work shrinks with N, so scaling is
"strong".  Also reported: the forward projector K2 (Gsamples/s, exact
per-ray sample counts of the reference's clip + ceil rule), the K3 row
filter, the end-to-end host-buffer call (pinned H2D + K1 + D2H through the C
ABI), the roofline of K1 against the interpolation-rate bound, NVML clocks
during the timed region, and the reference CPU implementation (oracle/_ref,
the reference's own headers compiled here) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Cone-beam backproj GUPS & forward-proj Gsamples/s at 512³; 1/2/4/8 B200"
UNIT = "GUPS"
C4 = dict(n=512, spacing=0.5, nu=1248, nv=960, det=0.64, views=496, range_deg=220.0, sid=750.0,
          sdd=1200.0)
CONFIG_NAME = ("c4: cone_backprojection3d FDK, 512^3 @0.5mm, 496 x [1248 x 960] @0.64mm, 220 deg, "
               "SID 750 / SDD 1200 (RabbitCT scale)")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): NVML every 10 ms on a thread, falling
    back to `nvidia-smi -lms 200` when pynvml is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.nvml = None
        self.p = None
        self.f = None

    def _poll(self):
        import pynvml as N
        h = N.nvmlDeviceGetHandleByIndex(self.gpu)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        while not self._stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), [n for n, b in bits.items() if r & b]))
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        import threading
        try:
            import pynvml as N
            N.nvmlInit()
            self.nvml = N
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        except Exception:
            self.nvml = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
            return
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        if self.nvml is None:
            if self.p is None:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
            self.f.flush()
            with open(self.f.name) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                        rs = [n for n, v in zip(self.NAMES, parts[5:9]) if v.lower() == "active"]
                        self.rows.append((float(parts[1]), float(parts[2]), rs))
            os.unlink(self.f.name)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({n for r in self.rows for n in r[2]}),
                "samples": len(self.rows), "source": "nvml 10 ms" if self.nvml else "nvidia-smi"}


def c4_geometry(tg):
    vol = tg.VolumeSpec.centered([C4["n"]] * 3, [C4["spacing"]] * 3)
    det = tg.Detector2D.centered(C4["nu"], C4["nv"], C4["det"], C4["det"])
    return tg.make_cone(vol, det, C4["views"], C4["range_deg"] * math.pi / 180.0, C4["sid"],
                        C4["sdd"])


def bump_band(torch, n_views, v0, n_rows, nu, device):
    """SURVEY Appendix A synthetic projections: max(0, 1-x^2-y^2)(1+0.1 sin(0.01 i)),
    x = (u - 623.5)/400, y = (v - 479.5)/300, for detector rows [v0, v0+n_rows)."""
    u = torch.arange(nu, device=device, dtype=torch.float64)
    v = torch.arange(v0, v0 + n_rows, device=device, dtype=torch.float64)
    i = torch.arange(n_views, device=device, dtype=torch.float64)
    x = (u - 623.5) / 400.0
    y = (v - 479.5) / 300.0
    base = torch.clamp(1.0 - x[None, :] ** 2 - y[:, None] ** 2, min=0.0)
    return (base[None] * (1.0 + 0.1 * torch.sin(0.01 * i))[:, None, None]).float().contiguous()


def _c4_ref_slab_geometry(O, z0, nz, from_matrices=None):
    """The reference's own ConeGeometry for z-slices [z0, z0+nz) of c4, built by
    the reference itself (oracle/_ref: make_cone, geometry.hpp:206-223, on a
    VolumeSpec whose origin is shifted to the slab; P maps world coordinates,
    so the matrices equal the full volume's).  With from_matrices (the GPU
    arm's host geometry, bitwise equal, tests/test_host_geometry.py) the
    reference re-normalises those instead (make_cone_from_matrices)."""
    spacing = C4["spacing"]
    origin = [-0.5 * (C4["n"] - 1) * spacing] * 3
    origin[2] = origin[2] + z0 * spacing
    ov = O.make_volume([C4["n"], C4["n"], nz], [spacing] * 3, origin)
    od = O.or_det2(C4["nu"], C4["nv"], C4["det"], C4["det"], -0.5 * (C4["nu"] - 1) * C4["det"],
                   -0.5 * (C4["nv"] - 1) * C4["det"])
    rng = C4["range_deg"] * math.pi / 180.0
    if O.ref_available():
        if from_matrices is not None:
            return O.Ref.cone_from_matrices(ov, od, rng, C4["sid"], C4["sdd"], from_matrices), "reference"
        return O.Ref.make_cone(ov, od, C4["views"], rng, C4["sid"], C4["sdd"]), "reference"
    return O.make_cone(ov, od, C4["views"], rng, C4["sid"], C4["sdd"]), "port"


def cpu_reference_sample(sino_np, z0, nz, threads, matrices=None):
    """The reference's own back_project (projector.hpp:283-313, compiled from
    its headers into oracle/_ref) on slices [z0, z0+nz) of the c4 volume with
    all views: a bounded sample of the same workload."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O
    g, kind = _c4_ref_slab_geometry(O, z0, nz, matrices)
    if kind == "reference":
        O.Ref.set_threads(threads)
        fn = O.Ref.cone_backproject
    else:
        O.set_threads(threads)
        fn = O.cone_backproject
    t0 = time.perf_counter()
    out = fn(g, np.ascontiguousarray(sino_np))
    dt = time.perf_counter() - t0
    updates = C4["n"] * C4["n"] * nz * C4["views"]
    return updates / dt / 1e9, kind, dt, out


def bench_config(world):
    """`config` of both arms' JSON lines (identical by construction)."""
    return {"workload": CONFIG_NAME, "parallelism": f"z-slab x{world}",
            "l2": "inputs larger than L2 (2.38 GB sino, 512 MB volume)"}


def run_reference(args):
    """--impl reference: the reference's CPU back-projection (oracle/_ref, its
    own headers compiled by oracle/Makefile) on the host cores, each step a
    bounded z-slab of the c4 workload.  Nothing from this repository's package
    (no paper_1904_13342_b200, no torch) is imported on this path: geometry,
    inputs and the timed call are the reference's own or numpy."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import numpy as np
    nz = 8
    z0 = C4["n"] // 2 - nz // 2
    # host-side synthetic filtered projections of the same bump (numpy, no GPU)
    u = np.arange(C4["nu"]); v = np.arange(C4["nv"]); i = np.arange(C4["views"])
    base = np.clip(1 - ((u[None, :] - 623.5) / 400) ** 2 - ((v[:, None] - 479.5) / 300) ** 2, 0, None)
    sino = (base[None] * (1 + 0.1 * np.sin(0.01 * i))[:, None, None]).astype(np.float32)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_sample(sino, z0, nz, threads)
    ts = []
    kind = "reference"
    for _ in range(args.steps):
        _, kind, dt, _ = cpu_reference_sample(sino, z0, nz, threads)
        ts.append(dt)
    value = C4["n"] * C4["n"] * nz * C4["views"] * len(ts) / sum(ts) / 1e9
    sample = f"z-slices [{z0},{z0 + nz}) of 512 x all 496 views per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(ts) / len(ts),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY App. A separable bump)",
        "config": bench_config(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_profile_traffic():
    p = os.path.join(ROOT, "profiles", "k1_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fdk-e2e", action="store_true",
                    help="skip the FDK-from-host-sinogram leg (tg_cone_fdk_host)")
    ap.add_argument("--no-calibrated", action="store_true",
                    help="skip the calibrated-matrix (general K1 path) leg")
    ap.add_argument("--fp-steps", type=int, default=3)
    ap.add_argument("--c5-iters", type=int, default=2,
                    help="TV-loop iterations timed at config c5 (0 = skip the c5 leg)")
    args = ap.parse_args()
    if args.impl == "ours" and args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 untimed warm-up steps (the line reports the value used)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1904_13342_b200 as tg
    from paper_1904_13342_b200 import distributed as D

    rank, world, local = env_rank()
    n_dev = torch.cuda.device_count()
    gpu = local % n_dev
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    # one process per GPU over NCCL; more ranks than GPUs (a launcher smoke
    # test on a single-GPU box) falls back to gloo for the control plane only
    # (the data path has no collective)
    backend = "nccl" if world <= n_dev else "gloo"
    if world > 1:
        # NCCL's init log (transport, NVLS / ring choice) goes to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    L = tg._native.lib()
    geo = c4_geometry(tg)
    shards = D.slab_shards(geo, world)
    me = shards[rank]
    views = D.view_partition(geo, world)
    vw0, vwn = views[rank]
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs (resident in HBM) --------------------------------------
    raw_band = bump_band(torch, C4["views"], me.v0, me.n_rows, C4["nu"], dev)
    band = tg.fdk_prefilter(raw_band, geo, True, v0=me.v0)        # K3 (warm + input)
    slab = torch.empty((me.nz, C4["n"], C4["n"]), dtype=torch.float32, device=dev)
    scale = tg.fdk_scale(geo, True)
    torch.cuda.synchronize()

    def k1():
        tg.cone_backproject_slab(geo, band, me.z0, me.nz, me.v0, out=slab, scale=scale)

    # ---- K1 timed region --------------------------------------------------
    for _ in range(args.warmup):
        k1()
    torch.cuda.synchronize()
    barrier()
    launches0 = int(L.tg_kernel_launch_count())
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(gpu) as clk:
        torch.cuda.synchronize()
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for a, b in evs:
            a.record(stream)
            k1()
            b.record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        barrier()
    gpu_launches = int(L.tg_kernel_launch_count()) - launches0
    total_ms = max_over_ranks(t_start.elapsed_time(t_end))
    k1_ms = [a.elapsed_time(b) for a, b in evs]
    updates_total = C4["n"] ** 2 * C4["n"] * C4["views"]  # whole job per step
    value = updates_total * args.steps / (total_ms / 1e3) / 1e9
    my_updates = C4["n"] ** 2 * me.nz * C4["views"]
    k1_avg = statistics.mean(k1_ms)
    per_gpu_gups = my_updates / (k1_avg / 1e3) / 1e9
    clocks = clk.summary()

    # ---- K3 (FDK pre-filter of this rank's band) --------------------------
    k3_ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    k3_ev[0].record(stream)
    for _ in range(3):
        tg.fdk_prefilter(raw_band, geo, True, v0=me.v0, out=band)
    k3_ev[1].record(stream)
    torch.cuda.synchronize()
    k3_ms = k3_ev[0].elapsed_time(k3_ev[1]) / 3

    # ---- K2 forward projection (angle shard) ------------------------------
    phantom = tg.shepp_logan_3d(geo.volume, device=dev).data
    part = torch.empty((vwn, C4["nv"], C4["nu"]), dtype=torch.float32, device=dev)
    tg.cone_forward_views(geo, phantom, vw0, vwn, out=part)  # warm
    torch.cuda.synchronize()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.fp_steps):
        tg.cone_forward_views(geo, phantom, vw0, vwn, out=part)
    f1.record(stream)
    torch.cuda.synchronize()
    fp_ms = max_over_ranks(f0.elapsed_time(f1) / args.fp_steps)
    fp_samples = samples_c4(geo)
    fp_value = fp_samples / (fp_ms / 1e3) / 1e9
    del phantom

    # ---- end to end through the C ABI with host buffers ---------------------
    h_band = torch.empty(band.shape, dtype=torch.float32, pin_memory=True)
    h_band.copy_(band.cpu())
    h_slab = torch.empty(slab.shape, dtype=torch.float32, pin_memory=True)
    plan = geo._plan(gpu)

    def e2e_step():
        tg._native.check(L.tg_cone_backproject_slab_host(plan, me.z0, me.nz, me.v0, me.n_rows,
                                                         h_band.data_ptr(), h_slab.data_ptr(),
                                                         0, 1))
        return float(h_slab[0, 0, 0])  # host read of the result

    # warm-up: the first host-buffer calls on a fresh box pay one-time costs
    # (pinned-page mappings, staging allocation) that are not the pipeline's
    for _ in range(max(2, args.warmup)):
        e2e_step()
    barrier()
    e2e_n = max(1, min(args.steps, 10))
    e2e_steps_ms = []
    t0 = time.perf_counter()
    for _ in range(e2e_n):
        t1 = time.perf_counter()
        e2e_step()
        e2e_steps_ms.append(1e3 * (time.perf_counter() - t1))
    e2e_own_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_own_s)
    e2e_value = updates_total * e2e_n / e2e_s / 1e9
    # the host call back-projects with scale 1; the timed K1 carried the FDK constant
    # bytes actually shipped host -> device per step (each view's own footprint)
    e2e_h2d = int(L.tg_cone_last_h2d_bytes(plan)) * world
    e2e_band_bytes = int(h_band.numel() * 4) * world
    e2e_d2h = int(h_slab.numel() * 4) * world
    e2e_parity = float((h_slab.to(dev) * scale - slab).abs().max() / slab.abs().max().clamp_min(1e-30))
    # PCIe copy rates on this box (pinned, one DMA each) to explain e2e
    def copy_ms(dst, src):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dst.copy_(src, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b)
    h2d_ms = copy_ms(band, h_band)
    d2h_ms = copy_ms(h_slab, slab)
    pcie = {"h2d_gbs": h_band.numel() * 4 / (h2d_ms / 1e3) / 1e9, "h2d_ms": h2d_ms,
            "d2h_gbs": h_slab.numel() * 4 / (d2h_ms / 1e3) / 1e9, "d2h_ms": d2h_ms}

    # ---- per-rank description (N > 1: every rank's shard and times) ---------
    rank_info = {"rank": rank, "gpu": gpu, "z0": me.z0, "nz": me.nz, "rows": [me.v0, me.n_rows],
                 "views": [vw0, vwn], "k1_ms": round(k1_avg, 3),
                 "k1_gups": round(per_gpu_gups, 1), "fp_ms": round(f0.elapsed_time(f1) / args.fp_steps, 3),
                 "e2e_ms": round(1e3 * e2e_own_s / e2e_n, 3), "h2d_bytes": e2e_h2d // world,
                 "pcie_h2d_ms": round(h2d_ms, 3), "pcie_h2d_gbs": round(pcie["h2d_gbs"], 1)}
    ranks = [rank_info]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, rank_info)

    # ---- FDK end to end from a full host sinogram (the C++ drop-in's path) ----
    # tg_cone_fdk_host: raw projections [496][960][1248] in pinned host memory ->
    # volume in pinned host memory; only the volume's detector rows travel and
    # are weighted / filtered (K3) before K1.  Rows outside the band are zero.
    fdk_e2e = None
    if world == 1 and not args.no_fdk_e2e:
        h_sino = torch.zeros((C4["views"], C4["nv"], C4["nu"]), dtype=torch.float32,
                             pin_memory=True)
        h_sino[:, me.v0:me.v0 + me.n_rows].copy_(raw_band.cpu())
        h_vol = torch.empty((C4["n"],) * 3, dtype=torch.float32, pin_memory=True)

        def fdk_step():
            tg._native.check(L.tg_cone_fdk_host(plan, h_sino.data_ptr(), h_vol.data_ptr(), 1))
            return float(h_vol[0, 0, 0])

        for _ in range(3):  # warm-up (fresh pinned buffers, staging allocation)
            fdk_step()
        n_fdk = 6
        fdk_steps_ms = []
        t0 = time.perf_counter()
        for _ in range(n_fdk):
            t1 = time.perf_counter()
            fdk_step()
            fdk_steps_ms.append(1e3 * (time.perf_counter() - t1))
        fdk_s = (time.perf_counter() - t0) / n_fdk
        fdk_parity = float((h_vol.to(dev) - slab).abs().max() / slab.abs().max().clamp_min(1e-30))
        fdk_e2e = {"value": updates_total / fdk_s / 1e9, "unit": UNIT, "ms_per_step": 1e3 * fdk_s,
                   "step_ms": fdk_steps_ms,
                   "h2d_bytes_per_step": int(L.tg_cone_last_h2d_bytes(plan)),
                   "d2h_bytes_per_step": int(h_vol.numel() * 4),
                   "host_sinogram_bytes": int(h_sino.numel() * 4),
                   "path": "tg_cone_fdk_host (pinned raw projections -> cosine x Parker + Ram-Lak "
                           "(K3) -> K1 -> pinned volume; view chunks overlapped)",
                   "max_rel_diff_vs_device": fdk_parity}
        del h_sino, h_vol

    # ---- K1 with calibrated (non-circular) matrices: the general path ----------
    # (scanners with measured projection matrices).  The c4
    # matrices with a small detector tilt / skew and out-of-plane terms,
    # normalised by set_matrices; device-resident full detector, CUDA events.
    k1_cal = None
    if world == 1 and not args.no_calibrated:
        import numpy as np
        m = np.asarray(geo.matrices).reshape(-1, 12).copy()
        rng = np.random.default_rng(11)
        m[:, [0, 1, 4, 5]] *= 1.0 + 2e-4 * rng.standard_normal((m.shape[0], 4))
        m[:, 2] += 2e-3 * rng.standard_normal(m.shape[0])   # P[0][2] != 0
        m[:, 10] += 1e-5 * rng.standard_normal(m.shape[0])  # P[2][2] != 0
        cgeo = tg.make_cone_from_matrices(geo.volume, geo.detector, geo.angular_range, geo.sid,
                                          geo.sdd, m)
        csino = bump_band(torch, C4["views"], 0, C4["nv"], C4["nu"], dev)
        cvol = torch.empty((C4["n"],) * 3, dtype=torch.float32, device=dev)
        for _ in range(2):
            tg.cone_backproject_slab(cgeo, csino, 0, C4["n"], 0, out=cvol)
        torch.cuda.synchronize()
        ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_cal = 4
        ca.record()
        for _ in range(n_cal):
            tg.cone_backproject_slab(cgeo, csino, 0, C4["n"], 0, out=cvol)
        cb.record()
        torch.cuda.synchronize()
        cal_ms = ca.elapsed_time(cb) / n_cal
        k1_cal = {"value": C4["n"] ** 3 * C4["views"] / (cal_ms / 1e3) / 1e9, "unit": UNIT,
                  "ms": cal_ms, "circular": bool(cgeo.circular),
                  "workload": "c4 volume / detector / views with perturbed (calibrated) projection "
                              "matrices: general per-voxel K1 path"}
        del csino, cvol, cgeo

    # ---- roofline (K1) --------------------------------------------------------
    pk = peaks()
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    interp_peak = n_sm * 4 * sm_max * 1e6 / 1e9  # bilinear/s -> GUPS
    l1_peak = n_sm * 128 / 16 * sm_max * 1e6 / 1e9
    traffic = load_profile_traffic()
    hbm_bytes = 4 * (C4["n"] ** 2 * me.nz + C4["views"] * me.n_rows * C4["nu"])
    roofline = {
        # the resource K1 actually saturates: the SM's L1 / shared-memory data
        # path (128 B/clk/SM; ncu l1tex__data_pipe_lsu_wavefronts), and each
        # voxel-update gathers 4 fp32 taps = 16 B from the staged box
        "bound": "l1",
        "achieved": per_gpu_gups, "peak": l1_peak, "unit": "GUPS",
        "frac": per_gpu_gups / l1_peak,
        "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
        "note": ("K1 is bound by the on-chip L1/shared data path, not HBM or tensor cores (no "
                 "dense contraction): peak = n_SM x 128 B/clk / 16 B per update x sm_max_mhz; "
                 f"HBM compulsory bytes {hbm_bytes / 1e9:.3f} GB/launch; traffic = ncu DRAM "
                 "bytes per launch (profiles/k1_traffic.json)"),
        "secondary": {
            # SURVEY §8d's graded interpolation bound (TMU rate: 4 bilinear/clk/SM);
            # the smem-lerp kernel is not limited by it and exceeds it
            "graded_interp_gups": interp_peak, "graded_interp_frac": per_gpu_gups / interp_peak,
            # scripts/tex_bench.cu on this pool's B200 (profiles/r1_tex_microbench.txt):
            # tex2D fp32 bilinear fetches measured at 1161 G/s = 3.99 / clk / SM
            "tex2d_bilinear_measured_gfetch_s": 1161.0,
            "hbm_peak_gbs": pk.get("hbm_gbs"),
            "hbm_compulsory_frac": (hbm_bytes / (k1_avg / 1e3) / 1e9) / float(pk.get("hbm_gbs", 6545.9))},
    }

    # ---- CPU baseline (rank 0, N = 1 only) ----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            nz_s = 8
            z0_s = C4["n"] // 2 - nz_s // 2
            # the same filtered array the GPU consumed, embedded in the full
            # detector (rows outside the band are never tapped by these slices)
            sino_np = np.zeros((C4["views"], C4["nv"], C4["nu"]), np.float32)
            sino_np[:, me.v0:me.v0 + me.n_rows] = band.cpu().numpy()
            gups, kind, dt, ref_out = cpu_reference_sample(sino_np, z0_s, nz_s,
                                                           os.cpu_count() or 1)
            ours = slab[z0_s:z0_s + nz_s].cpu().numpy()
            d = np.abs(ours.astype(np.float64) - ref_out.astype(np.float64) * scale)
            cpu = {"value": gups, "unit": UNIT, "cores": os.cpu_count(), "kind": kind,
                   "sample": f"z-slices [{z0_s},{z0_s + nz_s}) of 512, all 496 views ({dt:.1f} s)",
                   "parity_vs_gpu": {"max_rel": float(d.max() / (np.abs(ref_out).max() * scale)),
                                     "rel_rmse": float(np.linalg.norm(d) /
                                                       (np.linalg.norm(ref_out.astype(np.float64)) * scale))}}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    # ---- config c5: iterative TV loop (1024^3, 720 x [2048 x 1536]) ----------
    c5 = None
    if args.c5_iters > 0:
        del h_band, h_slab, band, raw_band, slab, part
        torch.cuda.empty_cache()
        c5 = run_c5(tg, D, torch, dist, dev, rank, world, backend, args.c5_iters, max_over_ranks,
                    barrier)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (SURVEY App. A separable bump, FDK-filtered by K3; Shepp-Logan for FP)",
            "config": bench_config(world),
            "slab": {"z0": me.z0, "nz": me.nz, "rows": [me.v0, me.n_rows]},
            "ranks": ranks, "backend": backend if world > 1 else None,
            "nccl_debug": os.environ.get("NCCL_DEBUG"),
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": e2e_h2d,
                    "d2h_bytes_per_step": e2e_d2h,
                    "path": "tg_cone_backproject_slab_host (pinned host band -> device; "
                            "centre-out z phases: each ring uploads only its new detector rows "
                            "of each view's own footprint (3D copies per 8-view group) in view "
                            "chunks overlapped with K1, finished rings download while later "
                            "rings upload)", "host_band_bytes": e2e_band_bytes, "max_rel_diff_vs_device": e2e_parity,
                    "ms_per_step": 1e3 * e2e_s / e2e_n, "step_ms": e2e_steps_ms, "pcie": pcie},
            "fp": {"metric": "cone forward projection Gsamples/s (c4, Shepp-Logan)",
                   "value": fp_value, "unit": "Gsamples/s", "ms": fp_ms, "samples": fp_samples,
                   "roofline": {"bound": "l1", "peak": l1_peak / 2, "frac": fp_value / (l1_peak / 2),
                                "note": "32 B of taps (two 16-B quad gathers) per trilinear sample"},
                   "graded_interp_frac": fp_value / (interp_peak / 2), "graded_interp_peak": interp_peak / 2,
                   # scripts/k2_tex_bench.cu: the same gather pattern with ideal coherence
                   "measured_gather_ceiling_gsamples": 611.0,
                   "measured_gather_ceiling_frac": fp_value / 611.0},
            "fdk_e2e": fdk_e2e,
            "k1_calibrated": k1_cal,
            "k3_fdk_prefilter_ms": k3_ms, "k1_ms_mean": k1_avg, "k1_ms_min": min(k1_ms),
            # FDK of this rank's slab (pipelines.hpp:73-84): K3 on the band + K1
            "fdk_ms": k3_ms + k1_avg,
            "roofline": roofline, "clocks": clocks, "gpu_launches": gpu_launches,
            "cpu_baseline": cpu,
            "c5_tv": c5,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


C5 = dict(n=1024, spacing=0.25, nu=2048, nv=1536, det=0.4, views=720, range_deg=360.0, sid=750.0,
          sdd=1200.0, lr=2e-7, tv_lambda=0.05)
C5_SAMPLES = 1.614458e12  # exact sum over rays of the reference's sample count


def run_c5(tg, D, torch, dist, dev, rank, world, backend, iters, max_over_ranks, barrier):
    """BASELINE config c5: the TV-regularised cone-beam loop (pipelines.hpp:
    273-299 over a cone geometry) at 1024^3, 720 views of 2048 x 1536, on the
    Shepp-Logan phantom.  N = 1: the device-resident C ABI loop
    (tg_cone_tv_reconstruct); N > 1 on one node: the fused loop (angle-sharded
    K2, K8 storing residual row bands into the slab owners' buffers, slab K1,
    K9 storing the updated slab into every replica — peer stores over NVLink);
    across nodes the NCCL loop (all_to_all + all_gather).  A call with I
    iterations runs I (forward, backward, step) rounds plus one final forward
    for the last loss, so seconds per iteration = (T(I) - T(0)) / I, both
    device-timed with CUDA events (max over ranks)."""
    vol = tg.VolumeSpec.centered([C5["n"]] * 3, [C5["spacing"]] * 3)
    det = tg.Detector2D.centered(C5["nu"], C5["nv"], C5["det"], C5["det"])
    geo = tg.make_cone(vol, det, C5["views"], C5["range_deg"] * math.pi / 180.0, C5["sid"],
                       C5["sdd"])
    views = D.view_partition(geo, world)
    vw0, vwn = views[rank]
    # all ranks on one node (NVSwitch): exchanges fused into the kernels as
    # CUDA-IPC peer stores; across nodes: NCCL all_to_all / all_gather
    single_node = int(os.environ.get("LOCAL_WORLD_SIZE", world)) == world
    ph = tg.shepp_logan_3d(vol, device=dev).data
    p = tg.cone_forward_views(geo, ph, vw0, vwn)
    del ph
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    cfg_name = ("c5: iterative TV cone loop, 1024^3 @0.25mm, 720 x [2048 x 1536] @0.4mm, 360 deg, "
                f"SID 750 / SDD 1200, lr {C5['lr']}, tv_lambda {C5['tv_lambda']}")

    mode = {"p2p": single_node and world > 1, "fallback": None}

    def timed(n_it):
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if world == 1:
            cfg = tg.ExperimentConfig(learning_rate=C5["lr"], iterations=n_it,
                                      tv_lambda=C5["tv_lambda"])
            sino = tg.Sinogram.cone_beam(geo.n_projections, det, data=p)
            _, hist = tg.tv_reconstruct(sino, geo, cfg)
        elif mode["p2p"]:
            try:
                _, hist = D.tv_reconstruct_p2p(geo, p, n_it, C5["lr"], C5["tv_lambda"])
            except D.P2PUnavailable as e:  # raised on every rank together
                mode["p2p"], mode["fallback"] = False, str(e)[:200]
                _, hist = D.tv_reconstruct_sharded(geo, p, n_it, C5["lr"], C5["tv_lambda"])
        else:
            _, hist = D.tv_reconstruct_sharded(geo, p, n_it, C5["lr"], C5["tv_lambda"])
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b)), hist

    timed(0)  # warm: plan buffers, the allocator pool, constant banks
    t0, _ = timed(0)
    tI, hist = timed(iters)
    s_per_it = (tI - t0) / iters / 1e3
    updates = float(C5["n"]) ** 3 * C5["views"]
    return {"workload": cfg_name, "iterations": iters, "s_per_iter": s_per_it,
            "final_forward_s": t0 / 1e3,
            "fp_plus_bp_units_per_s": {"Gsamples": C5_SAMPLES / s_per_it / 1e9,
                                       "GUPS": updates / s_per_it / 1e9},
            "loss_history": hist, "path": "tg_cone_tv_reconstruct" if world == 1 else
            ("distributed.tv_reconstruct_p2p (K8 residual scatter + K9 slab broadcast as "
             "CUDA-IPC peer stores)" if mode["p2p"] else
             "distributed.tv_reconstruct_sharded (NCCL all_to_all + all_gather)"),
            "p2p_fallback_reason": mode["fallback"],
            "views_per_rank": vwn}


_SAMPLES_CACHE = os.path.join(ROOT, "profiles", "c4_samples.json")


def samples_c4(geo):
    """Exact sum over rays of ceil((t1 - t0) / step) for c4 (SURVEY App. A:
    2.179549e11), from the reference's clip rule; cached."""
    try:
        with open(_SAMPLES_CACHE) as f:
            return int(json.load(f)["samples"])
    except Exception:
        pass
    return 217954900000  # SURVEY Appendix A (2.179549e11)


if __name__ == "__main__":
    main()
