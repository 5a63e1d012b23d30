"""Command-line front end on the device path: the
reference's ``tomograd`` subcommands (cli.hpp:1-358) over the file formats of
io.py, every operator running in the sm_100a kernels.

    python -m paper_1904_13342_b200.cli phantom     --geometry g.json --out phantom.json
    python -m paper_1904_13342_b200.cli project     --geometry g.json --image phantom.json --out sino.json
    python -m paper_1904_13342_b200.cli reconstruct fdk --geometry g.json --sino sino.json --out recon.json
    python -m paper_1904_13342_b200.cli export-pgm  --image recon.json --lo 0 --hi 0.05 --out recon.pgm

Exit codes as the reference (cli.hpp:9, 341-353): 0 success, 1 bad usage, 2 data
or processing error (message on stderr as "error: <what>").  Outputs are
byte-identical run to run (deterministic kernels; acceptance.cpp:486-548).

Differences, by design: ``reconstruct iterative --geometry`` accepts every
geometry type (the reference's graph nodes do; its CLI restricts to
parallel2d) so the config-5 cone loop is reachable from the shell.
``learn-filter`` (pipelines.hpp:191-261) trains the Fourier filter weights
through the device graph (graph.py).
"""
from __future__ import annotations

import argparse
import sys
from typing import List

import numpy as np

from . import io as tio
from ._native import Error


class _UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse exits 2 by default: the reference uses 1
        raise _UsageError(message)


def _device():
    import torch
    if not torch.cuda.is_available():
        raise Error("no CUDA device visible: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _expect(geo, cls, who, what):
    if not isinstance(geo, cls):
        raise Error(f"{who} expects a {what} geometry")
    return geo


def _slice_for_display(img, index: int):
    """cli.hpp:38-48"""
    if img.spec.dims() == 2:
        if index >= 0:
            raise Error("--slice only applies to 3D images")
        return img
    nz = img.spec.shape[2]
    iz = nz // 2 if index < 0 else index
    if iz >= nz:
        raise Error("slice index out of range")
    return tio.extract_slice(img, 2, iz)


def _history_rows(h):
    return [[float(i), float(v)] for i, v in enumerate(h)]


def _central_profile(path, img):
    """cli.hpp:59-64"""
    sl = tio.extract_slice(img, 2, img.spec.shape[2] // 2) if img.spec.dims() == 3 else img
    tio.write_profile_csv(path, tio.line_profile(sl, 0, sl.spec.shape[1] // 2))


def experiment_fdk_short_scan(geo, cfg, use_parker=True, device=None):
    """pipelines.hpp:140-154: phantom -> forward projection -> noise -> FDK."""
    from .iterative import add_gaussian_noise
    from .phantom import shepp_logan_3d
    from .pipelines import fdk_reconstruct
    from .projector import forward_project
    if cfg.phantom != "shepp-logan":
        raise Error("cone-beam experiment expects the head phantom")
    phantom = shepp_logan_3d(geo.volume, device)
    sino = forward_project(phantom, geo)
    if cfg.noise_relative_std > 0.0:
        sino = add_gaussian_noise(sino, cfg.noise_relative_std, cfg.seed)
    return phantom, sino, fdk_reconstruct(sino, geo, use_parker)


def _build() -> argparse.ArgumentParser:
    ap = _Parser(prog="tomograd", description="differentiable tomography toolkit (B200 path)")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    p = sub.add_parser("phantom", help="rasterize a test object onto a volume grid")
    p.add_argument("--geometry")
    p.add_argument("--out", required=True)
    p.add_argument("--name", default="shepp-logan")
    p.add_argument("--type", default="shepp-logan-2d",
                   choices=["shepp-logan-2d", "shepp-logan-3d", "disk"])
    p.add_argument("--size", type=int, default=0)
    p.add_argument("--spacing", type=float, default=1.0)

    p = sub.add_parser("trajectory", help="dump per-view angles, rays or projection matrices")
    p.add_argument("--geometry", required=True)
    p.add_argument("--out", required=True)

    p = sub.add_parser("project", help="forward project an image to a sinogram")
    p.add_argument("--geometry", required=True)
    p.add_argument("--image", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--noise-rel", type=float, default=0.0)
    p.add_argument("--seed", type=int, default=1337)

    rec = sub.add_parser("reconstruct", help="sinogram to image")
    rs = rec.add_subparsers(dest="method", required=True, parser_class=_Parser)
    p = rs.add_parser("fbp", help="filtered backprojection (parallel beam)")
    p.add_argument("--geometry", required=True)
    p.add_argument("--sino", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--filter", default="ramlak", choices=["ramlak", "ramp"])
    p.add_argument("--filter-csv", default="")
    p = rs.add_parser("fdk", help="cone-beam filtered backprojection (short scans supported)")
    p.add_argument("--config", default="")
    p.add_argument("--geometry", default="")
    p.add_argument("--sino", default="")
    p.add_argument("--out", default="")
    p.add_argument("--no-short-scan-weights", action="store_true")
    p = rs.add_parser("iterative", help="gradient-descent reconstruction with a TV prior")
    p.add_argument("--config", default="")
    p.add_argument("--geometry", default="")
    p.add_argument("--sino", default="")
    p.add_argument("--out", default="")
    p.add_argument("--loss-csv", default="")
    p.add_argument("--lambda", dest="tv_lambda", type=float, default=0.0)
    p.add_argument("--lr", type=float, default=1e-3)
    p.add_argument("--iterations", type=int, default=100)

    p = sub.add_parser("learn-filter",
                       help="train reconstruction-filter weights against a known phantom")
    p.add_argument("--config", required=True)

    p = sub.add_parser("profile", help="extract a line profile as CSV")
    p.add_argument("--image", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--axis", default="x", choices=["x", "y"])
    p.add_argument("--index", type=int, default=-1)
    p.add_argument("--slice", type=int, default=-1)

    p = sub.add_parser("export-pgm", help="window a 2D image (or a z slice) to 8-bit PGM")
    p.add_argument("--image", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--lo", type=float, default=None)
    p.add_argument("--hi", type=float, default=None)
    p.add_argument("--slice", type=int, default=-1)
    return ap


def _run(a) -> None:
    from .geometry import ConeGeometry, ParallelGeometry, VolumeSpec
    from .iterative import ExperimentConfig, add_gaussian_noise, experiment_iterative_tv, \
        make_phantom_2d, tv_reconstruct
    from .phantom import shepp_logan_3d
    from .pipelines import FilterKind, fbp_reconstruct, fdk_reconstruct
    from .projector import forward_project
    from .filtering import Filter1D

    if a.cmd == "phantom":  # cli.hpp:75-108
        if (a.geometry is None) == (a.size == 0):
            raise Error("pass exactly one of --geometry or --size")
        dev = _device()
        if a.geometry:
            geo = tio.load_geometry(a.geometry)
            if isinstance(geo, ConeGeometry):
                if a.name != "shepp-logan":
                    raise Error("3D geometries support the shepp-logan phantom only")
                tio.write_image(a.out, shepp_logan_3d(geo.volume, dev))
            else:
                tio.write_image(a.out, make_phantom_2d(a.name, geo.volume, dev))
            return
        if a.type == "shepp-logan-3d":
            vol = VolumeSpec.centered([a.size] * 3, [a.spacing] * 3)
            tio.write_image(a.out, shepp_logan_3d(vol, dev))
            return
        vol = VolumeSpec.centered([a.size] * 2, [a.spacing] * 2)
        tio.write_image(a.out, make_phantom_2d("disk" if a.type == "disk" else "shepp-logan",
                                               vol, dev))
    elif a.cmd == "trajectory":
        tio.write_trajectory(a.out, tio.load_geometry(a.geometry))
    elif a.cmd == "project":  # cli.hpp:126-147
        geo = tio.load_geometry(a.geometry)
        img = tio.read_image(a.image, device=_device())
        sino = forward_project(img, geo)
        if a.noise_rel > 0.0:
            sino = add_gaussian_noise(sino, a.noise_rel, a.seed)
        tio.write_sinogram(a.out, sino)
    elif a.cmd == "reconstruct" and a.method == "fbp":  # cli.hpp:152-176
        geo = tio.load_geometry(a.geometry)
        g = _expect(geo, ParallelGeometry, "fbp", "parallel2d")
        sino = tio.read_sinogram(a.sino, geo, device=_device())
        if a.filter_csv:
            w = np.array(tio.read_filter_csv(a.filter_csv))
            filt = Filter1D(g.detector.n_bins, len(w), g.detector.spacing, w)
            tio.write_image(a.out, fbp_reconstruct(sino, g, filt))
            return
        kind = FilterKind.ramp if a.filter == "ramp" else FilterKind.ramlak
        tio.write_image(a.out, fbp_reconstruct(sino, g, kind))
    elif a.cmd == "reconstruct" and a.method == "fdk":  # cli.hpp:178-215
        if a.config:
            if a.geometry or a.sino or a.out:
                raise Error("--config runs are self-contained; drop --geometry/--sino/--out")
            exp = tio.load_experiment_config(a.config)
            g = _expect(exp.geometry, ConeGeometry, "fdk", "cone3d")
            phantom, sino, rec = experiment_fdk_short_scan(g, exp.cfg, not a.no_short_scan_weights,
                                                           _device())
            for role, path in exp.outputs.items():
                if role == "image":
                    tio.write_image(path, rec)
                elif role == "phantom_image":
                    tio.write_image(path, phantom)
                elif role == "sinogram":
                    tio.write_sinogram(path, sino)
                elif role == "profile_csv":
                    _central_profile(path, rec)
                elif role == "phantom_profile_csv":
                    _central_profile(path, phantom)
                else:
                    raise Error(f"unknown output role '{role}'")
            return
        if not (a.geometry and a.sino and a.out):
            raise Error("need --config or all of --geometry, --sino, --out")
        geo = tio.load_geometry(a.geometry)
        g = _expect(geo, ConeGeometry, "fdk", "cone3d")
        sino = tio.read_sinogram(a.sino, geo, device=_device())
        tio.write_image(a.out, fdk_reconstruct(sino, g, not a.no_short_scan_weights))
    elif a.cmd == "reconstruct" and a.method == "iterative":  # cli.hpp:217-263
        if a.config:
            if a.geometry or a.sino or a.out:
                raise Error("--config runs are self-contained; drop --geometry/--sino/--out")
            exp = tio.load_experiment_config(a.config)
            g = _expect(exp.geometry, ParallelGeometry, "iterative", "parallel2d")
            r = experiment_iterative_tv(g, exp.cfg, device=_device())
            for role, path in exp.outputs.items():
                if role == "image":
                    tio.write_image(path, r.reconstruction)
                elif role == "fbp_image":
                    tio.write_image(path, r.fbp_reference)
                elif role == "phantom_image":
                    tio.write_image(path, r.phantom)
                elif role == "sinogram":
                    tio.write_sinogram(path, r.noisy_sinogram)
                elif role == "loss_csv":
                    tio.write_csv(path, ["iteration", "loss"], _history_rows(r.loss_history))
                elif role == "profile_csv":
                    _central_profile(path, r.reconstruction)
                elif role == "fbp_profile_csv":
                    _central_profile(path, r.fbp_reference)
                else:
                    raise Error(f"unknown output role '{role}'")
            return
        if not (a.geometry and a.sino and a.out):
            raise Error("need --config or all of --geometry, --sino, --out")
        geo = tio.load_geometry(a.geometry)
        sino = tio.read_sinogram(a.sino, geo, device=_device())
        cfg = ExperimentConfig(learning_rate=a.lr, iterations=a.iterations, tv_lambda=a.tv_lambda)
        rec, hist = tv_reconstruct(sino, geo, cfg)
        tio.write_image(a.out, rec)
        if a.loss_csv:
            tio.write_csv(a.loss_csv, ["iteration", "loss"], _history_rows(hist))
    elif a.cmd == "learn-filter":  # cli.hpp:265-288
        from .iterative import experiment_learn_filter
        exp = tio.load_experiment_config(a.config)
        g = _expect(exp.geometry, ParallelGeometry, "learn-filter", "parallel2d")
        r = experiment_learn_filter(g, exp.cfg, device=_device())
        for role, path in exp.outputs.items():
            if role == "filter_csv":
                tio.write_filter_csv(path, r.learned_weights)
            elif role == "ramp_csv":
                tio.write_filter_csv(path, r.ramp_init.weights)
            elif role == "ramlak_csv":
                tio.write_filter_csv(path, r.ramlak_reference.weights)
            elif role == "loss_csv":
                tio.write_csv(path, ["iteration", "loss"], _history_rows(r.loss_history))
            elif role == "distance_csv":
                tio.write_csv(path, ["iteration", "distance"], _history_rows(r.distance_history))
            elif role == "image":
                tio.write_image(path, r.reconstruction)
            elif role == "profile_csv":
                _central_profile(path, r.reconstruction)
            else:
                raise Error(f"unknown output role '{role}'")
    elif a.cmd == "profile":  # cli.hpp:290-313
        img = _slice_for_display(tio.read_image(a.image), a.slice)
        axis = 0 if a.axis == "x" else 1
        other_n = img.spec.shape[1 - axis]
        index = other_n // 2 if a.index < 0 else a.index
        tio.write_profile_csv(a.out, tio.line_profile(img, axis, index))
    elif a.cmd == "export-pgm":  # cli.hpp:315-339
        img = _slice_for_display(tio.read_image(a.image), a.slice)
        data = np.asarray(img.data, dtype=np.float64).ravel()
        lo, hi = a.lo, a.hi
        if lo is None or hi is None:
            mn = float(data.min()) if data.size else 0.0
            mx = float(data.max()) if data.size else 0.0
            lo = mn if lo is None else lo
            hi = mx if hi is None else hi
        tio.export_pgm(a.out, img, lo, hi)


def run(args: List[str]) -> int:
    """cli.hpp:67-357: one invocation; returns the exit code."""
    ap = _build()
    try:
        a = ap.parse_args(args)
    except _UsageError as e:
        print(f"tomograd: {e}", file=sys.stderr)
        return 1
    except SystemExit as e:  # --help
        return 0 if (e.code in (0, None)) else 1
    try:
        _run(a)
    except Exception as e:  # noqa: BLE001 — the reference maps any std::exception to 2
        print(f"error: {e}", file=sys.stderr)
        return 2
    return 0


def main() -> None:
    sys.exit(run(sys.argv[1:]))


if __name__ == "__main__":
    main()
