"""File formats around the projector path: io.hpp restated.

Arrays travel as a JSON sidecar plus a raw little-endian float32 payload
(io.hpp:1-19):  {"shape": [..] (fastest first), "spacing": [..],
"origin": [..], "dtype": "f32le", "data": "<name>.raw"}.  Geometry files
describe a scan, with optional explicit (calibrated) cone-beam projection
matrices normalised on load by set_matrices (io.hpp:353-410); they drive the
general (non-circular) K1 / K2 paths.  Error texts are the reference's.

Payloads are read straight into page-locked host memory when a device is
requested (``read_image(..., device=)`` / ``read_sinogram(..., device=)``), so
the copy to HBM is a single DMA.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Union

import numpy as np

from ._native import Error
from .containers import Image, Sinogram
from .geometry import (ConeGeometry, Detector1D, Detector2D, FanGeometry, ParallelGeometry,
                       VolumeSpec, check, make_cone, make_cone_from_matrices, make_fan,
                       make_parallel)
from .iterative import ExperimentConfig

AnyGeometry = Union[ParallelGeometry, FanGeometry, ConeGeometry]


@dataclass
class RawArray:
    """io.hpp:47-52"""
    shape: List[int] = field(default_factory=list)
    spacing: List[float] = field(default_factory=list)
    origin: List[float] = field(default_factory=list)
    data: np.ndarray = None  # float32, memory order


def _raw_path_for(sidecar: str) -> str:
    """io.hpp:56-60"""
    return os.path.splitext(sidecar)[0] + ".raw"


def _parse_json_file(path: str):
    """io.hpp:62-68"""
    try:
        f = open(path)
    except OSError:
        raise Error("cannot open " + path)
    with f:
        try:
            return json.load(f)
        except ValueError:
            raise Error("malformed JSON in " + path)


def _ensure_parent(path: str) -> None:
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)


def write_raw(sidecar: str, arr: RawArray) -> None:
    """io.hpp:78-107 (payload rounded to float32, little-endian)"""
    check(len(arr.shape) == len(arr.spacing) and len(arr.shape) == len(arr.origin),
          "shape, spacing and origin must have the same rank")
    raw = _raw_path_for(sidecar)
    _ensure_parent(sidecar)
    payload = np.ascontiguousarray(np.asarray(arr.data).ravel(), dtype="<f4")
    try:
        payload.tofile(raw)
    except OSError:
        raise Error("cannot write " + raw)
    j = {"shape": [int(s) for s in arr.shape], "spacing": [float(s) for s in arr.spacing],
         "origin": [float(s) for s in arr.origin], "dtype": "f32le",
         "data": os.path.basename(raw)}
    try:
        with open(sidecar, "w") as f:
            f.write(json.dumps(j, indent=2) + "\n")
    except OSError:
        raise Error("cannot write " + sidecar)


def read_raw(sidecar: str, pinned: bool = False) -> RawArray:
    """io.hpp:109-136.  ``pinned``: read the payload into page-locked memory
    (a torch tensor's storage) for a single-DMA upload."""
    j = _parse_json_file(sidecar)
    check(isinstance(j, dict) and "shape" in j and "dtype" in j and "data" in j,
          "sidecar misses required keys in " + sidecar)
    check(j["dtype"] == "f32le", "unsupported dtype in " + sidecar)
    shape = [int(s) for s in j["shape"]]
    rank = len(shape)
    spacing = [float(s) for s in j.get("spacing", [1.0] * rank)]
    origin = [float(s) for s in j.get("origin", [0.0] * rank)]
    check(len(spacing) == rank and len(origin) == rank, "sidecar rank mismatch in " + sidecar)
    count = 1
    for n in shape:
        count *= n
    raw = os.path.join(os.path.dirname(sidecar), j["data"])
    try:
        nbytes = os.path.getsize(raw)
    except OSError:
        raise Error("cannot open " + raw)
    check(nbytes == count * 4, "payload size does not match the header shape for " + raw)
    if pinned:
        import torch
        buf = torch.empty(count, dtype=torch.float32, pin_memory=True)
        data = buf.numpy()
        with open(raw, "rb") as f:
            got = f.readinto(memoryview(data).cast("B"))
        check(got == nbytes, "failed reading " + raw)
    else:
        data = np.fromfile(raw, dtype="<f4", count=count).astype(np.float32, copy=False)
        check(data.size == count, "failed reading " + raw)
    return RawArray(shape, spacing, origin, data)


def _to_device(data: np.ndarray, shape, device):
    import torch
    t = torch.from_numpy(data).view(*shape)
    return t.to(device, non_blocking=True) if device is not None else t


def write_image(sidecar: str, img: Image) -> None:
    """io.hpp:138-143"""
    data = img.data.detach().cpu().numpy() if hasattr(img.data, "detach") else img.data
    write_raw(sidecar, RawArray(list(img.spec.shape), list(img.spec.spacing),
                                list(img.spec.origin), data))


def read_image(sidecar: str, device=None) -> Image:
    """io.hpp:145-154.  device=None: host (numpy) image; else a CUDA tensor."""
    arr = read_raw(sidecar, pinned=device is not None)
    check(len(arr.shape) in (2, 3), "expected a 2D or 3D image in " + sidecar)
    spec = VolumeSpec(arr.shape, arr.spacing, arr.origin)
    spec.validate()
    shp = tuple(reversed(arr.shape))
    data = arr.data.reshape(shp) if device is None else _to_device(arr.data, shp, device)
    return Image(spec, data)


def write_sinogram(sidecar: str, s: Sinogram) -> None:
    """io.hpp:156-171 (cone: spacing {du, dv, 1}, origin {ou, ov, 0})"""
    data = s.data.detach().cpu().numpy() if hasattr(s.data, "detach") else s.data
    if s.is_cone():
        d = s.detector2d
        arr = RawArray([d.n_u, d.n_v, s.n_projections], [d.spacing_u, d.spacing_v, 1.0],
                       [d.origin_u, d.origin_v, 0.0], data)
    else:
        d = s.detector1d
        arr = RawArray([d.n_bins, s.n_projections], [d.spacing, 1.0], [d.origin, 0.0], data)
    write_raw(sidecar, arr)


def read_sinogram(sidecar: str, geo: AnyGeometry, device=None) -> Sinogram:
    """io.hpp:173-193: projection data bound to a known geometry."""
    arr = read_raw(sidecar, pinned=device is not None)
    if isinstance(geo, ConeGeometry):
        want = [geo.detector.n_u, geo.detector.n_v, geo.n_projections]
    else:
        want = [geo.detector.n_bins, geo.n_projections]
    check(arr.shape == want, "projection data in " + sidecar + " does not match the geometry")
    shp = tuple(reversed(want))
    data = arr.data.reshape(shp) if device is None else _to_device(arr.data, shp, device)
    if isinstance(geo, ConeGeometry):
        return Sinogram.cone_beam(geo.n_projections, geo.detector, data=data)
    return Sinogram.planar(geo.n_projections, geo.detector, data=data)


# ---- geometry files (io.hpp:353-433) -------------------------------------


def load_geometry_json(j: dict, origin_hint: str) -> AnyGeometry:
    """io.hpp:353-406"""
    for key in ("type", "volume_shape", "volume_spacing", "detector_shape", "detector_spacing",
                "n_projections", "angular_range_deg"):
        check(isinstance(j, dict) and key in j,
              f"geometry misses key '{key}' in {origin_hint}")
    typ = str(j["type"])
    vshape = [int(v) for v in j["volume_shape"]]
    vspacing = [float(v) for v in j["volume_spacing"]]
    dshape = [int(v) for v in j["detector_shape"]]
    dspacing = [float(v) for v in j["detector_spacing"]]
    n_proj = int(j["n_projections"])
    rng = float(j["angular_range_deg"]) * math.pi / 180.0
    check(len(vshape) == len(vspacing), "volume shape/spacing rank mismatch")
    check(len(dshape) == len(dspacing), "detector shape/spacing rank mismatch")
    if typ == "parallel2d":
        check(len(vshape) == 2 and len(dshape) == 1,
              "parallel2d expects a 2D volume and 1D detector")
        return make_parallel(VolumeSpec.centered(vshape, vspacing),
                             Detector1D.centered(dshape[0], dspacing[0]), n_proj, rng)
    if typ == "fan2d":
        check(len(vshape) == 2 and len(dshape) == 1, "fan2d expects a 2D volume and 1D detector")
        check("sid" in j and "sdd" in j, "fan2d needs sid and sdd")
        return make_fan(VolumeSpec.centered(vshape, vspacing),
                        Detector1D.centered(dshape[0], dspacing[0]), n_proj, rng,
                        float(j["sid"]), float(j["sdd"]))
    if typ == "cone3d":
        check(len(vshape) == 3 and len(dshape) == 2, "cone3d expects a 3D volume and 2D detector")
        check("sid" in j and "sdd" in j, "cone3d needs sid and sdd")
        vol = VolumeSpec.centered(vshape, vspacing)
        det = Detector2D.centered(dshape[0], dshape[1], dspacing[0], dspacing[1])
        sid, sdd = float(j["sid"]), float(j["sdd"])
        if "projection_matrices" in j:
            mats = []
            for jm in j["projection_matrices"]:
                vals = [float(v) for v in jm]
                check(len(vals) == 12, "projection matrices need 12 row-major entries")
                mats.append(vals)
            check(len(mats) == n_proj, "projection matrix count must equal n_projections")
            return make_cone_from_matrices(vol, det, rng, sid, sdd, np.array(mats))
        return make_cone(vol, det, n_proj, rng, sid, sdd)
    raise Error(f"unknown geometry type '{typ}' in {origin_hint}")


def load_geometry(path: str) -> AnyGeometry:
    """io.hpp:408-410"""
    return load_geometry_json(_parse_json_file(path), path)


def write_trajectory(path: str, geo: AnyGeometry) -> None:
    """io.hpp:412-438: per-view pose data"""
    j = {"angles_rad": [float(a) for a in geo.angles]}
    if isinstance(geo, ConeGeometry):
        j["type"] = "cone3d"
        j["projection_matrices"] = [[float(v) for v in m] for m in
                                    np.asarray(geo.matrices).reshape(-1, 12)]
    else:
        j["type"] = "fan2d" if isinstance(geo, FanGeometry) else "parallel2d"
        j["rays"] = [[float(r[0]), float(r[1])] for r in np.asarray(geo.rays).reshape(-1, 2)]
    _ensure_parent(path)
    try:
        with open(path, "w") as f:
            f.write(json.dumps(j, indent=2) + "\n")
    except OSError:
        raise Error("cannot write " + path)


@dataclass
class LoadedExperiment:
    """io.hpp:442-446"""
    geometry: AnyGeometry
    cfg: ExperimentConfig
    outputs: Dict[str, str]


def load_experiment_config(path: str) -> LoadedExperiment:
    """io.hpp:448-486"""
    j = _parse_json_file(path)
    check(isinstance(j, dict) and "geometry" in j, "experiment config needs a geometry")
    base = os.path.dirname(path)
    if isinstance(j["geometry"], str):
        gp = j["geometry"]
        if not os.path.isabs(gp):
            gp = os.path.join(base, gp)
        geo = load_geometry(gp)
    else:
        geo = load_geometry_json(j["geometry"], path)
    d = ExperimentConfig()
    cfg = ExperimentConfig(
        phantom=str(j.get("phantom", d.phantom)),
        noise_relative_std=float(j.get("noise_relative_std", d.noise_relative_std)),
        learning_rate=float(j.get("learning_rate", d.learning_rate)),
        iterations=int(j.get("iterations", d.iterations)),
        tv_lambda=float(j.get("tv_lambda", d.tv_lambda)),
        seed=int(j.get("seed", d.seed)),
        filter_window=int(j.get("filter_window", d.filter_window)))
    outputs = {}
    for k, v in (j.get("outputs") or {}).items():
        outputs[k] = v if os.path.isabs(v) else os.path.join(base, v)
    return LoadedExperiment(geo, cfg, outputs)


# ---- CSV, slices, profiles, PGM (io.hpp:195-351) ---------------------------


def format_double(v: float) -> str:
    """io.hpp:289-294: 17 significant digits (the C++ ostream default float
    format is printf's %g)"""
    return "%.17g" % v


def write_csv(path: str, header: List[str], rows: List[List[float]]) -> None:
    """io.hpp:296-309"""
    _ensure_parent(path)
    try:
        with open(path, "w") as f:
            f.write(",".join(header) + "\n")
            for row in rows:
                f.write(",".join(format_double(float(v)) for v in row) + "\n")
    except OSError:
        raise Error("cannot write " + path)


def read_csv(path: str):
    """io.hpp:316-338 -> (header, rows)"""
    try:
        f = open(path)
    except OSError:
        raise Error("cannot open " + path)
    header, rows, first = [], [], True
    with f:
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            cells = line.split(",")
            if first:
                header, first = cells, False
                continue
            rows.append([float(c) for c in cells])
    return header, rows


def write_filter_csv(path: str, weights) -> None:
    """io.hpp:347-352"""
    write_csv(path, ["bin_index", "weight"], [[float(k), float(w)] for k, w in enumerate(weights)])


def read_filter_csv(path: str) -> List[float]:
    """io.hpp:354-362"""
    _, rows = read_csv(path)
    out = []
    for row in rows:
        check(len(row) == 2, "filter CSV rows must be (bin_index, weight)")
        out.append(row[1])
    return out


def _host(img: Image) -> np.ndarray:
    return img.data.detach().cpu().numpy() if hasattr(img.data, "detach") else np.asarray(img.data)


def extract_slice(img: Image, axis: int, index: int) -> Image:
    """io.hpp:226-252: 2D slice of a 3D image perpendicular to ``axis``"""
    check(img.spec.dims() == 3, "slice extraction expects a 3D image")
    check(0 <= axis < 3, "axis out of range")
    check(0 <= index < img.spec.shape[axis], "slice index out of range")
    a1 = 1 if axis == 0 else 0
    a2 = 1 if axis == 2 else 2
    spec = VolumeSpec([img.spec.shape[a1], img.spec.shape[a2]],
                      [img.spec.spacing[a1], img.spec.spacing[a2]],
                      [img.spec.origin[a1], img.spec.origin[a2]])
    v = _host(img)  # [z][y][x]
    sl = [slice(None)] * 3
    sl[2 - axis] = index
    out = v[tuple(sl)]  # remaining axes in (slowest, fastest) = (a2, a1) order
    return Image(spec, np.ascontiguousarray(out, dtype=np.float32))


def line_profile(img: Image, axis: int, index: int):
    """io.hpp:260-274 -> list of (position, value)"""
    check(img.spec.dims() == 2, "line profiles run over 2D images (slice 3D first)")
    check(0 <= axis < 2, "axis out of range")
    other = 1 - axis
    check(0 <= index < img.spec.shape[other], "profile index out of range")
    v = _host(img)  # [y][x]
    pts = []
    for i in range(img.spec.shape[axis]):
        ix, iy = (i, index) if axis == 0 else (index, i)
        pts.append((img.spec.origin[axis] + float(i) * img.spec.spacing[axis], float(v[iy, ix])))
    return pts


def write_profile_csv(path: str, pts) -> None:
    """io.hpp:340-345"""
    write_csv(path, ["position_mm", "value"], [[p, v] for p, v in pts])


def export_pgm(path: str, img: Image, lo: float, hi: float) -> None:
    """io.hpp:198-222: binary PGM, window [lo, hi) -> 0..255 (floor), +y up"""
    check(img.spec.dims() == 2, "PGM export expects a 2D image")
    check(lo < hi, "window must satisfy lo < hi")
    nx, ny = img.spec.shape[0], img.spec.shape[1]
    _ensure_parent(path)
    scale = 255.0 / (hi - lo)
    v = np.floor((_host(img).astype(np.float64) - lo) * scale)
    v = np.clip(v, 0.0, 255.0).astype(np.uint8)[::-1]
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{nx} {ny}\n255\n".encode())
            f.write(np.ascontiguousarray(v).tobytes())
    except OSError:
        raise Error("cannot write " + path)
