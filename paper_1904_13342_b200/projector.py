"""forward_project / back_project — the reference's overload set
(projector.hpp:171-313) dispatched on the geometry type, running the sm_100a
kernels K1/K2 (cone), K4-K7 (fan / parallel) through the C ABI."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .containers import Image, Sinogram, is_host, require_f32, stream_of
from .geometry import ConeGeometry, FanGeometry, ParallelGeometry, check


def _check_volume_match(a, b):
    """projector.hpp:154-157"""
    check(list(a.shape) == list(b.shape) and list(a.spacing) == list(b.spacing)
          and list(a.origin) == list(b.origin),
          "volume does not match the geometry's volume spec")


def _check_planar_sino(s: Sinogram, geo):
    """projector.hpp:159-165"""
    check(not s.is_cone() and s.n_projections == geo.n_projections
          and s.detector1d.n_bins == geo.detector.n_bins,
          "sinogram shape does not match the geometry")


def _check_cone_sino(s: Sinogram, geo: ConeGeometry):
    """projector.hpp:285-288"""
    check(s.is_cone() and s.n_projections == geo.n_projections
          and s.detector2d.n_u == geo.detector.n_u and s.detector2d.n_v == geo.detector.n_v,
          "sinogram shape does not match the geometry")


def _check_shape(t, shape, what):
    """Full tensor shape against the geometry before any raw pointer crosses
    the C ABI (the reference's containers carry their shape; a mismatch here
    is the reference's check() error, never an out-of-bounds device access)."""
    check(tuple(t.shape) == tuple(int(x) for x in shape), f"{what} does not match the geometry")


def _out_tensor(out, shape, like, what):
    if out is None:
        return torch.empty(tuple(shape), dtype=torch.float32, device=like.device)
    check(isinstance(out, torch.Tensor) and out.dtype == torch.float32 and out.is_cuda
          and out.device == like.device, f"{what} must be a float32 tensor on the input's device")
    check(out.is_contiguous(), f"{what} must be contiguous")
    _check_shape(out, shape, what)
    return out


def _dev(t: torch.Tensor) -> int:
    return t.device.index if t.device.index is not None else torch.cuda.current_device()


def forward_project(img: Image, geo) -> Sinogram:
    """projector.hpp:171-184 (parallel), 212-230 (fan), 264-281 (cone)."""
    _check_volume_match(img.spec, geo.volume)
    data = require_f32(img.data, "image data")
    _check_shape(data, geo.volume.torch_shape, "volume data")
    L = N.lib()
    if isinstance(geo, ConeGeometry):
        shape = (geo.n_projections, geo.detector.n_v, geo.detector.n_u)
        if is_host(data):
            out = np.zeros(shape, np.float32)
            N.check(L.tg_cone_forward_host(geo._plan(0), data.ctypes.data, out.ctypes.data))
        else:
            out = torch.empty(shape, dtype=torch.float32, device=data.device)
            N.check(L.tg_cone_forward(geo._plan(_dev(data)), data.data_ptr(), out.data_ptr(),
                                      stream_of(data)))
        return Sinogram.cone_beam(geo.n_projections, geo.detector, data=out)
    check(isinstance(geo, (ParallelGeometry, FanGeometry)), "unknown geometry type")
    shape = (geo.n_projections, geo.detector.n_bins)
    if is_host(data):
        out = np.zeros(shape, np.float32)
        N.check(L.tg_planar_forward_host(geo._plan(0), data.ctypes.data, out.ctypes.data))
    else:
        out = torch.empty(shape, dtype=torch.float32, device=data.device)
        N.check(L.tg_planar_forward(geo._plan(_dev(data)), data.data_ptr(), out.data_ptr(),
                                    stream_of(data)))
    return Sinogram.planar(geo.n_projections, geo.detector, data=out)


def back_project(sino: Sinogram, geo, scale: float = 1.0) -> Image:
    """projector.hpp:186-208 (parallel), 232-260 (fan, 1/U^2), 283-313 (cone, 1/w^2).
    ``scale`` (default 1, the reference's behaviour) is fused into the epilogue."""
    L = N.lib()
    if isinstance(geo, ConeGeometry):
        _check_cone_sino(sino, geo)
        data = require_f32(sino.data, "sinogram data")
        _check_shape(data, (geo.n_projections, geo.detector.n_v, geo.detector.n_u),
                     "sinogram data")
        if is_host(data):
            check(scale == 1.0, "host back-projection has no scale argument")
            out = np.zeros(geo.volume.torch_shape, np.float32)
            N.check(L.tg_cone_backproject_host(geo._plan(0), data.ctypes.data, out.ctypes.data))
        else:
            out = torch.empty(geo.volume.torch_shape, dtype=torch.float32, device=data.device)
            N.check(L.tg_cone_backproject(geo._plan(_dev(data)), data.data_ptr(), out.data_ptr(),
                                          float(scale), 0, stream_of(data)))
        return Image(geo.volume, out)
    check(isinstance(geo, (ParallelGeometry, FanGeometry)), "unknown geometry type")
    _check_planar_sino(sino, geo)
    data = require_f32(sino.data, "sinogram data")
    _check_shape(data, (geo.n_projections, geo.detector.n_bins), "sinogram data")
    if is_host(data):
        check(scale == 1.0, "host back-projection has no scale argument")
        out = np.zeros(geo.volume.torch_shape, np.float32)
        N.check(L.tg_planar_backproject_host(geo._plan(0), data.ctypes.data, out.ctypes.data))
    else:
        out = torch.empty(geo.volume.torch_shape, dtype=torch.float32, device=data.device)
        N.check(L.tg_planar_backproject(geo._plan(_dev(data)), data.data_ptr(), out.data_ptr(),
                                        float(scale), 0, stream_of(data)))
    return Image(geo.volume, out)


# ---- lower-level device entry points (used by pipelines / distributed) ----


def cone_forward_views(geo: ConeGeometry, vol: torch.Tensor, view0: int, n_views: int,
                       out: torch.Tensor = None) -> torch.Tensor:
    """Angle-sharded cone forward projection: views [view0, view0 + n_views)."""
    vol = require_f32(vol, "volume")
    _check_shape(vol, geo.volume.torch_shape, "volume")
    check(0 <= int(view0) and int(n_views) >= 1 and int(view0) + int(n_views) <= geo.n_projections,
          "view range lies outside the geometry")
    out = _out_tensor(out, (n_views, geo.detector.n_v, geo.detector.n_u), vol, "projection buffer")
    N.check(N.lib().tg_cone_forward_views(geo._plan(_dev(vol)), int(view0), int(n_views),
                                          vol.data_ptr(), out.data_ptr(), stream_of(vol)))
    return out


def cone_slab_rows(geo: ConeGeometry, z0: int, nz: int, device: int = 0):
    """Detector rows [v0, v0 + n_rows) a z-slab projects onto (every view)."""
    v0, nr = C.c_uint64(), C.c_uint64()
    N.check(N.lib().tg_cone_slab_rows(geo._plan(device), int(z0), int(nz), C.byref(v0), C.byref(nr)))
    return int(v0.value), int(nr.value)


def cone_backproject_slab(geo: ConeGeometry, band: torch.Tensor, z0: int, nz: int, v0: int,
                          out: torch.Tensor = None, scale: float = 1.0,
                          accumulate: bool = False) -> torch.Tensor:
    """K1 on a z-slab [z0, z0 + nz) from a detector row band [v0, v0 + rows)."""
    band = require_f32(band, "row band")
    check(band.dim() == 3, "row band does not match the geometry")
    n_rows = band.shape[1]
    _check_shape(band, (geo.n_projections, n_rows, geo.detector.n_u), "row band")
    check(0 <= int(v0) and n_rows >= 1 and int(v0) + n_rows <= geo.detector.n_v,
          "detector row band lies outside the detector")
    nzv = geo.volume.shape[2]
    check(0 <= int(z0) and int(nz) >= 1 and int(z0) + int(nz) <= nzv,
          "z-slab lies outside the volume")
    out = _out_tensor(out, (nz, geo.volume.shape[1], geo.volume.shape[0]), band, "slab buffer")
    N.check(N.lib().tg_cone_backproject_slab(geo._plan(_dev(band)), int(z0), int(nz), int(v0),
                                             int(n_rows), band.data_ptr(), out.data_ptr(),
                                             float(scale), int(bool(accumulate)), stream_of(band)))
    return out


# ---- diagnostics -------------------------------------------------------------


def ray_sample_counts(geo, view0: int = 0, n_views: int = None, device: int = 0) -> torch.Tensor:
    """Per-ray sample counts n = ceil((t1 - t0) / step) the forward projector
    marches (projector.hpp:117,138; 0 = the ray misses the volume), computed by
    the device's own FP64 ray setup and clip (K2 / K5 / K7 prologue).  Cone:
    int64 [n_views][n_v][n_u]; planar: int64 [n_proj][n_bins]."""
    L = N.lib()
    dev = torch.device("cuda", device)
    st = torch.cuda.current_stream(dev).cuda_stream
    if isinstance(geo, ConeGeometry):
        n_views = geo.n_projections - int(view0) if n_views is None else int(n_views)
        check(0 <= int(view0) and n_views >= 1 and int(view0) + n_views <= geo.n_projections,
              "view range lies outside the geometry")
        out = torch.empty((n_views, geo.detector.n_v, geo.detector.n_u), dtype=torch.int64,
                          device=dev)
        N.check(L.tg_cone_ray_samples(geo._plan(device), int(view0), n_views, out.data_ptr(), st))
        return out
    check(isinstance(geo, (ParallelGeometry, FanGeometry)), "unknown geometry type")
    out = torch.empty((geo.n_projections, geo.detector.n_bins), dtype=torch.int64, device=dev)
    N.check(L.tg_planar_ray_samples(geo._plan(device), out.data_ptr(), st))
    return out


def set_cone_knob(geo: ConeGeometry, name: str, value: int, device: int = 0) -> None:
    """Plan knobs for experiments and tests (results are unchanged bit for bit):
    "k2_tu" 32 / 64 (K2 CTA width: 8- or 4-row detector bands), "k2_dual" 0 / 1
    (the y-fastest quad volume for x-dominant rays)."""
    N.check(N.lib().tg_cone_plan_set_knob(geo._plan(device), name.encode(), int(value)))
