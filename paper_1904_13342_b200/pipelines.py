"""FDK / FBP compositions (pipelines.hpp:41-84) on the device path.

fdk_reconstruct runs K3 (cosine x Parker weights fused into the Ram-Lak FFT
row filter) then K1 (back-projection with the FDK constant fused into the
epilogue); fbp_reconstruct runs K3 then K6 with pi/n fused.
"""
from __future__ import annotations

import math
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .containers import Image, Sinogram, is_host, require_f32, stream_of
from .filtering import Filter1D, apply_filter, ramlak_filter, ramp_filter
from .geometry import ConeGeometry, ParallelGeometry, check
from .projector import _check_cone_sino, _dev, back_project


class FilterKind(Enum):
    ramp = 0
    ramlak = 1


def make_filter(kind: FilterKind, n_bins: int, spacing: float, padded_n: int = 0) -> Filter1D:
    """pipelines.hpp:43-47"""
    return (ramp_filter if kind == FilterKind.ramp else ramlak_filter)(n_bins, spacing, padded_n)


def fbp_reconstruct(sino: Sinogram, geo: ParallelGeometry, filt=FilterKind.ramlak) -> Image:
    """pipelines.hpp:49-63: BP(filter(p)) * pi / n"""
    if isinstance(filt, FilterKind):
        filt = make_filter(filt, geo.detector.n_bins, geo.detector.spacing)
    if is_host(sino.data):
        # host buffers: one upload, K3 + K6 (pi/n fused) on the device, one download
        data = torch.from_numpy(np.ascontiguousarray(require_f32(sino.data, "sinogram data")))
        dev_sino = Sinogram(sino.n_projections, detector1d=sino.detector1d, cone=False,
                            data=data.to(torch.device("cuda", 0)))
        img = fbp_reconstruct(dev_sino, geo, filt)
        return Image(geo.volume, img.data.cpu().numpy())
    filtered = apply_filter(sino, filt)
    c = math.pi / float(geo.n_projections)
    return back_project(filtered, geo, scale=c)


def fdk_scale(geo: ConeGeometry, use_parker: bool = True) -> float:
    """pipelines.hpp:80-81"""
    return geo.angular_range / float(geo.n_projections) * (geo.sdd / geo.sid) * (
        1.0 if use_parker else 0.5)


def fdk_reconstruct(sino: Sinogram, geo: ConeGeometry, use_parker: bool = True,
                    work: torch.Tensor = None) -> Image:
    """pipelines.hpp:73-84: cosine, optional Parker, row-wise Ram-Lak, 1/w^2
    back-projection, times (range/n)(SDD/SID)(parker ? 1 : 1/2)."""
    _check_cone_sino(sino, geo)
    data = require_f32(sino.data, "sinogram data")
    L = N.lib()
    if is_host(data):
        out = np.zeros(geo.volume.torch_shape, np.float32)
        N.check(L.tg_cone_fdk_host(geo._plan(0), data.ctypes.data, out.ctypes.data,
                                   int(bool(use_parker))))
        return Image(geo.volume, out)
    if work is None:
        work = torch.empty_like(data)
    out = torch.empty(geo.volume.torch_shape, dtype=torch.float32, device=data.device)
    N.check(L.tg_cone_fdk(geo._plan(_dev(data)), data.data_ptr(), out.data_ptr(), work.data_ptr(),
                          int(bool(use_parker)), stream_of(data)))
    return Image(geo.volume, out)


def fdk_prefilter(sino: torch.Tensor, geo: ConeGeometry, use_parker: bool = True, v0: int = 0,
                  out: torch.Tensor = None) -> torch.Tensor:
    """K3 alone on detector rows [v0, v0 + rows) of every view (a z-slab's band)."""
    sino = require_f32(sino, "sinogram rows")
    check(sino.dim() == 3 and sino.shape[0] == geo.n_projections
          and sino.shape[2] == geo.detector.n_u, "sinogram shape does not match the geometry")
    if out is None:
        out = torch.empty_like(sino)
    N.check(N.lib().tg_cone_fdk_prefilter(geo._plan(_dev(sino)), sino.data_ptr(), out.data_ptr(),
                                          int(bool(use_parker)), int(v0), int(sino.shape[1]),
                                          stream_of(sino)))
    return out
