"""Analytic phantoms rasterised on the GPU (phantom.hpp:34-147), bit-exact
with the reference's FP64 rasterisation (csrc/phantom.cu)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .containers import Image
from .geometry import VolumeSpec, check


def head_phantom_ellipsoids(spec: VolumeSpec) -> np.ndarray:
    """phantom.hpp:107-122 scaled by fov_half_extent (phantom.hpp:124-128): (10, 8)"""
    out = np.zeros((10, 8))
    v = spec.c()
    N.check(N.lib().tg_head_phantom_ellipsoids(C.byref(v), N.dptr(out)))
    return out


def head_phantom_ellipses(spec: VolumeSpec) -> np.ndarray:
    """phantom.hpp:91-105: (10, 6)"""
    out = np.zeros((10, 6))
    v = spec.c()
    N.check(N.lib().tg_head_phantom_ellipses(C.byref(v), N.dptr(out)))
    return out


def rasterize(specs, spec: VolumeSpec, device=None, stream=None) -> Image:
    """phantom.hpp:34-88.  specs: (n, 8) ellipsoids {cx,cy,cz,a,b,c,phi_deg,I}
    for a 3D spec, (n, 6) ellipses {cx,cy,a,b,phi_deg,I} for a 2D spec."""
    spec.validate()
    specs = np.ascontiguousarray(specs, dtype=np.float64)
    device = torch.device("cuda") if device is None else torch.device(device)
    out = torch.empty(spec.torch_shape, dtype=torch.float32, device=device)
    st = torch.cuda.current_stream(out.device).cuda_stream if stream is None else stream
    v = spec.c()
    if spec.dims() == 3:
        specs = specs.reshape(-1, 8)
        N.check(N.lib().tg_rasterize_ellipsoids(C.byref(v), N.dptr(specs), len(specs),
                                                out.data_ptr(), st))
    else:
        specs = specs.reshape(-1, 6)
        N.check(N.lib().tg_rasterize_ellipses(C.byref(v), N.dptr(specs), len(specs),
                                              out.data_ptr(), st))
    return Image(spec, out)


def shepp_logan_3d(spec: VolumeSpec, device=None) -> Image:
    """phantom.hpp:136-140"""
    check(spec.dims() == 3, "3D head phantom needs a 3D volume")
    return rasterize(head_phantom_ellipsoids(spec), spec, device)


def shepp_logan_2d(spec: VolumeSpec, device=None) -> Image:
    """phantom.hpp:130-134"""
    check(spec.dims() == 2, "2D head phantom needs a 2D volume")
    return rasterize(head_phantom_ellipses(spec), spec, device)


def disk_phantom(spec: VolumeSpec, radius: float, intensity: float, device=None) -> Image:
    """phantom.hpp:142-147"""
    check(radius > 0.0, "disk radius must be positive")
    return rasterize(np.array([[0.0, 0.0, radius, radius, 0.0, intensity]]), spec, device)
