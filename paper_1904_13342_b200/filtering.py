"""Reconstruction filters and projection weight maps (filtering.hpp:27-251).

Host-side weight vectors/maps are produced by the library's bit-exact host
code; applying them to device data runs the K3 row filter (FFT, fp32) and the
weight kernels.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import _native as N
from .containers import Sinogram, is_host, require_f32, stream_of
from .geometry import ConeGeometry, FanGeometry, check


def is_pow2(n: int) -> bool:
    return n != 0 and (n & (n - 1)) == 0


def next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p <<= 1
    return p


@dataclass
class Filter1D:
    """filtering.hpp:27-32"""
    n_bins: int = 0
    padded_n: int = 0
    spacing: float = 1.0
    weights: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __post_init__(self):
        self.weights = np.ascontiguousarray(self.weights, dtype=np.float64)
        self._plans = {}

    def _plan(self, row_len: int, row_spacing: float, device: int):
        key = (row_len, row_spacing, device)
        p = self._plans.get(key)
        if p is None:
            h = C.c_void_p()
            N.check(N.lib().tg_filter_plan_create(int(row_len), float(row_spacing), int(self.n_bins),
                                                  int(self.padded_n), float(self.spacing),
                                                  N.dptr(self.weights), len(self.weights),
                                                  int(device), C.byref(h)))
            p = h
            self._plans[key] = p
        return p

    def __del__(self):
        try:
            for p in self._plans.values():
                N.lib().tg_filter_plan_destroy(p)
        except Exception:
            pass


def filter_window(n_bins: int) -> int:
    """filtering.hpp:34-37"""
    check(n_bins >= 1, "filter needs at least one detector bin")
    return int(N.lib().tg_filter_window(int(n_bins)))


def ramp_weights(padded_n: int, spacing: float) -> np.ndarray:
    """filtering.hpp:40-50"""
    w = np.zeros(max(int(padded_n), 1))
    N.check(N.lib().tg_ramp_weights(int(padded_n), float(spacing), N.dptr(w)))
    return w[: int(padded_n)]


def ramp_filter(n_bins: int, spacing: float, padded_n: int = 0) -> Filter1D:
    """filtering.hpp:52-57"""
    padded = padded_n if padded_n else filter_window(n_bins)
    check(padded >= n_bins, "filter window is smaller than the detector row")
    return Filter1D(n_bins, padded, spacing, ramp_weights(padded, spacing))


def ramlak_spatial(m: int, spacing: float) -> float:
    """filtering.hpp:60-65"""
    if m == 0:
        return 1.0 / (4.0 * spacing * spacing)
    if m % 2 == 0:
        return 0.0
    mpi = float(m) * math.pi * spacing
    return -1.0 / (mpi * mpi)


def ramlak_weights(padded_n: int, spacing: float) -> np.ndarray:
    """filtering.hpp:68-82"""
    w = np.zeros(max(int(padded_n), 1))
    N.check(N.lib().tg_ramlak_weights(int(padded_n), float(spacing), N.dptr(w)))
    return w[: int(padded_n)]


def ramlak_filter(n_bins: int, spacing: float, padded_n: int = 0) -> Filter1D:
    """filtering.hpp:84-89"""
    padded = padded_n if padded_n else filter_window(n_bins)
    check(padded >= n_bins, "filter window is smaller than the detector row")
    return Filter1D(n_bins, padded, spacing, ramlak_weights(padded, spacing))


def apply_filter(sino: Sinogram, filt: Filter1D) -> Sinogram:
    """filtering.hpp:115-125: filter every detector row (cone data along u)."""
    cone = sino.is_cone()
    n = sino.detector2d.n_u if cone else sino.detector1d.n_bins
    ds = sino.detector2d.spacing_u if cone else sino.detector1d.spacing
    data = require_f32(sino.data, "sinogram data")
    rows = data.size // n if is_host(data) else data.numel() // n
    if is_host(data):
        out = np.empty_like(data)
        N.check(N.lib().tg_filter_apply_host(filt._plan(n, ds, 0), data.ctypes.data,
                                             out.ctypes.data, rows))
    else:
        out = torch.empty_like(data)
        dev = data.device.index or 0
        N.check(N.lib().tg_filter_apply(filt._plan(n, ds, dev), data.data_ptr(), out.data_ptr(),
                                        rows, stream_of(data)))
    return Sinogram(sino.n_projections, sino.detector1d, sino.detector2d, sino.cone, out)


@dataclass
class WeightMap:
    """filtering.hpp:131-134.  ``shape`` fastest-first; equals the sinogram
    shape (per element) or the detector shape (broadcast over views).  A cone
    Parker map keeps one u-profile per view in ``row_profile`` ([views][n_u])
    and materialises ``data`` only on request (it is identical on every row,
    filtering.hpp:246-247)."""
    shape: List[int]
    data: np.ndarray = None
    row_profile: np.ndarray = None

    def full(self) -> np.ndarray:
        if self.data is None and self.row_profile is not None:
            nu, nv, npj = self.shape
            self.data = np.repeat(self.row_profile[:, None, :], nv, axis=1).reshape(-1)
        return self.data


def cosine_weights(geo) -> WeightMap:
    """filtering.hpp:157-181"""
    if isinstance(geo, ConeGeometry):
        out = np.zeros(geo.detector.n_u * geo.detector.n_v)
        g = geo.c()
        N.check(N.lib().tg_cosine_weights_cone(C.byref(g), N.dptr(out)))
        return WeightMap([geo.detector.n_u, geo.detector.n_v], out)
    check(isinstance(geo, FanGeometry), "cosine weights need a fan or cone geometry")
    out = np.zeros(geo.detector.n_bins)
    g = geo.c()
    N.check(N.lib().tg_cosine_weights_fan(C.byref(g), N.dptr(out)))
    return WeightMap([geo.detector.n_bins], out)


def parker_weights(geo) -> WeightMap:
    """filtering.hpp:215-251"""
    if isinstance(geo, ConeGeometry):
        out = np.zeros((geo.n_projections, geo.detector.n_u))
        g = geo.c()
        N.check(N.lib().tg_parker_weights_cone(C.byref(g), N.dptr(out)))
        return WeightMap([geo.detector.n_u, geo.detector.n_v, geo.n_projections], None, out)
    check(isinstance(geo, FanGeometry), "redundancy weights need a fan or cone geometry")
    out = np.zeros((geo.n_projections, geo.detector.n_bins))
    g = geo.c()
    N.check(N.lib().tg_parker_weights_fan(C.byref(g), N.dptr(out)))
    return WeightMap([geo.detector.n_bins, geo.n_projections], out.reshape(-1))


def apply_weights(sino: Sinogram, wmap: WeightMap) -> Sinogram:
    """filtering.hpp:136-154: out = T(double(x) * w), per element or broadcast."""
    ss = list(sino.shape())
    data = require_f32(sino.data, "sinogram data")
    host = is_host(data)
    dev_data = torch.from_numpy(data).cuda() if host else data
    out = torch.empty_like(dev_data)
    st = stream_of(dev_data)
    L = N.lib()
    if list(wmap.shape) == ss:
        if wmap.row_profile is not None and sino.is_cone():
            m = torch.from_numpy(np.ascontiguousarray(wmap.row_profile)).to(dev_data.device)
            N.check(L.tg_apply_row_weights(dev_data.data_ptr(), out.data_ptr(), sino.n_projections,
                                           sino.detector2d.n_v, sino.detector2d.n_u, m.data_ptr(),
                                           st))
        else:
            m = torch.from_numpy(np.ascontiguousarray(wmap.full())).to(dev_data.device)
            N.check(L.tg_apply_weights(dev_data.data_ptr(), out.data_ptr(), out.numel(),
                                       m.data_ptr(), m.numel(), st))
    else:
        check(list(wmap.shape) == ss[:-1],
              "weight map shape matches neither the sinogram nor its detector")
        m = torch.from_numpy(np.ascontiguousarray(wmap.data)).to(dev_data.device)
        N.check(L.tg_apply_weights(dev_data.data_ptr(), out.data_ptr(), out.numel(), m.data_ptr(),
                                   m.numel(), st))
    if host:
        out = out.cpu().numpy()
    return Sinogram(sino.n_projections, sino.detector1d, sino.detector2d, sino.cone, out)
