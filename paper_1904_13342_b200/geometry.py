"""Containers and acquisition geometries, mirroring the reference's
image.hpp / geometry.hpp API (names, fields, argument meaning, error text).

Every double the geometry holds is produced by the library's host geometry
(csrc/host_geometry.cpp) through the C ABI, which is bit-exact with the
reference; nothing here recomputes geometry in Python.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import Error

PI = math.pi


def check(cond: bool, msg: str) -> None:
    """core.hpp:24-26"""
    if not cond:
        raise Error(msg)


@dataclass
class VolumeSpec:
    """image.hpp:18-54.  shape/spacing/origin in world-axis order (x, y[, z]);
    memory is x-fastest, so a 3D tensor is indexed [z][y][x]."""
    shape: List[int]
    spacing: List[float]
    origin: List[float] = field(default_factory=list)

    @staticmethod
    def centered(shape: Sequence[int], spacing: Sequence[float]) -> "VolumeSpec":
        s = VolumeSpec([int(v) for v in shape], [float(v) for v in spacing], [])
        s.validate_shape()
        s.origin = [-0.5 * float(n - 1) * d for n, d in zip(s.shape, s.spacing)]
        return s

    def validate_shape(self) -> None:
        check(len(self.shape) in (2, 3), "volume must be 2D or 3D")
        check(len(self.spacing) == len(self.shape), "spacing rank mismatch")
        for n in self.shape:
            check(n >= 1, "volume shape entries must be >= 1")
        for d in self.spacing:
            check(d > 0.0, "volume spacing must be positive")

    def validate(self) -> None:
        self.validate_shape()
        check(len(self.origin) == len(self.shape), "origin rank mismatch")

    def dims(self) -> int:
        return len(self.shape)

    def element_count(self) -> int:
        return int(np.prod(self.shape))

    def extent(self, a: int) -> float:
        return float(self.shape[a]) * self.spacing[a]

    @property
    def torch_shape(self):
        """tensor shape of the x-fastest layout: (nz, ny, nx) or (ny, nx)"""
        return tuple(reversed(self.shape))

    def c(self) -> N.tg_volume_spec:
        v = N.tg_volume_spec()
        v.dims = len(self.shape)
        for a in range(len(self.shape)):
            v.shape[a] = int(self.shape[a])
            v.spacing[a] = float(self.spacing[a])
            v.origin[a] = float(self.origin[a]) if a < len(self.origin) else 0.0
        return v


@dataclass
class Detector1D:
    """image.hpp:57-67"""
    n_bins: int = 0
    spacing: float = 1.0
    origin: float = 0.0

    @staticmethod
    def centered(n: int, spacing: float) -> "Detector1D":
        check(n >= 1, "detector needs at least one bin")
        check(spacing > 0.0, "detector spacing must be positive")
        return Detector1D(int(n), float(spacing), -0.5 * float(n - 1) * float(spacing))

    def c(self) -> N.tg_detector1d:
        return N.tg_detector1d(int(self.n_bins), float(self.spacing), float(self.origin))


@dataclass
class Detector2D:
    """image.hpp:70-81 (u = columns, fastest in memory; v = rows)"""
    n_u: int = 0
    n_v: int = 0
    spacing_u: float = 1.0
    spacing_v: float = 1.0
    origin_u: float = 0.0
    origin_v: float = 0.0

    @staticmethod
    def centered(n_u: int, n_v: int, du: float, dv: float) -> "Detector2D":
        check(n_u >= 1 and n_v >= 1, "detector needs at least one pixel per axis")
        check(du > 0.0 and dv > 0.0, "detector spacing must be positive")
        return Detector2D(int(n_u), int(n_v), float(du), float(dv), -0.5 * float(n_u - 1) * du,
                          -0.5 * float(n_v - 1) * dv)

    def c(self) -> N.tg_detector2d:
        return N.tg_detector2d(int(self.n_u), int(self.n_v), float(self.spacing_u),
                               float(self.spacing_v), float(self.origin_u), float(self.origin_v))


def view_angles(n_projections: int, angular_range: float) -> np.ndarray:
    """geometry.hpp:30-39"""
    out = np.zeros(max(int(n_projections), 1))
    N.check(N.lib().tg_view_angles(int(n_projections), float(angular_range), N.dptr(out)))
    return out[: int(n_projections)]


class _PlanHolder:
    """Caches one device plan per geometry and device; frees it with the geometry."""

    _destroy_name = ""

    def __init__(self):
        self._plans = {}

    def _plan(self, device: int):
        p = self._plans.get(device)
        if p is None:
            p = self._create_plan(device)
            self._plans[device] = p
        return p

    def invalidate(self):
        plans, self._plans = self._plans, {}
        for p in plans.values():
            getattr(N.lib(), self._destroy_name)(p)

    def __del__(self):
        try:
            self.invalidate()
        except Exception:
            pass


class _Planar(_PlanHolder):
    _destroy_name = "tg_planar_plan_destroy"

    def __init__(self, volume, detector, n_projections, angular_range, sid, sdd, rays, angles):
        super().__init__()
        self.volume = volume
        self.detector = detector
        self.n_projections = int(n_projections)
        self.angular_range = float(angular_range)
        self.sid = float(sid)
        self.sdd = float(sdd)
        self.rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 2)
        self.angles = np.ascontiguousarray(angles, dtype=np.float64)

    def ray(self, i):
        return self.rays[i]

    def detector_axis(self, i):
        r = self.rays[i]
        return np.array([-r[1], r[0]])

    def c(self) -> N.tg_planar_geometry:
        self._keep = (self.rays, self.angles)
        return N.tg_planar_geometry(self.volume.c(), self.detector.c(), self.n_projections,
                                    self.angular_range, self.sid, self.sdd, N.dptr(self.rays),
                                    N.dptr(self.angles))

    def _create_plan(self, device):
        h = C.c_void_p()
        g = self.c()
        N.check(N.lib().tg_planar_plan_create(C.byref(g), int(device), C.byref(h)))
        return h

    def set_custom_rays(self, r):
        """geometry.hpp:62-70"""
        r = np.asarray(r, dtype=np.float64).reshape(-1, 2)
        check(len(r) == self.n_projections, "ray count must match projection count")
        for v in r:
            check(abs(math.hypot(v[0], v[1]) - 1.0) <= 1e-9, "trajectory rays must be unit length")
        self.angles = np.array([math.atan2(v[1], v[0]) for v in r])
        self.rays = np.ascontiguousarray(r)
        self.invalidate()


class ParallelGeometry(_Planar):
    """geometry.hpp:50-71"""

    def __init__(self, volume, detector, n_projections, angular_range, rays, angles):
        super().__init__(volume, detector, n_projections, angular_range, 0.0, 0.0, rays, angles)


class FanGeometry(_Planar):
    """geometry.hpp:88-106"""

    def source(self, i):
        return -self.sid * self.rays[i]

    def fan_half_angle(self) -> float:
        return math.atan(0.5 * float(self.detector.n_bins) * self.detector.spacing / self.sdd)


def _make_planar(volume: VolumeSpec, detector: Detector1D, n, rng, sid, sdd):
    n = int(n)
    rays = np.zeros((max(n, 1), 2))
    ang = np.zeros(max(n, 1))
    v, d = volume.c(), detector.c()
    N.check(N.lib().tg_make_planar(C.byref(v), C.byref(d), n, float(rng), float(sid), float(sdd),
                                   N.dptr(rays), N.dptr(ang)))
    return rays[:n], ang[:n]


def make_parallel(volume: VolumeSpec, detector: Detector1D, n_projections: int,
                  angular_range: float) -> ParallelGeometry:
    """geometry.hpp:73-86"""
    volume.validate()
    rays, ang = _make_planar(volume, detector, n_projections, angular_range, 0.0, 0.0)
    return ParallelGeometry(volume, detector, n_projections, angular_range, rays, ang)


def make_fan(volume: VolumeSpec, detector: Detector1D, n_projections: int, angular_range: float,
             sid: float, sdd: float) -> FanGeometry:
    """geometry.hpp:108-124"""
    volume.validate()
    check(volume.dims() == 2, "fan beam geometry expects a 2D volume")
    check(sid > 0.0 and sdd > sid, "fan beam requires 0 < SID < SDD")
    rays, ang = _make_planar(volume, detector, n_projections, angular_range, sid, sdd)
    return FanGeometry(volume, detector, n_projections, angular_range, sid, sdd, rays, ang)


class ConeGeometry(_PlanHolder):
    """geometry.hpp:126-178.  matrices (n, 12) are normalised so the
    iso-centre's homogeneous depth equals SID; sources (n, 3); inv_blocks
    (n, 9); angles (n,) measured from the first view."""
    _destroy_name = "tg_cone_plan_destroy"

    def __init__(self, volume, detector, n_projections, angular_range, sid, sdd):
        super().__init__()
        self.volume = volume
        self.detector = detector
        self.n_projections = int(n_projections)
        self.angular_range = float(angular_range)
        self.sid = float(sid)
        self.sdd = float(sdd)
        self.angles = np.zeros(0)
        self.matrices = np.zeros((0, 12))
        self.sources = np.zeros((0, 3))
        self.inv_blocks = np.zeros((0, 9))

    def fan_half_angle(self) -> float:
        return math.atan(0.5 * float(self.detector.n_u) * self.detector.spacing_u / self.sdd)

    def set_matrices(self, mats) -> None:
        """geometry.hpp:144-177"""
        mats = np.ascontiguousarray(mats, dtype=np.float64).reshape(-1, 12)
        check(len(mats) == self.n_projections, "matrix count must match projection count")
        n = len(mats)
        out = np.zeros_like(mats)
        src = np.zeros((n, 3))
        inv = np.zeros((n, 9))
        ang = np.zeros(n)
        N.check(N.lib().tg_cone_set_matrices(n, self.sid, N.dptr(mats), N.dptr(out), N.dptr(src),
                                             N.dptr(inv), N.dptr(ang)))
        self.matrices, self.sources, self.inv_blocks, self.angles = out, src, inv, ang
        self.invalidate()

    @property
    def circular(self) -> bool:
        return bool(np.all(self.matrices[:, 2] == 0.0) and np.all(self.matrices[:, 10] == 0.0))

    def c(self) -> N.tg_cone_geometry:
        self._keep = (self.matrices, self.sources, self.inv_blocks, self.angles)
        return N.tg_cone_geometry(self.volume.c(), self.detector.c(), self.n_projections,
                                  self.angular_range, self.sid, self.sdd, N.dptr(self.matrices),
                                  N.dptr(self.sources), N.dptr(self.inv_blocks),
                                  N.dptr(self.angles))

    def _create_plan(self, device):
        h = C.c_void_p()
        g = self.c()
        N.check(N.lib().tg_cone_plan_create(C.byref(g), int(device), C.byref(h)))
        return h


def cone_projection_matrix(theta: float, sid: float, sdd: float, det: Detector2D) -> np.ndarray:
    """geometry.hpp:181-194"""
    out = np.zeros(12)
    d = det.c()
    N.check(N.lib().tg_cone_projection_matrix(float(theta), float(sid), float(sdd), C.byref(d),
                                              N.dptr(out)))
    return out


def projection_matrices_circular(n_projections, angular_range, sid, sdd, det) -> np.ndarray:
    """geometry.hpp:196-204"""
    check(sid > 0.0 and sdd > sid, "cone beam requires 0 < SID < SDD")
    return np.stack([cone_projection_matrix(t, sid, sdd, det)
                     for t in view_angles(n_projections, angular_range)])


def make_cone(volume: VolumeSpec, detector: Detector2D, n_projections: int, angular_range: float,
              sid: float, sdd: float) -> ConeGeometry:
    """geometry.hpp:206-223"""
    volume.validate()
    n = int(n_projections)
    g = ConeGeometry(volume, detector, n, angular_range, sid, sdd)
    mats = np.zeros((max(n, 1), 12))
    src = np.zeros((max(n, 1), 3))
    inv = np.zeros((max(n, 1), 9))
    ang = np.zeros(max(n, 1))
    v, d = volume.c(), detector.c()
    N.check(N.lib().tg_make_cone(C.byref(v), C.byref(d), n, float(angular_range), float(sid),
                                 float(sdd), N.dptr(mats), N.dptr(src), N.dptr(inv), N.dptr(ang)))
    g.matrices, g.sources, g.inv_blocks, g.angles = mats[:n], src[:n], inv[:n], ang[:n]
    return g


def make_cone_from_matrices(volume: VolumeSpec, detector: Detector2D, angular_range: float,
                            sid: float, sdd: float, mats) -> ConeGeometry:
    """geometry.hpp:226-242"""
    volume.validate()
    check(volume.dims() == 3, "cone beam geometry expects a 3D volume")
    check(sid > 0.0 and sdd > sid, "cone beam requires 0 < SID < SDD")
    mats = np.asarray(mats, dtype=np.float64).reshape(-1, 12)
    check(len(mats) > 0, "need at least one projection matrix")
    g = ConeGeometry(volume, detector, len(mats), angular_range, sid, sdd)
    g.set_matrices(mats)
    return g


Geometry = Optional[object]
