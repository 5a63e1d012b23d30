"""Image / Sinogram containers (image.hpp:83-166) over device or host data.

``data`` is either a CUDA float32 torch tensor (the device path; operators
run on the tensor's device and the caller's current stream) or a float32
numpy array (host path: the operator copies in and out through the C ABI's
*_host entry points, the reference's by-value semantics).  Layouts are the
reference's: volumes [z][y][x] (x fastest), cone sinograms [view][v][u],
planar sinograms [view][bin].
"""
from __future__ import annotations

from typing import Union

import numpy as np
import torch

from .geometry import Detector1D, Detector2D, VolumeSpec, check

Array = Union[torch.Tensor, np.ndarray]


def _zeros(shape, like=None, device=None):
    if isinstance(like, np.ndarray):
        return np.zeros(shape, dtype=np.float32)
    if device is None:
        device = like.device if isinstance(like, torch.Tensor) else torch.device("cuda")
    return torch.zeros(shape, dtype=torch.float32, device=device)


class Image:
    """image.hpp:83-114"""

    def __init__(self, spec: VolumeSpec, data: Array = None, device=None, host: bool = False):
        spec.validate()
        self.spec = spec
        if data is None:
            data = np.zeros(spec.torch_shape, np.float32) if host else _zeros(spec.torch_shape,
                                                                               device=device)
        check(tuple(data.shape) == tuple(spec.torch_shape), "image data does not match its spec")
        self.data = data

    def dims(self):
        return self.spec.dims()

    def nx(self):
        return self.spec.shape[0]

    def ny(self):
        return self.spec.shape[1]

    def nz(self):
        return self.spec.shape[2] if self.spec.dims() == 3 else 1

    def coord(self, a: int, idx: int) -> float:
        return self.spec.origin[a] + float(idx) * self.spec.spacing[a]


class Sinogram:
    """image.hpp:118-166.  Planar data (n_projections, n_bins); cone data
    (n_projections, n_v, n_u)."""

    def __init__(self, n_projections: int, detector1d: Detector1D = None,
                 detector2d: Detector2D = None, cone: bool = False, data: Array = None):
        self.n_projections = int(n_projections)
        self.detector1d = detector1d or Detector1D()
        self.detector2d = detector2d or Detector2D()
        self.cone = bool(cone)
        if data is not None:
            want = ((self.n_projections, int(self.detector2d.n_v), int(self.detector2d.n_u))
                    if self.cone else (self.n_projections, int(self.detector1d.n_bins)))
            check(tuple(data.shape) == want, "sinogram data does not match its detector")
        self.data = data

    @staticmethod
    def planar(n_proj: int, det: Detector1D, data: Array = None, device=None, host=False):
        check(n_proj >= 1, "need at least one projection")
        shape = (int(n_proj), int(det.n_bins))
        if data is None:
            data = np.zeros(shape, np.float32) if host else _zeros(shape, device=device)
        return Sinogram(n_proj, detector1d=det, cone=False, data=data)

    @staticmethod
    def cone_beam(n_proj: int, det: Detector2D, data: Array = None, device=None, host=False):
        check(n_proj >= 1, "need at least one projection")
        shape = (int(n_proj), int(det.n_v), int(det.n_u))
        if data is None:
            data = np.zeros(shape, np.float32) if host else _zeros(shape, device=device)
        return Sinogram(n_proj, detector2d=det, cone=True, data=data)

    def is_cone(self) -> bool:
        return self.cone

    def n_bins(self) -> int:
        return self.detector1d.n_bins

    def shape(self):
        """fastest axis first, like VolumeSpec.shape (image.hpp:159-163)"""
        if self.cone:
            return [self.detector2d.n_u, self.detector2d.n_v, self.n_projections]
        return [self.detector1d.n_bins, self.n_projections]


def is_host(a: Array) -> bool:
    return isinstance(a, np.ndarray)


def require_f32(a: Array, what: str):
    if isinstance(a, np.ndarray):
        check(a.dtype == np.float32, f"{what} must be float32")
        return np.ascontiguousarray(a)
    check(isinstance(a, torch.Tensor), f"{what} must be a torch tensor or numpy array")
    check(a.dtype == torch.float32, f"{what} must be float32")
    check(a.is_cuda, f"{what} must live on a CUDA device (the B200 path has no CPU fallback)")
    return a.contiguous()


def stream_of(t: torch.Tensor):
    return torch.cuda.current_stream(t.device).cuda_stream
