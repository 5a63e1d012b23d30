"""CPU ORACLE bindings (TEST INFRASTRUCTURE ONLY).

ctypes access to
  * ``oracle/liboracle.so``            — the C restatement (tg_oracle.c), and
  * ``oracle/_ref/libtomograd_ref.so`` — the reference's own headers compiled
    by ``oracle/Makefile`` (ref_capi.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
reported CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtomograd_ref.so")


class OracleError(RuntimeError):
    pass


class or_volume(C.Structure):
    _fields_ = [("dims", C.c_uint32), ("shape", C.c_uint64 * 3),
                ("spacing", C.c_double * 3), ("origin", C.c_double * 3)]


class or_det1(C.Structure):
    _fields_ = [("n_bins", C.c_uint64), ("spacing", C.c_double), ("origin", C.c_double)]


class or_det2(C.Structure):
    _fields_ = [("n_u", C.c_uint64), ("n_v", C.c_uint64), ("spacing_u", C.c_double),
                ("spacing_v", C.c_double), ("origin_u", C.c_double), ("origin_v", C.c_double)]


_dp = C.POINTER(C.c_double)


class or_planar(C.Structure):
    _fields_ = [("vol", or_volume), ("det", or_det1), ("n_proj", C.c_uint64),
                ("range", C.c_double), ("sid", C.c_double), ("sdd", C.c_double),
                ("rays", _dp), ("angles", _dp)]


class or_cone(C.Structure):
    _fields_ = [("vol", or_volume), ("det", or_det2), ("n_proj", C.c_uint64),
                ("range", C.c_double), ("sid", C.c_double), ("sdd", C.c_double),
                ("mats", _dp), ("sources", _dp), ("invs", _dp), ("angles", _dp)]


def _ptr(a: np.ndarray, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OracleError(f"{LIB_PATH} missing: run `make -C oracle`")
        _lib = C.CDLL(LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
        _lib.or_filter_window.restype = C.c_uint64
        _lib.or_filter_window.argtypes = [C.c_uint64]
        _lib.or_ramlak_spatial.restype = C.c_double
        _lib.or_ramlak_spatial.argtypes = [C.c_long, C.c_double]
        _lib.or_parker_weight.restype = C.c_double
        _lib.or_parker_weight.argtypes = [C.c_double] * 4
        _lib.or_fov_half_extent.restype = C.c_double
        _lib.or_ramp_weights.argtypes = [C.c_uint64, C.c_double, _dp]
        _lib.or_ramlak_weights.argtypes = [C.c_uint64, C.c_double, _dp]
        _lib.or_view_angles.argtypes = [C.c_uint64, C.c_double, _dp]
        _lib.or_circular_rays_2d.argtypes = [C.c_uint64, C.c_double, _dp]
        _lib.or_make_cone.argtypes = [C.POINTER(or_det2), C.c_uint64, C.c_double, C.c_double,
                                      C.c_double, _dp, _dp, _dp, _dp]
        _lib.or_cone_set_matrices.argtypes = [C.c_uint64, C.c_double, _dp, _dp, _dp, _dp, _dp]
        _lib.or_cone_projection_matrix.argtypes = [C.c_double, C.c_double, C.c_double,
                                                   C.POINTER(or_det2), _dp]
        _lib.or_head_ellipsoids.argtypes = [C.c_double, _dp]
        _lib.or_head_ellipses.argtypes = [C.c_double, _dp]
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise OracleError(f"{REF_PATH} missing: build it with `make -C oracle` where "
                              "/root/reference is mounted")
        _ref = C.CDLL(REF_PATH)
        _ref.ref_last_error.restype = C.c_char_p
        _ref.ref_num_threads.restype = C.c_int
    return _ref


def _check(rc: int, which=None):
    if rc != 0:
        l = which if which is not None else lib()
        fn = l.or_last_error if hasattr(l, "or_last_error") else l.ref_last_error
        raise OracleError(fn().decode())


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


# --------------------------------------------------------------------------
# geometry descriptions (python-side plain data; arrays owned here)


def centered_volume(shape, spacing):
    """image.hpp:23-32 VolumeSpec::centered"""
    shape = [int(s) for s in shape]
    spacing = [float(s) for s in spacing]
    origin = [-0.5 * float(n - 1) * s for n, s in zip(shape, spacing)]
    return shape, spacing, origin


def make_volume(shape, spacing, origin=None) -> or_volume:
    if origin is None:
        shape, spacing, origin = centered_volume(shape, spacing)
    v = or_volume()
    v.dims = len(shape)
    for a in range(len(shape)):
        v.shape[a] = int(shape[a])
        v.spacing[a] = float(spacing[a])
        v.origin[a] = float(origin[a])
    return v


def det1_centered(n, spacing) -> or_det1:
    return or_det1(int(n), float(spacing), -0.5 * float(n - 1) * float(spacing))


def det2_centered(nu, nv, du, dv) -> or_det2:
    return or_det2(int(nu), int(nv), float(du), float(dv),
                   -0.5 * float(nu - 1) * float(du), -0.5 * float(nv - 1) * float(dv))


@dataclass
class Cone:
    vol: or_volume
    det: or_det2
    n_proj: int
    range: float
    sid: float
    sdd: float
    mats: np.ndarray
    sources: np.ndarray
    invs: np.ndarray
    angles: np.ndarray
    circular: bool = True

    def struct(self) -> or_cone:
        return or_cone(self.vol, self.det, self.n_proj, self.range, self.sid, self.sdd,
                       _ptr(self.mats), _ptr(self.sources), _ptr(self.invs), _ptr(self.angles))

    @property
    def vol_shape_zyx(self):
        return (int(self.vol.shape[2]), int(self.vol.shape[1]), int(self.vol.shape[0]))

    @property
    def sino_shape(self):
        return (self.n_proj, int(self.det.n_v), int(self.det.n_u))


@dataclass
class Planar:
    vol: or_volume
    det: or_det1
    n_proj: int
    range: float
    sid: float
    sdd: float
    rays: np.ndarray
    angles: np.ndarray

    def struct(self) -> or_planar:
        return or_planar(self.vol, self.det, self.n_proj, self.range, self.sid, self.sdd,
                         _ptr(self.rays), _ptr(self.angles))

    @property
    def fan(self):
        return self.sdd > 0.0

    @property
    def img_shape_yx(self):
        return (int(self.vol.shape[1]), int(self.vol.shape[0]))

    @property
    def sino_shape(self):
        return (self.n_proj, int(self.det.n_bins))


def make_cone(vol: or_volume, det: or_det2, n, rng, sid, sdd) -> Cone:
    """geometry.hpp:206-223 make_cone (restated)"""
    n = int(n)
    mats = np.zeros((n, 12)); src = np.zeros((n, 3)); invs = np.zeros((n, 9)); ang = np.zeros(n)
    _check(lib().or_make_cone(C.byref(det), n, float(rng), float(sid), float(sdd), _ptr(mats),
                              _ptr(src), _ptr(invs), _ptr(ang)))
    return Cone(vol, det, n, float(rng), float(sid), float(sdd), mats, src, invs, ang)


def cone_from_matrices(vol, det, rng, sid, sdd, mats_in) -> Cone:
    """geometry.hpp:226-242 make_cone_from_matrices (restated)"""
    mats_in = np.ascontiguousarray(mats_in, dtype=np.float64).reshape(-1, 12)
    n = mats_in.shape[0]
    mats = np.zeros((n, 12)); src = np.zeros((n, 3)); invs = np.zeros((n, 9)); ang = np.zeros(n)
    _check(lib().or_cone_set_matrices(n, float(sid), _ptr(mats_in), _ptr(mats), _ptr(src),
                                      _ptr(invs), _ptr(ang)))
    return Cone(vol, det, n, float(rng), float(sid), float(sdd), mats, src, invs, ang, circular=False)


def make_planar(vol, det, n, rng, sid=0.0, sdd=0.0) -> Planar:
    """geometry.hpp:73-86 make_parallel / 108-124 make_fan (restated)"""
    n = int(n)
    rays = np.zeros((n, 2)); ang = np.zeros(n)
    _check(lib().or_circular_rays_2d(n, float(rng), _ptr(rays)))
    _check(lib().or_view_angles(n, float(rng), _ptr(ang)))
    return Planar(vol, det, n, float(rng), float(sid), float(sdd), rays, ang)


# --------------------------------------------------------------------------
# operators (restatement)


def _typed(dtype):
    return ("f32", C.c_float) if np.dtype(dtype) == np.float32 else ("f64", C.c_double)


def cone_forward(g: Cone, vol: np.ndarray) -> np.ndarray:
    suf, ct = _typed(vol.dtype)
    vol = np.ascontiguousarray(vol)
    out = np.zeros(g.sino_shape, dtype=vol.dtype)
    s = g.struct()
    _check(getattr(lib(), f"or_cone_forward_{suf}")(C.byref(s), _ptr(vol, ct), _ptr(out, ct)))
    return out


def cone_backproject(g: Cone, sino: np.ndarray) -> np.ndarray:
    suf, ct = _typed(sino.dtype)
    sino = np.ascontiguousarray(sino)
    out = np.zeros(g.vol_shape_zyx, dtype=sino.dtype)
    s = g.struct()
    _check(getattr(lib(), f"or_cone_backproject_{suf}")(C.byref(s), _ptr(sino, ct), _ptr(out, ct)))
    return out


def fdk_reconstruct(g: Cone, sino: np.ndarray, use_parker=True) -> np.ndarray:
    suf, ct = _typed(sino.dtype)
    sino = np.ascontiguousarray(sino)
    out = np.zeros(g.vol_shape_zyx, dtype=sino.dtype)
    s = g.struct()
    _check(getattr(lib(), f"or_fdk_reconstruct_{suf}")(C.byref(s), _ptr(sino, ct), _ptr(out, ct),
                                                        int(bool(use_parker))))
    return out


def planar_forward(g: Planar, img: np.ndarray) -> np.ndarray:
    suf, ct = _typed(img.dtype)
    img = np.ascontiguousarray(img)
    out = np.zeros(g.sino_shape, dtype=img.dtype)
    s = g.struct()
    fn = f"or_fan_forward_{suf}" if g.fan else f"or_parallel_forward_{suf}"
    _check(getattr(lib(), fn)(C.byref(s), _ptr(img, ct), _ptr(out, ct)))
    return out


def planar_backproject(g: Planar, sino: np.ndarray) -> np.ndarray:
    suf, ct = _typed(sino.dtype)
    sino = np.ascontiguousarray(sino)
    out = np.zeros(g.img_shape_yx, dtype=sino.dtype)
    s = g.struct()
    fn = f"or_fan_backproject_{suf}" if g.fan else f"or_parallel_backproject_{suf}"
    _check(getattr(lib(), fn)(C.byref(s), _ptr(sino, ct), _ptr(out, ct)))
    return out


def fbp_reconstruct(g: Planar, sino: np.ndarray, weights: np.ndarray) -> np.ndarray:
    suf, ct = _typed(sino.dtype)
    sino = np.ascontiguousarray(sino)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros(g.img_shape_yx, dtype=sino.dtype)
    s = g.struct()
    _check(getattr(lib(), f"or_fbp_reconstruct_{suf}")(C.byref(s), _ptr(sino, ct), _ptr(out, ct),
                                                        _ptr(weights), C.c_uint64(len(weights))))
    return out


def apply_filter(rows: np.ndarray, weights: np.ndarray) -> np.ndarray:
    suf, ct = _typed(rows.dtype)
    out = np.array(rows, copy=True, order="C")
    n = out.shape[-1]
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    _check(getattr(lib(), f"or_apply_filter_{suf}")(_ptr(out, ct), C.c_uint64(out.size // n),
                                                     C.c_uint64(n), _ptr(weights),
                                                     C.c_uint64(len(weights))))
    return out


def apply_weights(data: np.ndarray, wmap: np.ndarray) -> np.ndarray:
    suf, ct = _typed(data.dtype)
    out = np.array(data, copy=True, order="C")
    wmap = np.ascontiguousarray(wmap, dtype=np.float64).ravel()
    getattr(lib(), f"or_apply_weights_{suf}")(_ptr(out, ct), C.c_uint64(out.size), _ptr(wmap),
                                              C.c_uint64(wmap.size))
    return out


def cone_ray_samples(g: Cone) -> np.ndarray:
    out = np.zeros(g.sino_shape, dtype=np.uint64)
    s = g.struct()
    _check(lib().or_cone_ray_samples(C.byref(s), _ptr(out, C.c_uint64)))
    return out


def planar_ray_samples(g: Planar) -> np.ndarray:
    out = np.zeros(g.sino_shape, dtype=np.uint64)
    s = g.struct()
    _check(lib().or_planar_ray_samples(C.byref(s), _ptr(out, C.c_uint64)))
    return out


def filter_window(n) -> int:
    return int(lib().or_filter_window(int(n)))


def ramlak_weights(P, spacing) -> np.ndarray:
    w = np.zeros(int(P))
    lib().or_ramlak_weights(int(P), float(spacing), _ptr(w))
    return w


def ramp_weights(P, spacing) -> np.ndarray:
    w = np.zeros(int(P))
    lib().or_ramp_weights(int(P), float(spacing), _ptr(w))
    return w


def ramlak_spatial(m, spacing) -> float:
    return float(lib().or_ramlak_spatial(int(m), float(spacing)))


def parker_weight(beta, gamma, delta, rng) -> float:
    return float(lib().or_parker_weight(beta, gamma, delta, rng))


def cosine_weights_cone(g: Cone) -> np.ndarray:
    out = np.zeros((int(g.det.n_v), int(g.det.n_u)))
    s = g.struct()
    lib().or_cosine_weights_cone(C.byref(s), _ptr(out))
    return out


def cosine_weights_fan(g: Planar) -> np.ndarray:
    out = np.zeros(int(g.det.n_bins))
    s = g.struct()
    lib().or_cosine_weights_fan(C.byref(s), _ptr(out))
    return out


def parker_weights_cone(g: Cone) -> np.ndarray:
    out = np.zeros((g.n_proj, int(g.det.n_u)))
    s = g.struct()
    _check(lib().or_parker_weights_cone(C.byref(s), _ptr(out)))
    return out


def parker_weights_fan(g: Planar) -> np.ndarray:
    out = np.zeros((g.n_proj, int(g.det.n_bins)))
    s = g.struct()
    _check(lib().or_parker_weights_fan(C.byref(s), _ptr(out)))
    return out


def head_ellipsoids(fov_half) -> np.ndarray:
    out = np.zeros((10, 8))
    lib().or_head_ellipsoids(float(fov_half), _ptr(out))
    return out


def fov_half_extent(vol: or_volume) -> float:
    return float(lib().or_fov_half_extent(C.byref(vol)))


def shepp_logan_3d(vol: or_volume, dtype=np.float32) -> np.ndarray:
    """phantom.hpp:136-140 (restated)"""
    suf, ct = _typed(dtype)
    specs = head_ellipsoids(fov_half_extent(vol))
    out = np.zeros((int(vol.shape[2]), int(vol.shape[1]), int(vol.shape[0])), dtype=dtype)
    _check(getattr(lib(), f"or_rasterize_ellipsoids_{suf}")(C.byref(vol), _ptr(specs), C.c_uint64(10),
                                                             _ptr(out, ct)))
    return out


def shepp_logan_2d(vol: or_volume, dtype=np.float32) -> np.ndarray:
    """phantom.hpp:130-134 (restated)"""
    suf, ct = _typed(dtype)
    specs = np.zeros((10, 6))
    lib().or_head_ellipses(fov_half_extent(vol), _ptr(specs))
    out = np.zeros((int(vol.shape[1]), int(vol.shape[0])), dtype=dtype)
    _check(getattr(lib(), f"or_rasterize_ellipses_{suf}")(C.byref(vol), _ptr(specs), C.c_uint64(10),
                                                           _ptr(out, ct)))
    return out


def rasterize_ellipsoids(vol: or_volume, specs, dtype=np.float64) -> np.ndarray:
    suf, ct = _typed(dtype)
    specs = np.ascontiguousarray(specs, dtype=np.float64).reshape(-1, 8)
    out = np.zeros((int(vol.shape[2]), int(vol.shape[1]), int(vol.shape[0])), dtype=dtype)
    _check(getattr(lib(), f"or_rasterize_ellipsoids_{suf}")(C.byref(vol), _ptr(specs), C.c_uint64(len(specs)),
                                                             _ptr(out, ct)))
    return out


def rasterize_ellipses(vol: or_volume, specs, dtype=np.float64) -> np.ndarray:
    suf, ct = _typed(dtype)
    specs = np.ascontiguousarray(specs, dtype=np.float64).reshape(-1, 6)
    out = np.zeros((int(vol.shape[1]), int(vol.shape[0])), dtype=dtype)
    _check(getattr(lib(), f"or_rasterize_ellipses_{suf}")(C.byref(vol), _ptr(specs), C.c_uint64(len(specs)),
                                                           _ptr(out, ct)))
    return out


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref)


class Ref:
    """Thin access to the reference's own implementation (oracle/_ref)."""

    @staticmethod
    def set_threads(n):
        ref().ref_set_threads(int(n))

    @staticmethod
    def num_threads():
        return int(ref().ref_num_threads())

    @staticmethod
    def _chk(rc):
        if rc != 0:
            raise OracleError(ref().ref_last_error().decode())

    @staticmethod
    def make_cone(vol, det, n, rng, sid, sdd) -> Cone:
        n = int(n)
        mats = np.zeros((n, 12)); src = np.zeros((n, 3)); invs = np.zeros((n, 9)); ang = np.zeros(n)
        Ref._chk(ref().ref_make_cone(C.byref(vol), C.byref(det), C.c_uint64(n), C.c_double(rng),
                                     C.c_double(sid), C.c_double(sdd), _ptr(mats), _ptr(src),
                                     _ptr(invs), _ptr(ang)))
        return Cone(vol, det, n, float(rng), float(sid), float(sdd), mats, src, invs, ang)

    @staticmethod
    def cone_from_matrices(vol, det, rng, sid, sdd, mats_in) -> Cone:
        mats_in = np.ascontiguousarray(mats_in, dtype=np.float64).reshape(-1, 12)
        n = mats_in.shape[0]
        mats = np.zeros((n, 12)); src = np.zeros((n, 3)); invs = np.zeros((n, 9)); ang = np.zeros(n)
        Ref._chk(ref().ref_cone_from_matrices(C.byref(vol), C.byref(det), C.c_uint64(n),
                                              C.c_double(rng), C.c_double(sid), C.c_double(sdd),
                                              _ptr(mats_in), _ptr(mats), _ptr(src), _ptr(invs),
                                              _ptr(ang)))
        return Cone(vol, det, n, float(rng), float(sid), float(sdd), mats, src, invs, ang,
                    circular=False)

    @staticmethod
    def planar_geometry(vol, det, n, rng, sid=0.0, sdd=0.0) -> Planar:
        n = int(n)
        rays = np.zeros((n, 2)); ang = np.zeros(n)
        Ref._chk(ref().ref_planar_rays(C.byref(vol), C.byref(det), C.c_uint64(n), C.c_double(rng),
                                       C.c_double(sid), C.c_double(sdd), _ptr(rays), _ptr(ang)))
        return Planar(vol, det, n, float(rng), float(sid), float(sdd), rays, ang)

    @staticmethod
    def cone_forward(g: Cone, vol):
        suf, ct = _typed(vol.dtype)
        vol = np.ascontiguousarray(vol)
        out = np.zeros(g.sino_shape, dtype=vol.dtype)
        s = g.struct()
        Ref._chk(getattr(ref(), f"ref_cone_forward_{suf}")(C.byref(s), int(g.circular),
                                                            _ptr(vol, ct), _ptr(out, ct)))
        return out

    @staticmethod
    def cone_backproject(g: Cone, sino):
        suf, ct = _typed(sino.dtype)
        sino = np.ascontiguousarray(sino)
        out = np.zeros(g.vol_shape_zyx, dtype=sino.dtype)
        s = g.struct()
        Ref._chk(getattr(ref(), f"ref_cone_backproject_{suf}")(C.byref(s), int(g.circular),
                                                                _ptr(sino, ct), _ptr(out, ct)))
        return out

    @staticmethod
    def fdk_reconstruct(g: Cone, sino, use_parker=True):
        suf, ct = _typed(sino.dtype)
        sino = np.ascontiguousarray(sino)
        out = np.zeros(g.vol_shape_zyx, dtype=sino.dtype)
        s = g.struct()
        Ref._chk(getattr(ref(), f"ref_fdk_reconstruct_{suf}")(C.byref(s), int(g.circular),
                                                               _ptr(sino, ct), _ptr(out, ct),
                                                               int(bool(use_parker))))
        return out

    @staticmethod
    def planar_forward(g: Planar, img):
        suf, ct = _typed(img.dtype)
        img = np.ascontiguousarray(img)
        out = np.zeros(g.sino_shape, dtype=img.dtype)
        s = g.struct()
        Ref._chk(getattr(ref(), f"ref_planar_forward_{suf}")(C.byref(s), _ptr(img, ct),
                                                              _ptr(out, ct)))
        return out

    @staticmethod
    def planar_backproject(g: Planar, sino):
        suf, ct = _typed(sino.dtype)
        sino = np.ascontiguousarray(sino)
        out = np.zeros(g.img_shape_yx, dtype=sino.dtype)
        s = g.struct()
        Ref._chk(getattr(ref(), f"ref_planar_backproject_{suf}")(C.byref(s), _ptr(sino, ct),
                                                                  _ptr(out, ct)))
        return out

    @staticmethod
    def fbp_reconstruct(g: Planar, sino, ramlak=True):
        suf, ct = _typed(sino.dtype)
        sino = np.ascontiguousarray(sino)
        out = np.zeros(g.img_shape_yx, dtype=sino.dtype)
        s = g.struct()
        Ref._chk(getattr(ref(), f"ref_fbp_reconstruct_{suf}")(C.byref(s), _ptr(sino, ct),
                                                               _ptr(out, ct), int(bool(ramlak))))
        return out

    @staticmethod
    def apply_filter(rows, spacing, weights, padded_n=None):
        suf, ct = _typed(rows.dtype)
        out = np.array(rows, copy=True, order="C")
        n = out.shape[-1]
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        P = len(weights) if padded_n is None else int(padded_n)
        Ref._chk(getattr(ref(), f"ref_apply_filter_{suf}")(
            _ptr(out, ct), C.c_uint64(out.size // n), C.c_uint64(n), C.c_double(spacing),
            _ptr(weights), C.c_uint64(P), C.c_uint64(len(weights))))
        return out

    @staticmethod
    def ramlak_weights(P, spacing):
        w = np.zeros(int(P))
        Ref._chk(ref().ref_ramlak_weights(C.c_uint64(P), C.c_double(spacing), _ptr(w)))
        return w

    @staticmethod
    def ramp_weights(P, spacing):
        w = np.zeros(int(P))
        Ref._chk(ref().ref_ramp_weights(C.c_uint64(P), C.c_double(spacing), _ptr(w)))
        return w

    @staticmethod
    def cosine_weights_cone(g: Cone):
        out = np.zeros((int(g.det.n_v), int(g.det.n_u)))
        s = g.struct()
        Ref._chk(ref().ref_cosine_weights_cone(C.byref(s), _ptr(out)))
        return out

    @staticmethod
    def parker_weights_cone(g: Cone):
        out = np.zeros((g.n_proj, int(g.det.n_u)))
        s = g.struct()
        Ref._chk(ref().ref_parker_weights_cone(C.byref(s), _ptr(out)))
        return out

    @staticmethod
    def parker_weights_fan(g: Planar):
        out = np.zeros((g.n_proj, int(g.det.n_bins)))
        s = g.struct()
        Ref._chk(ref().ref_parker_weights_fan(C.byref(s), _ptr(out)))
        return out

    @staticmethod
    def cosine_weights_fan(g: Planar):
        out = np.zeros(int(g.det.n_bins))
        s = g.struct()
        Ref._chk(ref().ref_cosine_weights_fan(C.byref(s), _ptr(out)))
        return out

    @staticmethod
    def shepp_logan_3d(vol, dtype=np.float32):
        suf, ct = _typed(dtype)
        out = np.zeros((int(vol.shape[2]), int(vol.shape[1]), int(vol.shape[0])), dtype=dtype)
        Ref._chk(getattr(ref(), f"ref_shepp_logan_3d_{suf}")(C.byref(vol), _ptr(out, ct)))
        return out

    @staticmethod
    def shepp_logan_2d(vol, dtype=np.float32):
        suf, ct = _typed(dtype)
        out = np.zeros((int(vol.shape[1]), int(vol.shape[0])), dtype=dtype)
        Ref._chk(getattr(ref(), f"ref_shepp_logan_2d_{suf}")(C.byref(vol), _ptr(out, ct)))
        return out


    @staticmethod
    def tv_reconstruct_planar(g: Planar, sino, iterations, lr, lam):
        """pipelines.hpp:273-299 (parallel: the reference function itself; fan:
        the same graph over FanGeometry).  float64 storage (Tensor<double>)."""
        sino = np.ascontiguousarray(sino, dtype=np.float64)
        x = np.zeros(g.img_shape_yx)
        hist = np.zeros(int(iterations) + 1)
        s = g.struct()
        fn = ref().ref_tv_reconstruct_fan if g.fan else ref().ref_tv_reconstruct_parallel
        Ref._chk(fn(C.byref(s), _ptr(sino), _ptr(x), C.c_uint64(int(iterations)),
                    C.c_double(lr), C.c_double(lam), _ptr(hist)))
        return x, hist

    @staticmethod
    def tv_reconstruct_cone(g: Cone, sino, iterations, lr, lam):
        sino = np.ascontiguousarray(sino, dtype=np.float64)
        x = np.zeros(g.vol_shape_zyx)
        hist = np.zeros(int(iterations) + 1)
        s = g.struct()
        Ref._chk(ref().ref_tv_reconstruct_cone(C.byref(s), int(g.circular), _ptr(sino), _ptr(x),
                                               C.c_uint64(int(iterations)), C.c_double(lr),
                                               C.c_double(lam), _ptr(hist)))
        return x, hist

    @staticmethod
    def add_gaussian_noise(data, rel, seed):
        suf, ct = _typed(data.dtype)
        data = np.ascontiguousarray(data)
        out = np.empty_like(data)
        Ref._chk(getattr(ref(), f"ref_add_gaussian_noise_{suf}")(
            _ptr(data, ct), _ptr(out, ct), C.c_uint64(data.size), C.c_double(rel),
            C.c_uint64(int(seed))))
        return out


    @staticmethod
    def learn_filter_graph(g: Planar, sino, P, lr, iterations):
        """experiment_learn_filter's graph (pipelines.hpp:211-259) run by the
        reference's own Graph on a given float64 sinogram."""
        sino = np.ascontiguousarray(sino, dtype=np.float64)
        it = int(iterations)
        loss = np.zeros(it + 1); dist = np.zeros(it + 1); w = np.zeros(int(P))
        rec = np.zeros(g.img_shape_yx)
        s = g.struct()
        Ref._chk(ref().ref_learn_filter_graph(C.byref(s), _ptr(sino), C.c_uint64(int(P)),
                                              C.c_double(lr), C.c_uint64(it), _ptr(loss),
                                              _ptr(dist), _ptr(w), _ptr(rec)))
        return loss, dist, w, rec

    @staticmethod
    def experiment_learn_filter(g: Planar, phantom, noise, seed, window, lr, iterations):
        """pipelines.hpp:196-261 itself; returns (loss, dist, weights, recon)."""
        it = int(iterations)
        P = int(window) if window else filter_window(int(g.det.n_bins))
        loss = np.zeros(it + 1); dist = np.zeros(it + 1); w = np.zeros(P)
        rec = np.zeros(g.img_shape_yx)
        padded = C.c_uint64(0)
        s = g.struct()
        Ref._chk(ref().ref_experiment_learn_filter(
            C.byref(s), phantom.encode(), C.c_double(noise), C.c_uint64(int(seed)),
            C.c_uint64(int(window)), C.c_double(lr), C.c_uint64(it), _ptr(loss), _ptr(dist),
            _ptr(w), _ptr(rec), C.byref(padded)))
        assert padded.value == P
        return loss, dist, w, rec

    @staticmethod
    def graph_probe(g: Planar, x0, w0, sino, lam):
        """loss = l2(multiply_weights(forward_project(x), w), p) + scale(tv(x), lam):
        the value and the gradients of x and w after one backward (reference Graph)."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        w0 = np.ascontiguousarray(w0, dtype=np.float64)
        sino = np.ascontiguousarray(sino, dtype=np.float64)
        loss = C.c_double(0.0)
        gx = np.zeros(g.img_shape_yx); gw = np.zeros(int(g.det.n_bins))
        s = g.struct()
        Ref._chk(ref().ref_graph_probe(C.byref(s), int(g.fan), _ptr(x0), _ptr(w0), _ptr(sino),
                                       C.c_double(lam), C.byref(loss), _ptr(gx), _ptr(gw)))
        return loss.value, gx, gw


def rel_errors(out: np.ndarray, ref_: np.ndarray):
    """(max|d| / max|ref|, relRMSE = ||d||2 / ||ref||2) — SURVEY §8c metrics."""
    d = out.astype(np.float64) - ref_.astype(np.float64)
    mref = float(np.max(np.abs(ref_))) if ref_.size else 0.0
    nref = float(np.linalg.norm(ref_.astype(np.float64)))
    mx = float(np.max(np.abs(d))) if d.size else 0.0
    return (mx / mref if mref > 0 else mx, float(np.linalg.norm(d)) / nref if nref > 0 else 0.0)


PI = math.pi


# --------------------------------------------------------------------------
# iterative reconstruction pieces (restatement; graph.hpp / pipelines.hpp)


def l2_value(a, b) -> float:
    suf, ct = _typed(a.dtype)
    a = np.ascontiguousarray(a); b = np.ascontiguousarray(b, dtype=a.dtype)
    fn = getattr(lib(), f"or_l2_value_{suf}")
    fn.restype = C.c_double
    return float(fn(_ptr(a, ct), _ptr(b, ct), C.c_uint64(a.size)))


def _shape_fastest_first(x):
    return np.array(list(reversed(x.shape)), dtype=np.uint64)


def tv_value(x) -> float:
    suf, ct = _typed(x.dtype)
    x = np.ascontiguousarray(x)
    shp = _shape_fastest_first(x)
    fn = getattr(lib(), f"or_tv_value_{suf}")
    fn.restype = C.c_double
    return float(fn(_ptr(x, ct), _ptr(shp, C.c_uint64), C.c_uint32(len(shp))))


def tv_subgrad(x, gs=1.0) -> np.ndarray:
    """graph.hpp:511-528 into a zero gradient (FP64)"""
    suf, ct = _typed(x.dtype)
    x = np.ascontiguousarray(x)
    shp = _shape_fastest_first(x)
    gx = np.zeros(x.shape)
    getattr(lib(), f"or_tv_subgrad_acc_{suf}")(_ptr(x, ct), _ptr(shp, C.c_uint64),
                                                C.c_uint32(len(shp)), C.c_double(gs), _ptr(gx))
    return gx


def tv_reconstruct_planar(g: Planar, sino, iterations, lr, lam):
    suf, ct = _typed(sino.dtype)
    sino = np.ascontiguousarray(sino)
    x = np.zeros(g.img_shape_yx, dtype=sino.dtype)
    hist = np.zeros(int(iterations) + 1)
    s = g.struct()
    _check(getattr(lib(), f"or_tv_reconstruct_planar_{suf}")(
        C.byref(s), _ptr(sino, ct), _ptr(x, ct), C.c_uint64(int(iterations)), C.c_double(lr),
        C.c_double(lam), _ptr(hist)))
    return x, hist


def tv_reconstruct_cone(g: Cone, sino, iterations, lr, lam):
    suf, ct = _typed(sino.dtype)
    sino = np.ascontiguousarray(sino)
    x = np.zeros(g.vol_shape_zyx, dtype=sino.dtype)
    hist = np.zeros(int(iterations) + 1)
    s = g.struct()
    _check(getattr(lib(), f"or_tv_reconstruct_cone_{suf}")(
        C.byref(s), _ptr(sino, ct), _ptr(x, ct), C.c_uint64(int(iterations)), C.c_double(lr),
        C.c_double(lam), _ptr(hist)))
    return x, hist


def add_gaussian_noise(data, rel, seed):
    suf, ct = _typed(data.dtype)
    data = np.ascontiguousarray(data)
    out = np.empty_like(data)
    _check(getattr(lib(), f"or_add_gaussian_noise_{suf}")(
        _ptr(data, ct), _ptr(out, ct), C.c_uint64(data.size), C.c_double(rel),
        C.c_uint64(int(seed))))
    return out


def mt19937_64(seed, k) -> int:
    fn = lib().or_mt19937_64_first
    fn.restype = C.c_uint64
    return int(fn(C.c_uint64(int(seed)), C.c_uint64(int(k))))


def learn_filter_planar(g: Planar, sino, P, lr, iterations):
    """Restatement of experiment_learn_filter's graph loop (pipelines.hpp:211-259)
    on storage sino.dtype; returns (loss, dist, weights, recon)."""
    suf, ct = _typed(sino.dtype)
    sino = np.ascontiguousarray(sino)
    it = int(iterations)
    loss = np.zeros(it + 1); dist = np.zeros(it + 1); w = np.zeros(int(P))
    rec = np.zeros(g.img_shape_yx, dtype=sino.dtype)
    s = g.struct()
    _check(getattr(lib(), f"or_learn_filter_planar_{suf}")(
        C.byref(s), _ptr(sino, ct), C.c_uint64(int(P)), C.c_double(lr), C.c_uint64(it),
        _ptr(loss), _ptr(dist), _ptr(w), _ptr(rec, ct)))
    return loss, dist, w, rec
