"""ctypes binding of the C ABI (include/tomograd_b200.h).

The library is built in-tree by ``paper_1904_13342_b200.build`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing, or no CUDA device is visible, every operator raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtomograd_b200.so")

c_u64 = C.c_uint64
c_dbl = C.c_double
c_int = C.c_int
c_f32p = C.POINTER(C.c_float)
c_dblp = C.POINTER(C.c_double)
c_u64p = C.POINTER(C.c_uint64)
c_vp = C.c_void_p


class tg_volume_spec(C.Structure):
    _fields_ = [("dims", C.c_uint32), ("shape", c_u64 * 3), ("spacing", c_dbl * 3),
                ("origin", c_dbl * 3)]


class tg_detector1d(C.Structure):
    _fields_ = [("n_bins", c_u64), ("spacing", c_dbl), ("origin", c_dbl)]


class tg_detector2d(C.Structure):
    _fields_ = [("n_u", c_u64), ("n_v", c_u64), ("spacing_u", c_dbl), ("spacing_v", c_dbl),
                ("origin_u", c_dbl), ("origin_v", c_dbl)]


class tg_planar_geometry(C.Structure):
    _fields_ = [("volume", tg_volume_spec), ("detector", tg_detector1d), ("n_projections", c_u64),
                ("angular_range", c_dbl), ("sid", c_dbl), ("sdd", c_dbl), ("rays", c_dblp),
                ("angles", c_dblp)]


class tg_cone_geometry(C.Structure):
    _fields_ = [("volume", tg_volume_spec), ("detector", tg_detector2d), ("n_projections", c_u64),
                ("angular_range", c_dbl), ("sid", c_dbl), ("sdd", c_dbl), ("matrices", c_dblp),
                ("sources", c_dblp), ("inv_blocks", c_dblp), ("angles", c_dblp)]


class tg_band_dest(C.Structure):
    _fields_ = [("band", c_vp), ("v0", c_u64), ("n_rows", c_u64)]


_P = C.POINTER
# name -> (restype, argtypes); mirrors include/tomograd_b200.h one to one
SIGNATURES = {
    "tg_last_error": (C.c_char_p, []),
    "tg_abi_version": (c_int, []),
    "tg_view_angles": (c_int, [c_u64, c_dbl, c_dblp]),
    "tg_make_planar": (c_int, [_P(tg_volume_spec), _P(tg_detector1d), c_u64, c_dbl, c_dbl, c_dbl,
                               c_dblp, c_dblp]),
    "tg_cone_projection_matrix": (c_int, [c_dbl, c_dbl, c_dbl, _P(tg_detector2d), c_dblp]),
    "tg_make_cone": (c_int, [_P(tg_volume_spec), _P(tg_detector2d), c_u64, c_dbl, c_dbl, c_dbl,
                             c_dblp, c_dblp, c_dblp, c_dblp]),
    "tg_cone_set_matrices": (c_int, [c_u64, c_dbl, c_dblp, c_dblp, c_dblp, c_dblp, c_dblp]),
    "tg_filter_window": (c_u64, [c_u64]),
    "tg_ramp_weights": (c_int, [c_u64, c_dbl, c_dblp]),
    "tg_ramlak_weights": (c_int, [c_u64, c_dbl, c_dblp]),
    "tg_cosine_weights_fan": (c_int, [_P(tg_planar_geometry), c_dblp]),
    "tg_cosine_weights_cone": (c_int, [_P(tg_cone_geometry), c_dblp]),
    "tg_parker_weights_fan": (c_int, [_P(tg_planar_geometry), c_dblp]),
    "tg_parker_weights_cone": (c_int, [_P(tg_cone_geometry), c_dblp]),
    "tg_cone_plan_create": (c_int, [_P(tg_cone_geometry), c_int, _P(c_vp)]),
    "tg_cone_plan_destroy": (c_int, [c_vp]),
    "tg_cone_forward": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "tg_cone_forward_views": (c_int, [c_vp, c_u64, c_u64, c_vp, c_vp, c_vp]),
    "tg_cone_backproject": (c_int, [c_vp, c_vp, c_vp, C.c_float, c_int, c_vp]),
    "tg_cone_slab_rows": (c_int, [c_vp, c_u64, c_u64, c_u64p, c_u64p]),
    "tg_cone_slab_rows_geom": (c_int, [_P(tg_cone_geometry), c_u64, c_u64, c_u64p, c_u64p]),
    "tg_cone_backproject_slab": (c_int, [c_vp, c_u64, c_u64, c_u64, c_u64, c_vp, c_vp, C.c_float,
                                         c_int, c_vp]),
    "tg_cone_fdk_prefilter": (c_int, [c_vp, c_vp, c_vp, c_int, c_u64, c_u64, c_vp]),
    "tg_cone_fdk_scale": (c_dbl, [c_vp, c_int]),
    "tg_cone_fdk": (c_int, [c_vp, c_vp, c_vp, c_vp, c_int, c_vp]),
    "tg_cone_forward_host": (c_int, [c_vp, c_vp, c_vp]),
    "tg_cone_backproject_host": (c_int, [c_vp, c_vp, c_vp]),
    "tg_cone_fdk_host": (c_int, [c_vp, c_vp, c_vp, c_int]),
    "tg_cone_backproject_slab_host": (c_int, [c_vp, c_u64, c_u64, c_u64, c_u64, c_vp, c_vp, c_int,
                                              c_int]),
    "tg_cone_last_h2d_bytes": (c_u64, [c_vp]),
    "tg_planar_plan_create": (c_int, [_P(tg_planar_geometry), c_int, _P(c_vp)]),
    "tg_planar_plan_destroy": (c_int, [c_vp]),
    "tg_planar_forward": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "tg_planar_backproject": (c_int, [c_vp, c_vp, c_vp, C.c_float, c_int, c_vp]),
    "tg_planar_forward_host": (c_int, [c_vp, c_vp, c_vp]),
    "tg_planar_backproject_host": (c_int, [c_vp, c_vp, c_vp]),
    "tg_filter_plan_create": (c_int, [c_u64, c_dbl, c_u64, c_u64, c_dbl, c_dblp, c_u64, c_int,
                                      _P(c_vp)]),
    "tg_filter_plan_destroy": (c_int, [c_vp]),
    "tg_filter_apply": (c_int, [c_vp, c_vp, c_vp, c_u64, c_vp]),
    "tg_filter_apply_host": (c_int, [c_vp, c_vp, c_vp, c_u64]),
    "tg_apply_weights": (c_int, [c_vp, c_vp, c_u64, c_vp, c_u64, c_vp]),
    "tg_apply_row_weights": (c_int, [c_vp, c_vp, c_u64, c_u64, c_u64, c_vp, c_vp]),
    "tg_rasterize_ellipsoids": (c_int, [_P(tg_volume_spec), c_dblp, c_u64, c_vp, c_vp]),
    "tg_rasterize_ellipses": (c_int, [_P(tg_volume_spec), c_dblp, c_u64, c_vp, c_vp]),
    "tg_head_phantom_ellipsoids": (c_int, [_P(tg_volume_spec), c_dblp]),
    "tg_head_phantom_ellipses": (c_int, [_P(tg_volume_spec), c_dblp]),
    "tg_cone_plan_shape": (c_int, [c_vp, _P(tg_volume_spec), _P(tg_detector2d), c_u64p]),
    "tg_planar_plan_shape": (c_int, [c_vp, _P(tg_volume_spec), _P(tg_detector1d), c_u64p]),
    "tg_l2_residual": (c_int, [c_vp, c_vp, c_vp, c_u64, c_vp, c_vp]),
    "tg_tv_step": (c_int, [c_vp, c_vp, c_vp, c_u64, c_u64, c_u64, c_int, c_int, c_dbl, c_dbl, c_vp,
                           c_vp]),
    "tg_l2_residual_scatter": (c_int, [c_vp, c_vp, c_u64, c_u64, c_u64, c_u64, _P(tg_band_dest),
                                       c_int, c_vp, c_vp]),
    "tg_tv_step_multi": (c_int, [c_vp, c_vp, _P(c_vp), c_int, c_u64, c_u64, c_u64, c_int, c_int,
                                 c_dbl, c_dbl, c_vp, c_vp]),
    "tg_device_alloc": (c_int, [c_u64, c_int, _P(c_vp)]),
    "tg_device_free": (c_int, [c_vp]),
    "tg_ipc_get_handle": (c_int, [c_vp, _P(C.c_ubyte)]),
    "tg_ipc_open_handle": (c_int, [_P(C.c_ubyte), c_int, _P(c_vp)]),
    "tg_ipc_close_handle": (c_int, [c_vp]),
    "tg_cone_tv_reconstruct": (c_int, [c_vp, c_vp, c_vp, c_u64, c_dbl, c_dbl, c_dblp, c_vp]),
    "tg_planar_tv_reconstruct": (c_int, [c_vp, c_vp, c_vp, c_u64, c_dbl, c_dbl, c_dblp, c_vp]),
    "tg_cone_tv_reconstruct_host": (c_int, [c_vp, c_vp, c_vp, c_u64, c_dbl, c_dbl, c_dblp]),
    "tg_planar_tv_reconstruct_host": (c_int, [c_vp, c_vp, c_vp, c_u64, c_dbl, c_dbl, c_dblp]),
    "tg_add_gaussian_noise": (c_int, [c_vp, c_vp, c_u64, c_dbl, c_u64]),
    "tg_axpby": (c_int, [c_vp, c_vp, c_vp, c_u64, c_dbl, c_dbl, c_vp]),
    "tg_multiply_weights": (c_int, [c_vp, c_vp, c_vp, c_u64, c_u64, c_vp]),
    "tg_multiply_weights_grad": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_u64, c_u64, c_vp]),
    "tg_fourier_filter": (c_int, [c_vp, c_vp, c_vp, c_u64, c_u64, c_u64, c_vp]),
    "tg_fourier_filter_weight_grad": (c_int, [c_vp, c_vp, c_vp, c_u64, c_u64, c_u64, c_vp]),
    "tg_l2_grad": (c_int, [c_vp, c_vp, c_vp, c_vp, c_u64, c_dbl, c_vp]),
    "tg_tv_grad": (c_int, [c_vp, c_vp, c_u64, c_u64, c_u64, c_dbl, c_vp, c_vp]),
    "tg_planar_learn_filter": (c_int, [c_vp, c_vp, c_vp, c_vp, c_u64, c_dblp, c_dblp, c_dbl, c_u64,
                                       c_dblp, c_dblp, c_vp, c_vp]),
    "tg_planar_learn_filter_host": (c_int, [c_vp, c_vp, c_vp, c_vp, c_u64, c_dblp, c_dblp, c_dbl,
                                            c_u64, c_dblp, c_dblp, c_vp]),
    "tg_nan_count": (c_int, [c_vp, c_u64, c_vp, c_vp]),
    "tg_cone_ray_samples": (c_int, [c_vp, c_u64, c_u64, c_vp, c_vp]),
    "tg_cone_plan_set_knob": (c_int, [c_vp, C.c_char_p, C.c_int64]),
    "tg_planar_ray_samples": (c_int, [c_vp, c_vp, c_vp]),
    "tg_kernel_launch_count": (c_u64, []),
    "tg_set_timing": (None, [c_int]),
    "tg_last_kernel_ms": (c_dbl, []),
}

TG_OK, TG_ERROR, TG_ERROR_CUDA, TG_ERROR_NO_DEVICE = 0, 1, 2, 3


class Error(RuntimeError):
    """tomograd::Error (core.hpp:19-22): carries the reference's exact message."""


class CudaError(RuntimeError):
    """A CUDA runtime/driver failure inside the B200 path."""


_lib = None


def lib():
    """Load libtomograd_b200.so (no fallback: raises when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing; build it with `python -m paper_1904_13342_b200.build` "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == TG_OK:
        return
    msg = lib().tg_last_error().decode()
    if status == TG_ERROR:
        raise Error(msg)
    raise CudaError(msg)


def dptr(a) -> C.POINTER(C.c_double):
    """numpy float64 array -> double*"""
    return a.ctypes.data_as(c_dblp)
