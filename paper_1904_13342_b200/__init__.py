"""B200-native (sm_100a) projector / FDK path with the reference toolkit's
operator API (tomograd: image.hpp, geometry.hpp, projector.hpp,
filtering.hpp, pipelines.hpp, phantom.hpp).

The compute runs in hand-written CUDA kernels inside libtomograd_b200.so,
reached through its C ABI (include/tomograd_b200.h).  There is no CPU
fallback: without the library or a CUDA device the operators raise.
"""
from ._native import CudaError, Error  # noqa: F401
from .containers import Image, Sinogram  # noqa: F401
from .filtering import (Filter1D, WeightMap, apply_filter, apply_weights,  # noqa: F401
                        cosine_weights, filter_window, parker_weights, ramlak_filter,
                        ramlak_spatial, ramlak_weights, ramp_filter, ramp_weights)
from .geometry import (ConeGeometry, Detector1D, Detector2D, FanGeometry,  # noqa: F401
                       ParallelGeometry, VolumeSpec, cone_projection_matrix, make_cone,
                       make_cone_from_matrices, make_fan, make_parallel,
                       projection_matrices_circular, view_angles)
from .phantom import (disk_phantom, head_phantom_ellipses, head_phantom_ellipsoids,  # noqa: F401
                      rasterize, shepp_logan_2d, shepp_logan_3d)
from .iterative import (ExperimentConfig, FilterLearningResult, TvResult,  # noqa: F401
                        add_gaussian_noise, experiment_iterative_tv, experiment_learn_filter,
                        l2_residual, learn_filter, tv_reconstruct, tv_step)
from .graph import (BackProject, FourierFilter, ForwardProject, Graph, OpKind,  # noqa: F401
                    back_project_op, forward_project_op, fourier_filter_op,
                    gradient_descent_step)
from .pipelines import (FilterKind, fbp_reconstruct, fdk_prefilter, fdk_reconstruct,  # noqa: F401
                        fdk_scale, make_filter)
from .projector import (back_project, cone_backproject_slab, cone_forward_views,  # noqa: F401
                        ray_sample_counts, set_cone_knob,
                        cone_slab_rows, forward_project)


def kernel_launch_count() -> int:
    """Kernels this library has launched in this process."""
    from . import _native
    return int(_native.lib().tg_kernel_launch_count())
