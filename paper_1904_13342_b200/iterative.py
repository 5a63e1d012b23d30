"""Iterative TV-regularised reconstruction on the device
path: pipelines.hpp:273-312 over the graph pieces of graph.hpp.

    tv_reconstruct(sino, geo, cfg) -> (Image, loss_history)      pipelines.hpp:273-299
    experiment_iterative_tv(geo, cfg) -> TvResult                pipelines.hpp:301-312
    add_gaussian_noise(sino, relative_std, seed)                 pipelines.hpp:119-132
    l2_residual(a, b, grad=None) -> float                        graph.hpp:345-353, 498-509
    tv_step(x, grad, out, lambda, lr) -> float                   graph.hpp:365-377, 511-546

The reference's ``tv_reconstruct`` is typed for ParallelGeometry; its graph
nodes take any geometry (graph.hpp:117-135), so here every geometry type
(parallel, fan, cone) runs the same loop — the cone case is BASELINE config
c5.  The whole loop is device resident (K2/K1 or K5-K7, then K8 residual and
K9 fused TV + descent); only the loss history returns to the host.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import math

import numpy as np
import torch

from . import _native as N
from .containers import Image, Sinogram, is_host, require_f32, stream_of
from .geometry import ConeGeometry, FanGeometry, ParallelGeometry, check
from .projector import _check_cone_sino, _check_planar_sino, _dev


@dataclass
class ExperimentConfig:
    """pipelines.hpp:156-164"""
    phantom: str = "shepp-logan"
    noise_relative_std: float = 0.0
    learning_rate: float = 1e-3
    iterations: int = 100
    tv_lambda: float = 0.0
    seed: int = 1337
    filter_window: int = 0


@dataclass
class TvResult:
    """pipelines.hpp:264-270"""
    phantom: Image = None
    noisy_sinogram: Sinogram = None
    reconstruction: Image = None
    fbp_reference: Image = None
    loss_history: List[float] = field(default_factory=list)


def add_gaussian_noise(sino: Sinogram, relative_std: float, seed: int) -> Sinogram:
    """pipelines.hpp:119-132: additive white noise, sigma = relative_std *
    max(sino), from the reference's mt19937_64 Box-Muller stream (bit-exact,
    host)."""
    data = sino.data
    on_dev = isinstance(data, torch.Tensor)
    host = np.ascontiguousarray(data.detach().cpu().numpy() if on_dev else data, dtype=np.float32)
    out = np.empty_like(host)
    N.check(N.lib().tg_add_gaussian_noise(host.ctypes.data, out.ctypes.data, host.size,
                                          float(relative_std), int(seed)))
    new = torch.from_numpy(out).to(data.device) if on_dev else out
    s = Sinogram.__new__(Sinogram)
    s.__dict__.update(sino.__dict__)
    s.data = new
    return s


def l2_residual(a: torch.Tensor, b: torch.Tensor, grad: torch.Tensor = None) -> float:
    """graph.hpp:345-353 value sum (a - b)^2 (FP64, deterministic); with
    ``grad`` also writes the l2 gradient 2 (a - b) (graph.hpp:498-509)."""
    check(a.shape == b.shape, "l2_loss expects matching shapes")
    a, b = require_f32(a, "a"), require_f32(b, "b")
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    N.check(N.lib().tg_l2_residual(a.data_ptr(), b.data_ptr(),
                                   grad.data_ptr() if grad is not None else None, a.numel(),
                                   out.data_ptr(), stream_of(a)))
    return float(out.item())


def tv_step(x: torch.Tensor, grad: torch.Tensor = None, out: torch.Tensor = None,
            tv_lambda: float = 0.0, learning_rate: float = 0.0, has_lo: bool = False,
            has_hi: bool = False, x_base: torch.Tensor = None) -> float:
    """graph.hpp:365-377 TV value, 511-528 subgradient, 533-546 descent, fused:
    out = x - lr (tv_lambda * dTV(x) + grad); returns TV(x) (FP64).  ``x`` is a
    [ny][nx] image or a [nz][ny][nx] block; for a z-slab of a full replica pass
    the slab view as ``x`` and has_lo / has_hi when the neighbouring slices
    exist in the same storage."""
    x = require_f32(x, "x")
    check(x.is_contiguous(), "tv_step expects a contiguous block")
    nz, ny, nx = (1,) + tuple(x.shape) if x.dim() == 2 else tuple(x.shape)
    if has_lo or has_hi:
        base = x_base if x_base is not None else x
        lo = x.data_ptr() - base.data_ptr()
        check(not has_lo or lo >= 4 * nx * ny, "tv_step: no slice before the block")
        check(not has_hi or lo + 4 * x.numel() + 4 * nx * ny <= 4 * base.numel(),
              "tv_step: no slice after the block")
    v = torch.empty(1, dtype=torch.float64, device=x.device)
    N.check(N.lib().tg_tv_step(x.data_ptr(), grad.data_ptr() if grad is not None else None,
                               out.data_ptr() if out is not None else None, nx, ny, nz,
                               int(has_lo), int(has_hi), float(tv_lambda), float(learning_rate),
                               v.data_ptr(), stream_of(x)))
    return float(v.item())


def tv_reconstruct(sino: Sinogram, geo, cfg: ExperimentConfig,
                   init: torch.Tensor = None) -> Tuple[Image, List[float]]:
    """pipelines.hpp:273-299: min_x |Ax - p|^2 + tv_lambda TV(x), plain
    gradient descent from zero (or ``init``), cfg.iterations steps at
    cfg.learning_rate; returns the image and the iterations + 1 losses.
    Raises the reference's "optimization diverged ..." Error on a non-finite
    loss."""
    if isinstance(geo, ConeGeometry):
        _check_cone_sino(sino, geo)
    else:
        check(isinstance(geo, (ParallelGeometry, FanGeometry)), "unknown geometry type")
        _check_planar_sino(sino, geo)
    data = require_f32(sino.data, "sinogram data")
    on_host = is_host(data)
    if on_host:
        data = torch.from_numpy(np.ascontiguousarray(data)).cuda()
    L = N.lib()
    x = torch.zeros(geo.volume.torch_shape, dtype=torch.float32, device=data.device)
    if init is not None:
        x.copy_(init)
    hist = np.zeros(int(cfg.iterations) + 1, np.float64)
    args = (data.data_ptr(), x.data_ptr(), int(cfg.iterations), float(cfg.learning_rate),
            float(cfg.tv_lambda), hist.ctypes.data_as(N.c_dblp), stream_of(data))
    if isinstance(geo, ConeGeometry):
        N.check(L.tg_cone_tv_reconstruct(geo._plan(_dev(data)), *args))
    else:
        N.check(L.tg_planar_tv_reconstruct(geo._plan(_dev(data)), *args))
    img = Image(geo.volume, x.cpu().numpy() if on_host else x)
    return img, hist.tolist()


def make_phantom_2d(name: str, vol, device=None) -> Image:
    """pipelines.hpp:166-172"""
    from .phantom import disk_phantom, shepp_logan_2d
    if name == "shepp-logan":
        return shepp_logan_2d(vol, device)
    if name == "disk":
        # phantom.hpp:124-128 fov_half_extent
        h = vol.extent(0)
        for a in range(1, vol.dims()):
            h = min(h, vol.extent(a))
        return disk_phantom(vol, 0.4 * 2.0 * (0.5 * h), 1.0, device)
    raise N.Error("unknown phantom: " + name)


def experiment_iterative_tv(geo: ParallelGeometry, cfg: ExperimentConfig, device=None) -> TvResult:
    """pipelines.hpp:301-312: phantom -> forward projection -> noise -> FBP
    reference and TV reconstruction, all on the device."""
    from .pipelines import FilterKind, fbp_reconstruct
    from .projector import forward_project
    r = TvResult()
    r.phantom = make_phantom_2d(cfg.phantom, geo.volume, device)
    sino = forward_project(r.phantom, geo)
    r.noisy_sinogram = add_gaussian_noise(sino, cfg.noise_relative_std, cfg.seed)
    r.fbp_reference = fbp_reconstruct(r.noisy_sinogram, geo, FilterKind.ramlak)
    r.reconstruction, r.loss_history = tv_reconstruct(r.noisy_sinogram, geo, cfg)
    return r


# ---- reconstruction-filter learning (pipelines.hpp:181-261) ---------------


@dataclass
class FilterLearningResult:
    """pipelines.hpp:183-190"""
    loss_history: List[float] = field(default_factory=list)
    distance_history: List[float] = field(default_factory=list)
    learned_weights: np.ndarray = None
    ramp_init: object = None
    ramlak_reference: object = None
    reconstruction: Image = None


def learn_filter(sino: Sinogram, geo: ParallelGeometry, cfg: ExperimentConfig,
                 via_graph: bool = False) -> FilterLearningResult:
    """pipelines.hpp:202-259 on a given sinogram: frequency weights K start at
    the ramp and descend on |pi/n BP(filter(p, K)) - FBP_ramlak(p)|^2.

    Default: the device-resident loop (tg_planar_learn_filter — K3 filter, K6
    back-projection, K8, K7, weight gradient and descent per step, one step
    captured in a CUDA graph and replayed).  ``via_graph``: the same loop
    built node by node on graph.Graph, exactly as the reference builds it."""
    from .filtering import ramlak_filter, ramp_filter
    from .pipelines import fbp_reconstruct
    check(isinstance(geo, ParallelGeometry), "learn-filter expects a parallel-beam geometry")
    r = FilterLearningResult()
    r.ramp_init = ramp_filter(geo.detector.n_bins, geo.detector.spacing, cfg.filter_window)
    r.ramlak_reference = ramlak_filter(geo.detector.n_bins, geo.detector.spacing,
                                       cfg.filter_window)
    padded = r.ramp_init.padded_n
    data = sino.data
    check(isinstance(data, torch.Tensor) and data.is_cuda,
          "learn_filter runs on the device: pass a CUDA sinogram")
    data = data.contiguous()
    reference = fbp_reconstruct(sino, geo, r.ramlak_reference)
    if via_graph:
        return _learn_filter_graph(r, data, reference.data, geo, cfg)
    k = torch.from_numpy(r.ramp_init.weights.astype(np.float32)).to(data.device)
    it = int(cfg.iterations)
    loss = np.zeros(it + 1)
    dist = np.zeros(it + 1)
    recon = torch.empty_like(reference.data)
    N.check(N.lib().tg_planar_learn_filter(
        geo._plan(_dev(data)), data.data_ptr(), reference.data.data_ptr(), k.data_ptr(), padded,
        N.dptr(r.ramp_init.weights), N.dptr(r.ramlak_reference.weights),
        float(cfg.learning_rate), it, N.dptr(loss), N.dptr(dist), recon.data_ptr(),
        stream_of(data)))
    r.loss_history = [float(v) for v in loss]
    r.distance_history = [float(v) for v in dist]
    r.learned_weights = k.double().cpu().numpy()
    r.reconstruction = Image(geo.volume, recon)
    return r


def _learn_filter_graph(r, data, target_data, geo, cfg) -> FilterLearningResult:
    from .graph import Graph, gradient_descent_step
    padded = r.ramp_init.padded_n
    ramlak_w = r.ramlak_reference.weights
    gap = float(np.sqrt(np.sum((r.ramp_init.weights - ramlak_w) ** 2)))
    g = Graph(device=data.device)
    p = g.input(list(reversed(data.shape)))
    K = g.parameter(torch.from_numpy(r.ramp_init.weights.astype(np.float32)), trainable=True)
    target = g.parameter(target_data, trainable=False)
    filtered = g.fourier_filter(p, K, padded)
    bp = g.backproject(filtered, geo)
    recon = g.scale(bp, math.pi / float(geo.n_projections))
    loss = g.l2_loss(recon, target)
    feeds = {p: data}

    def record():
        r.loss_history.append(float(g.value(loss)))
        w = g.node(K).value.double().cpu().numpy()
        d = float(np.sqrt(np.sum((w - ramlak_w) ** 2)))
        r.distance_history.append(d / gap if gap > 0.0 else 0.0)

    def converging(it):
        if not math.isfinite(r.loss_history[-1]):
            raise N.Error(f"optimization diverged at iteration {it} (loss is not finite); "
                          "lower the learning rate")

    for it in range(int(cfg.iterations)):
        g.forward(feeds)
        record()
        converging(it)
        grads = g.backward(loss)
        gradient_descent_step(g, grads, cfg.learning_rate)
    g.forward(feeds)
    record()
    converging(int(cfg.iterations))
    r.learned_weights = g.node(K).value.double().cpu().numpy()
    r.reconstruction = Image(geo.volume, g.value(recon).clone())
    return r


def experiment_learn_filter(geo: ParallelGeometry, cfg: ExperimentConfig,
                            device=None) -> FilterLearningResult:
    """pipelines.hpp:196-261: phantom -> forward projection -> optional noise ->
    filter learning, all on the device."""
    from .projector import forward_project
    check(isinstance(geo, ParallelGeometry), "learn-filter expects a parallel-beam geometry")
    phantom = make_phantom_2d(cfg.phantom, geo.volume, device)
    sino = forward_project(phantom, geo)
    if cfg.noise_relative_std > 0.0:
        sino = add_gaussian_noise(sino, cfg.noise_relative_std, cfg.seed)
    return learn_filter(sino, geo, cfg)
