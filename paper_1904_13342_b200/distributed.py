"""Multi-GPU sharding of the projector path, one process per GPU.

* Back-projection / FDK shards the volume into z-slabs.  Each rank needs only
  the detector row band its slab projects onto (``slab_rows``), filters that
  band locally (the Ram-Lak filter runs along u) and back-projects it: single
  pass FDK has no data-path collective at all.  Slab boundaries are aligned
  to K1's 32-voxel z tiles so a slab is bitwise equal to the same z range of
  the single-GPU result.
* Forward projection shards by angle: every rank holds the volume and
  projects its view range.
* Collectives (NCCL over NVLink on a B200 box, gloo in the CPU tests) exist
  only to reassemble results between passes of an iterative loop:
  ``gather_slabs`` (all_gather of z-slabs), ``gather_views`` and
  ``exchange_bands`` (all_to_all of residual row bands from angle owners to
  slab owners).
* ``tv_reconstruct_sharded`` is the config-5 loop (pipelines.hpp:273-299 on a
  cone geometry) over that decomposition: per iteration each rank projects
  its views from its volume replica (K2), forms the l2 residual (K8), sends
  every slab owner the rows of it that slab needs (one all_to_all), back-
  projects its own slab from the received band (K1), applies the fused TV
  subgradient + descent step to its slab with one-slice halos read from the
  replica (K9), and all_gathers the slabs into the next replica.  The two
  loss partials travel in one small all_gather and are summed in rank order
  (bit-identical on every rank).  The image is bitwise independent of the
  world size (32-aligned slabs, per-view projections, per-voxel updates).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Tuple

import torch
import torch.distributed as dist

from . import _native as N
from .geometry import ConeGeometry

Z_ALIGN = 32  # K1 z tile (csrc/cone.cu default_k1_k)


def even_partition(n: int, parts: int, align: int = 1) -> List[Tuple[int, int]]:
    """Split [0, n) into `parts` contiguous ranges whose starts are multiples
    of `align` (except possibly when n is not); returns (start, count)."""
    assert parts >= 1
    units = (n + align - 1) // align
    base, extra = divmod(units, parts)
    out, u = [], 0
    for r in range(parts):
        cnt = base + (1 if r < extra else 0)
        s, e = u * align, min((u + cnt) * align, n)
        out.append((s, max(0, e - s)))
        u += cnt
    return out


def slab_rows(geo: ConeGeometry, z0: int, nz: int) -> Tuple[int, int]:
    """Detector rows [v0, v0 + n_rows) every view of slab [z0, z0 + nz) can
    touch (host-only, no device needed)."""
    v0, nr = C.c_uint64(), C.c_uint64()
    g = geo.c()
    N.check(N.lib().tg_cone_slab_rows_geom(C.byref(g), int(z0), int(nz), C.byref(v0), C.byref(nr)))
    return int(v0.value), int(nr.value)


@dataclass
class SlabShard:
    rank: int
    world: int
    z0: int
    nz: int
    v0: int
    n_rows: int


def slab_shards(geo: ConeGeometry, world: int, align: int = Z_ALIGN) -> List[SlabShard]:
    parts = even_partition(geo.volume.shape[2], world, align)
    out = []
    for r, (z0, nz) in enumerate(parts):
        v0, nr = slab_rows(geo, z0, nz) if nz > 0 else (0, 1)
        out.append(SlabShard(r, world, z0, nz, v0, nr))
    return out


def view_partition(geo: ConeGeometry, world: int) -> List[Tuple[int, int]]:
    return even_partition(geo.n_projections, world, 1)


def fdk_slab(geo: ConeGeometry, band: torch.Tensor, shard: SlabShard,
             use_parker: bool = True) -> torch.Tensor:
    """FDK of one z-slab from its raw (unfiltered) detector row band
    [n_proj][n_rows][n_u]: K3 on the band, then K1 on the slab."""
    from .pipelines import fdk_prefilter, fdk_scale
    from .projector import cone_backproject_slab
    filtered = fdk_prefilter(band, geo, use_parker, v0=shard.v0)
    return cone_backproject_slab(geo, filtered, shard.z0, shard.nz, shard.v0,
                                 scale=fdk_scale(geo, use_parker))


def gather_slabs(slab: torch.Tensor, shards: List[SlabShard], group=None) -> torch.Tensor:
    """all_gather the z-slabs into the full [nz][ny][nx] volume on every rank."""
    ny, nx = slab.shape[1], slab.shape[2]
    zmax = max(s.nz for s in shards)
    pad = torch.zeros((zmax, ny, nx), dtype=slab.dtype, device=slab.device)
    pad[: slab.shape[0]] = slab
    bufs = [torch.empty_like(pad) for _ in shards]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: s.nz] for b, s in zip(bufs, shards)], dim=0)


def gather_views(part: torch.Tensor, parts: List[Tuple[int, int]], group=None) -> torch.Tensor:
    """all_gather angle shards [n_views_r][n_v][n_u] into the full sinogram."""
    vmax = max(c for _, c in parts)
    pad = torch.zeros((vmax,) + tuple(part.shape[1:]), dtype=part.dtype, device=part.device)
    pad[: part.shape[0]] = part
    bufs = [torch.empty_like(pad) for _ in parts]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, (_, c) in zip(bufs, parts)], dim=0)


# ---------------------------------------------------------------------------
# collectives over CPU (gloo) or device (NCCL) tensors


def _staged(t: torch.Tensor, group=None):
    """gloo has no device collectives: stage CUDA tensors through the host."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        return t.cpu(), True
    return t, False


def exchange_bands(grad_part: torch.Tensor, view_parts: List[Tuple[int, int]],
                   shards: List[SlabShard], rank: int, group=None) -> torch.Tensor:
    """all_to_all: this rank holds the residual of its views
    ``grad_part`` [n_views_r][n_v][n_u]; every slab owner s receives rows
    [v0_s, v0_s + n_rows_s) of every view.  Returns this rank's band
    [n_proj][n_rows][n_u] (views arrive in rank order = view order)."""
    nu = grad_part.shape[2]
    me = shards[rank]
    send = torch.cat([grad_part[:, s.v0:s.v0 + s.n_rows, :].reshape(-1) for s in shards])
    in_splits = [grad_part.shape[0] * s.n_rows * nu for s in shards]
    out_splits = [c * me.n_rows * nu for _, c in view_parts]
    send_t, staged = _staged(send, group)
    recv = torch.empty(sum(out_splits), dtype=send.dtype, device=send_t.device)
    dist.all_to_all_single(recv, send_t, out_splits, in_splits, group=group)
    if staged:
        recv = recv.to(grad_part.device)
    n_proj = sum(c for _, c in view_parts)
    return recv.view(n_proj, me.n_rows, nu)


def gather_slabs_into(slab: torch.Tensor, shards: List[SlabShard], out: torch.Tensor,
                      group=None) -> torch.Tensor:
    """all_gather z-slabs into the preallocated full volume ``out``."""
    full = gather_slabs(*_staged(slab, group)[:1], shards, group=group)
    out.copy_(full)
    return out


def sum_in_rank_order(values: List[float], device, group=None) -> List[float]:
    """all_gather small FP64 partials and sum them in rank order (the same
    bits on every rank, independent of the collective's reduction order)."""
    t = torch.tensor(values, dtype=torch.float64,
                     device=device if dist.get_backend(group) != "gloo" else "cpu")
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    tot = [0.0] * len(values)
    for b in bufs:
        for i, v in enumerate(b.tolist()):
            tot[i] += v
    return tot


class CudaTvOps:
    """The device operations of one rank of the sharded TV loop (the product
    path: K2, K8, K1, K9 through the C ABI)."""

    def __init__(self, geo: ConeGeometry):
        self.geo = geo

    def forward_views(self, x, v0, n, out):
        from .projector import cone_forward_views
        return cone_forward_views(self.geo, x, v0, n, out=out)

    def residual(self, fp, p, grad):
        from .iterative import l2_residual
        return l2_residual(fp, p, grad)

    def backproject_slab(self, band, shard, out):
        from .projector import cone_backproject_slab
        return cone_backproject_slab(self.geo, band, shard.z0, shard.nz, shard.v0, out=out,
                                     scale=1.0)

    def tv_step(self, x, shard, grad, out, lam, lr):
        from .iterative import tv_step
        nz_all = x.shape[0]
        xs = x[shard.z0:shard.z0 + shard.nz]
        return tv_step(xs, grad, out, lam, lr, has_lo=shard.z0 > 0,
                       has_hi=shard.z0 + shard.nz < nz_all, x_base=x)

    def zeros(self, shape, like):
        return torch.zeros(shape, dtype=torch.float32, device=like.device)


def tv_reconstruct_sharded(geo: ConeGeometry, p_part: torch.Tensor, iterations: int,
                           learning_rate: float, tv_lambda: float, group=None, ops=None,
                           align: int = Z_ALIGN, x0: torch.Tensor = None):
    """pipelines.hpp:273-299 over world ranks.

    p_part: this rank's views [view_partition(geo, world)[rank]] of the
    measured sinogram.  Returns (full image replica, loss history
    [iterations + 1]); raises the reference's divergence Error."""
    from ._native import Error
    ops = ops or CudaTvOps(geo)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    shards = slab_shards(geo, world, align)
    views = view_partition(geo, world)
    me = shards[rank]
    vw0, vwn = views[rank]
    nx, ny, nz = geo.volume.shape
    x = ops.zeros((nz, ny, nx), p_part) if x0 is None else x0.clone()
    fp = ops.zeros((vwn, geo.detector.n_v, geo.detector.n_u), p_part)
    bp = ops.zeros((me.nz, ny, nx), p_part)
    xs = ops.zeros((me.nz, ny, nx), p_part)
    hist = []
    for it in range(iterations + 1):
        ops.forward_views(x, vw0, vwn, fp)
        last = it == iterations
        data = ops.residual(fp, p_part, None if last else fp)
        if last:
            tv = ops.tv_step(x, me, None, None, tv_lambda, learning_rate) if me.nz else 0.0
        else:
            band = exchange_bands(fp, views, shards, rank, group)
            tv = 0.0
            if me.nz:  # more ranks than 32-slice slabs: this rank only projects
                ops.backproject_slab(band, me, bp)
                tv = ops.tv_step(x, me, bp, xs, tv_lambda, learning_rate)
        d, t = sum_in_rank_order([data, tv], p_part.device, group)
        loss = d + t * tv_lambda
        hist.append(loss)
        if not math.isfinite(loss):
            raise Error(f"optimization diverged at iteration {it} (loss is not finite); "
                        "lower the learning rate")
        if not last:
            gather_slabs_into(xs, shards, x, group)
    return x, hist


# ---------------------------------------------------------------------------
# single-node fused path: the exchanges as peer stores inside the kernels


def _device_view(ptr: int, shape, device) -> torch.Tensor:
    """zero-copy float32 tensor over a raw device pointer"""
    class _A:
        __cuda_array_interface__ = {"shape": tuple(int(v) for v in shape), "typestr": "<f4",
                                    "data": (int(ptr), False), "version": 3, "strides": None}
    return torch.as_tensor(_A(), device=device)


class PeerBuffers:
    """Device buffers of this rank that every rank of the node maps through
    CUDA IPC (tg_device_alloc + tg_ipc_*), with the peers' mappings."""

    def __init__(self, nbytes: List[int], device: int, group=None):
        L = N.lib()
        self.device = device
        self.own = []
        for nb in nbytes:
            p = C.c_void_p()
            N.check(L.tg_device_alloc(int(nb), device, C.byref(p)))
            self.own.append(p.value)
        handles = []
        for p in self.own:
            h = (C.c_ubyte * 64)()
            N.check(L.tg_ipc_get_handle(p, h))
            handles.append(bytes(h))
        world = dist.get_world_size(group)
        everyone = [None] * world
        dist.all_gather_object(everyone, handles, group=group)
        me = dist.get_rank(group)
        self.peer = []  # peer[r][i]: buffer i of rank r in this process
        self._opened = []
        for r in range(world):
            if r == me:
                self.peer.append(list(self.own))
                continue
            ptrs = []
            for hb in everyone[r]:
                p = C.c_void_p()
                h = (C.c_ubyte * 64).from_buffer_copy(hb)
                N.check(L.tg_ipc_open_handle(h, device, C.byref(p)))
                ptrs.append(p.value)
                self._opened.append(p.value)
            self.peer.append(ptrs)

    def close(self, group=None):
        """Unmap the peers' buffers, wait until every rank has, then free our own
        (an exporter must outlive every importer's mapping)."""
        L = N.lib()
        for p in self._opened:
            L.tg_ipc_close_handle(p)
        self._opened = []
        dist.barrier(group=group)
        for p in self.own:
            L.tg_device_free(p)
        self.own = []


class P2PUnavailable(RuntimeError):
    """Raised on every rank together when the CUDA-IPC peer buffers of
    tv_reconstruct_p2p cannot be set up on some rank."""


def tv_reconstruct_p2p(geo: ConeGeometry, p_part: torch.Tensor, iterations: int,
                       learning_rate: float, tv_lambda: float, group=None,
                       align: int = Z_ALIGN):
    """The config-5 loop on one node with both exchanges fused into the
    kernels that produce the data (no NCCL data-path collective):

    * K8 scatter (tg_l2_residual_scatter) stores every residual row of this
      rank's views straight into the row band of each slab owner that needs it
      (peer memory over NVLink / NVSwitch);
    * K9 broadcast (tg_tv_step_multi) stores the updated slab into the next
      volume replica of every rank.
    Replicas are double-buffered (ranks read x_i while peers write x_{i+1});
    a stream sync + barrier separates the phases: two host barriers per
    iteration (~0.1 ms each) against ~0.6 s of kernels per iteration per GPU
    at c5 on 8 GPUs, so device-side peer flags would buy < 0.1%.  Bitwise
    equal to tv_reconstruct_sharded and to the single-GPU loop."""
    from ._native import Error
    L = N.lib()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = p_part.device
    dix = dev.index if dev.index is not None else torch.cuda.current_device()
    shards = slab_shards(geo, world, align)
    views = view_partition(geo, world)
    me = shards[rank]
    vw0, vwn = views[rank]
    nx, ny, nz = geo.volume.shape
    nu, nv = geo.detector.n_u, geo.detector.n_v
    plane = nx * ny
    vol_bytes = 4 * nx * ny * nz
    band_bytes = 4 * geo.n_projections * me.n_rows * nu
    # the peer mappings must succeed on every rank, or no rank uses them: the
    # decision is collective (MIN of a flag), so every rank raises
    # P2PUnavailable together and the caller can fall back to the NCCL loop
    # without a half-entered barrier
    bufs, why = None, ""
    try:
        bufs = PeerBuffers([band_bytes, vol_bytes, vol_bytes], dix, group)
    except Exception as e:  # reported collectively below
        why = f"{type(e).__name__}: {e}"
    ok = torch.tensor([0.0 if bufs is None else 1.0], dtype=torch.float64,
                      device="cpu" if dist.get_backend(group) == "gloo" else dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if float(ok) < 1.0:
        if bufs is not None:
            bufs.close(group)
        raise P2PUnavailable(why or "a peer rank could not map the CUDA-IPC buffers")
    plan = geo._plan(dix)
    st = torch.cuda.current_stream(dev).cuda_stream
    fp = torch.empty((vwn, nv, nu), dtype=torch.float32, device=dev)
    bp = torch.empty((me.nz, ny, nx), dtype=torch.float32, device=dev)
    sums = torch.zeros(2 * (iterations + 1), dtype=torch.float64, device=dev)
    p_part = p_part.contiguous()
    dests = (N.tg_band_dest * world)(*[N.tg_band_dest(bufs.peer[r][0], s.v0, s.n_rows)
                                       for r, s in enumerate(shards)])
    band = bufs.own[0]
    cur, nxt = 1, 2

    def sync_all():
        torch.cuda.current_stream(dev).synchronize()
        dist.barrier(group=group)

    try:
        sync_all()  # every rank's buffers exist and are zero
        for it in range(iterations + 1):
            last = it == iterations
            x_own = bufs.peer[rank][cur]
            N.check(L.tg_cone_forward_views(plan, vw0, vwn, x_own, fp.data_ptr(), st))
            d_sum = sums.data_ptr() + 8 * (2 * it)
            d_tv = sums.data_ptr() + 8 * (2 * it + 1)
            if last:
                N.check(L.tg_l2_residual(fp.data_ptr(), p_part.data_ptr(), None, fp.numel(), d_sum, st))
                if me.nz:
                    N.check(L.tg_tv_step(x_own + 4 * me.z0 * plane, None, None, nx, ny, me.nz,
                                         int(me.z0 > 0), int(me.z0 + me.nz < nz), float(tv_lambda),
                                         float(learning_rate), d_tv, st))
                break
            N.check(L.tg_l2_residual_scatter(fp.data_ptr(), p_part.data_ptr(), vwn, nv, nu, vw0,
                                             dests, world, d_sum, st))
            sync_all()  # every band complete
            if me.nz:  # more ranks than 32-slice slabs: this rank only projects
                N.check(L.tg_cone_backproject_slab(plan, me.z0, me.nz, me.v0, me.n_rows, band,
                                                   bp.data_ptr(), 1.0, 0, st))
                outs = (C.c_void_p * world)(*[bufs.peer[r][nxt] + 4 * me.z0 * plane
                                              for r in range(world)])
                N.check(L.tg_tv_step_multi(x_own + 4 * me.z0 * plane, bp.data_ptr(), outs, world,
                                           nx, ny, me.nz, int(me.z0 > 0), int(me.z0 + me.nz < nz),
                                           float(tv_lambda), float(learning_rate), d_tv, st))
            sync_all()  # every slab in every next replica
            cur, nxt = nxt, cur
            # stop together at the first non-finite loss (pipelines.hpp:166-170
            # checks every iteration): this rank's two partials of iteration
            # `it` are final after the barrier; one MIN over ranks of a flag
            part = sums[2 * it:2 * it + 2].cpu()
            ok = torch.tensor([1.0 if math.isfinite(float(part[0]) + float(part[1])) else 0.0],
                              dtype=torch.float64,
                              device="cpu" if dist.get_backend(group) == "gloo" else dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if float(ok) < 1.0:
                iterations = it
                break
        # loss partials of all ranks, summed in rank order
        world_sums = [torch.empty_like(sums) for _ in range(world)]
        if dist.get_backend(group) == "gloo":
            host = sums.cpu()
            tmp = [torch.empty_like(host) for _ in range(world)]
            dist.all_gather(tmp, host, group=group)
            world_sums = tmp
        else:
            dist.all_gather(world_sums, sums, group=group)
        tot = torch.zeros(2 * (iterations + 1), dtype=torch.float64)
        for w in world_sums:
            tot += w.cpu()
        hist = []
        for it in range(iterations + 1):
            loss = float(tot[2 * it]) + float(tot[2 * it + 1]) * tv_lambda
            hist.append(loss)
            if not math.isfinite(loss):
                raise Error(f"optimization diverged at iteration {it} (loss is not finite); "
                            "lower the learning rate")
        x = _device_view(bufs.peer[rank][cur], (nz, ny, nx), dev).clone()
        return x, hist
    finally:
        sync_all()
        bufs.close(group)
