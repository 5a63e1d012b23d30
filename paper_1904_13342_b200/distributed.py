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
  ``gather_slabs`` (all_gather of z-slabs) and ``gather_views``.
"""
from __future__ import annotations

import ctypes as C
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


def slab_shards(geo: ConeGeometry, world: int) -> List[SlabShard]:
    parts = even_partition(geo.volume.shape[2], world, Z_ALIGN)
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
