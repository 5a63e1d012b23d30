"""Multi-process sharding logic on CPU (gloo, world_size 2): each rank owns a
32-aligned z-slab and only the detector row band its slab projects onto,
back-projects it (CPU oracle standing in for K1), and the slabs are
all_gathered; the result must equal the single-process full volume.  The
forward projector shards by angle and gathers views the same way."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    import paper_1904_13342_b200 as tg
    from paper_1904_13342_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vol = tg.VolumeSpec.centered([24, 24, 40], [1.0, 1.0, 1.0])
        det = tg.Detector2D.centered(40, 48, 1.5, 1.5)
        geo = tg.make_cone(vol, det, 18, 2 * math.pi, 120.0, 220.0)
        shards = D.slab_shards(geo, world)
        me = shards[rank]
        assert me.z0 % D.Z_ALIGN == 0
        sino = np.random.default_rng(3).uniform(-1, 1, (18, 48, 40)).astype(np.float32)
        band = sino[:, me.v0:me.v0 + me.n_rows]
        # this rank's slab from its band only: the full detector with zeros
        # outside the band (rows the slab never taps)
        only_band = np.zeros_like(sino)
        only_band[:, me.v0:me.v0 + me.n_rows] = band
        origin = list(vol.origin)
        origin[2] = vol.origin[2] + me.z0 * vol.spacing[2]
        ov = O.make_volume([24, 24, me.nz], vol.spacing, origin)
        od = O.det2_centered(40, 48, 1.5, 1.5)
        og = O.cone_from_matrices(ov, od, geo.angular_range, geo.sid, geo.sdd, geo.matrices)
        slab = torch.from_numpy(O.cone_backproject(og, only_band))
        full = D.gather_slabs(slab, shards)
        # forward projection sharded by angle
        ph = O.shepp_logan_3d(O.make_volume(vol.shape, vol.spacing))
        parts = D.view_partition(geo, world)
        v0, vn = parts[rank]
        ogf = O.cone_from_matrices(O.make_volume(vol.shape, vol.spacing), od, geo.angular_range,
                                   geo.sid, geo.sdd, geo.matrices[v0:v0 + vn])
        sinos = D.gather_views(torch.from_numpy(O.cone_forward(ogf, ph)), parts)
        if rank == 0:
            q.put((full.numpy(), sinos.numpy()))
    finally:
        dist.destroy_process_group()


def test_slab_and_view_sharding_world2():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, sinos = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    vol = O.make_volume([24, 24, 40], [1.0] * 3)
    og = O.make_cone(vol, O.det2_centered(40, 48, 1.5, 1.5), 18, 2 * math.pi, 120.0, 220.0)
    sino = np.random.default_rng(3).uniform(-1, 1, (18, 48, 40)).astype(np.float32)
    ref = O.cone_backproject(og, sino)
    mx, rr = O.rel_errors(full, ref)
    assert rr < 1e-12 and mx < 1e-12  # shifted-origin slabs: last-bit coordinate differences only
    assert np.array_equal(sinos, O.cone_forward(og, O.shepp_logan_3d(vol)))


def test_even_partition():
    from paper_1904_13342_b200.distributed import even_partition
    assert even_partition(512, 8, 16) == [(i * 64, 64) for i in range(8)]
    p = even_partition(100, 3, 16)
    assert sum(c for _, c in p) == 100 and all(s % 16 == 0 for s, _ in p)
    assert even_partition(496, 8) == [(i * 62, 62) for i in range(8)]
