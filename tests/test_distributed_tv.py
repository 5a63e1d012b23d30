"""The sharded config-5 loop (distributed.tv_reconstruct_sharded) on CPU with
gloo at world_size 1, 2 and 3: angle-sharded forward projection, the
all_to_all of residual row bands to slab owners, slab back-projection, the
halo TV step and the slab all_gather.  The device operations are replaced by
the CPU oracle (test infrastructure: ``OracleTvOps`` below), so the test
checks the decomposition itself: the image must be BIT-identical to the
single-process fp32-storage oracle loop at every world size (the loss equal
to 1e-12: only the FP64 summation grouping differs)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPE, DET, NPROJ = (20, 18, 24), (30, 26, 1.5, 1.5), 14
ITERS, LR, LAM = 4, 5e-4, 0.5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleTvOps:
    """CPU stand-ins for K2 / K8 / K1 / K9 (checker only)."""

    def __init__(self, O, og):
        self.O, self.og = O, og

    def zeros(self, shape, like):
        return torch.zeros(shape, dtype=torch.float32)

    def forward_views(self, x, v0, n, out):
        out.copy_(torch.from_numpy(self.O.cone_forward(self.og, x.numpy())[v0:v0 + n]))

    def residual(self, fp, p, grad):
        d = fp.numpy().astype(np.float64) - p.numpy().astype(np.float64)
        if grad is not None:
            grad.copy_(torch.from_numpy((2.0 * d).astype(np.float32)))
        return float(np.sum(d * d))

    def backproject_slab(self, band, shard, out):
        full = np.zeros((self.og.n_proj, int(self.og.det.n_v), int(self.og.det.n_u)), np.float32)
        full[:, shard.v0:shard.v0 + shard.n_rows] = band.numpy()
        out.copy_(torch.from_numpy(self.O.cone_backproject(self.og, full)[shard.z0:shard.z0 + shard.nz]))

    def tv_step(self, x, shard, grad, out, lam, lr):
        xa = x.numpy()
        z0, z1 = shard.z0, shard.z0 + shard.nz
        tv = self.O.tv_value(np.ascontiguousarray(xa[z0:z1]))
        if z1 < xa.shape[0]:
            tv += float(np.sum(np.abs(xa[z1].astype(np.float64) - xa[z1 - 1].astype(np.float64))))
        if out is not None:
            s = self.O.tv_subgrad(xa, 1.0)[z0:z1]
            new = xa[z0:z1].astype(np.float64) - lr * (lam * s + grad.numpy().astype(np.float64))
            out.copy_(torch.from_numpy(new.astype(np.float32)))
        return tv


def _setup(O):
    import paper_1904_13342_b200 as tg
    vol = tg.VolumeSpec.centered(list(SHAPE), [1.0] * 3)
    geo = tg.make_cone(vol, tg.Detector2D.centered(*DET), NPROJ, 2 * math.pi, 100.0, 200.0)
    ov = O.make_volume(vol.shape, vol.spacing, vol.origin)
    og = O.make_cone(ov, O.det2_centered(*DET), NPROJ, 2 * math.pi, 100.0, 200.0)
    sino = O.cone_forward(og, O.shepp_logan_3d(ov))
    return geo, og, sino


def _worker(rank, world, port, q, align=1):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_1904_13342_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        geo, og, sino = _setup(O)
        v0, vn = D.view_partition(geo, world)[rank]
        p = torch.from_numpy(np.ascontiguousarray(sino[v0:v0 + vn]))
        x, hist = D.tv_reconstruct_sharded(geo, p, ITERS, LR, LAM, ops=OracleTvOps(O, og),
                                           align=align)
        q.put((rank, x.numpy(), hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,align", [(1, 1), (2, 1), (3, 1), (3, 16)])
def test_sharded_tv_loop_bitwise_vs_single_process(world, align):
    """(3, 16): slabs of 16, 8 and 0 slices — the last rank only projects"""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, align)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, og, sino = _setup(O)
    xr, hr = O.tv_reconstruct_cone(og, sino, ITERS, LR, LAM)
    for rank, x, hist in got:
        assert np.array_equal(x, xr), f"rank {rank} image differs"
        assert np.max(np.abs(np.array(hist) - hr) / hr) <= 1e-12
    # every rank reports the same loss bits
    assert all(g[2] == got[0][2] for g in got)


def test_exchange_bands_layout():
    """single process: the band a slab owner receives is the row band of the
    full residual, views in order"""
    from paper_1904_13342_b200 import distributed as D
    f = os.path.join("/tmp", f"tg_pg_{os.getpid()}")
    dist.init_process_group("gloo", init_method=f"file://{f}", rank=0, world_size=1)
    try:
        g = torch.arange(5 * 7 * 3, dtype=torch.float32).view(5, 7, 3)
        shard = D.SlabShard(0, 1, 0, 4, 2, 3)
        band = D.exchange_bands(g, [(0, 5)], [shard], 0)
        assert torch.equal(band, g[:, 2:5, :])
    finally:
        dist.destroy_process_group()
        if os.path.exists(f):
            os.unlink(f)
