"""CPU: the Python mirror fails loudly and with the reference's messages
before any device work — no CPU fallback for the iterative pieces, shape
checks of tv_reconstruct, distributed partition helpers."""
import math

import numpy as np
import pytest
import torch


def test_iterative_pieces_need_device_tensors(tg):
    x = torch.zeros(4, 5)
    with pytest.raises(tg.Error, match="must live on a CUDA device"):
        tg.tv_step(x)
    with pytest.raises(tg.Error, match="must live on a CUDA device"):
        tg.l2_residual(x, x)
    with pytest.raises(tg.Error, match="l2_loss expects matching shapes"):
        tg.l2_residual(torch.zeros(3), torch.zeros(4))


def test_tv_reconstruct_checks_the_sinogram_shape(tg):
    vol = tg.VolumeSpec.centered([16, 16], [1.0, 1.0])
    geo = tg.make_parallel(vol, tg.Detector1D.centered(23, 1.0), 8, math.pi)
    bad = tg.Sinogram.planar(8, tg.Detector1D.centered(25, 1.0), host=True)
    with pytest.raises(tg.Error, match="sinogram shape does not match the geometry"):
        tg.tv_reconstruct(bad, geo, tg.ExperimentConfig(iterations=1))


def test_make_phantom_2d_unknown_name(tg):
    from paper_1904_13342_b200.iterative import make_phantom_2d
    with pytest.raises(tg.Error, match="unknown phantom: spiral"):
        make_phantom_2d("spiral", tg.VolumeSpec.centered([8, 8], [1.0, 1.0]))


def test_slab_shards_cover_the_volume_once(tg):
    from paper_1904_13342_b200 import distributed as D
    vol = tg.VolumeSpec.centered([64, 64, 200], [1.0] * 3)
    geo = tg.make_cone(vol, tg.Detector2D.centered(96, 200, 1.0, 1.0), 12, 2 * math.pi, 300.0, 600.0)
    for world in (1, 2, 3, 5, 8):
        sh = D.slab_shards(geo, world)
        z = 0
        for s in sh:
            assert s.z0 == z and s.z0 % D.Z_ALIGN == 0 or s.nz == 0
            assert s.v0 + s.n_rows <= 200
            z += s.nz
        assert z == 200
        views = D.view_partition(geo, world)
        assert sum(c for _, c in views) == 12


def test_band_rows_contain_every_tap(tg):
    """slab_rows is conservative: every voxel of the slab projects inside the
    band on every view (FP64 host check against the projection matrices)"""
    from paper_1904_13342_b200 import distributed as D
    vol = tg.VolumeSpec.centered([32, 32, 64], [1.0] * 3)
    geo = tg.make_cone(vol, tg.Detector2D.centered(64, 128, 1.2, 1.2), 24, 2 * math.pi, 200.0, 400.0)
    P = np.asarray(geo.matrices).reshape(-1, 3, 4)
    o = np.asarray(vol.origin)
    sp = np.asarray(vol.spacing)
    for s in D.slab_shards(geo, 4):
        if s.nz == 0:
            continue
        zs = o[2] + sp[2] * np.arange(s.z0, s.z0 + s.nz)
        xs = o[0] + sp[0] * np.arange(32)
        ys = o[1] + sp[1] * np.arange(32)
        X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
        pts = np.stack([X.ravel(), Y.ravel(), Z.ravel(), np.ones(X.size)])
        for M in P:
            h = M @ pts
            v = h[1] / h[2]
            assert np.floor(v).min() >= s.v0 - 1e-9
            assert np.floor(v).max() + 1 <= s.v0 + s.n_rows - 1 + 1e-9
