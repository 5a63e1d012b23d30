"""Re-entrancy of the drop-in on ONE plan (projector.hpp:16-17: the
reference's operators are pure functions, callable from any thread).

Several host threads call back_project / forward_project with the same
geometry (hence the same cached plan) at once — through the host-buffer
C-ABI path (plan-owned staging and pipeline streams) and through the device
path on per-thread torch streams (plan-owned scratch: the K2 transposed
volume, the K1 re-pitch buffer, the shared constant bank).  Every result must
equal the single-threaded one bit for bit.  ctypes releases the GIL inside
the C calls, so the calls really overlap."""
import math
import threading

import numpy as np
import pytest
import torch

from _helpers import rand

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def geo(tg):
    vol = tg.VolumeSpec.centered([64, 60, 56], [1.0] * 3)
    det = tg.Detector2D.centered(90, 80, 1.3, 1.3)
    return tg.make_cone(vol, det, 72, 2 * math.pi, 300.0, 600.0)


def _run_threads(fn, n):
    errs, outs = [], [None] * n

    def body(i):
        try:
            outs[i] = fn(i)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=body, args=(i,)) for i in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return outs


def test_two_threads_host_backproject_one_plan(tg, geo):
    sinos = [rand((72, 80, 90), 40 + i, -1, 1) for i in range(2)]
    want = [tg.back_project(tg.Sinogram.cone_beam(72, geo.detector, data=s), geo).data
            for s in sinos]

    def call(i):
        res = []
        for _ in range(4):
            res.append(tg.back_project(tg.Sinogram.cone_beam(72, geo.detector, data=sinos[i]),
                                       geo).data.copy())
        return res

    outs = _run_threads(call, 2)
    for i in range(2):
        for o in outs[i]:
            assert np.array_equal(o, want[i])


def test_threads_device_paths_one_plan(tg, geo):
    """forward and back projection of different inputs on per-thread streams"""
    vols = [torch.from_numpy(rand((56, 60, 64), 50 + i)).to(DEV) for i in range(3)]
    sinos = [torch.from_numpy(rand((72, 80, 90), 60 + i, -1, 1)).to(DEV) for i in range(3)]
    want_fp = [tg.forward_project(tg.Image(geo.volume, v), geo).data.clone() for v in vols]
    want_bp = [tg.back_project(tg.Sinogram.cone_beam(72, geo.detector, data=s), geo).data.clone()
               for s in sinos]
    torch.cuda.synchronize()

    def call(i):
        st = torch.cuda.Stream(device=DEV)
        res = []
        with torch.cuda.stream(st):
            for _ in range(3):
                fp = tg.forward_project(tg.Image(geo.volume, vols[i]), geo).data
                bp = tg.back_project(tg.Sinogram.cone_beam(72, geo.detector, data=sinos[i]),
                                     geo).data
                res.append((fp, bp))
        st.synchronize()
        return res

    outs = _run_threads(call, 3)
    for i in range(3):
        for fp, bp in outs[i]:
            assert torch.equal(fp, want_fp[i])
            assert torch.equal(bp, want_bp[i])


def test_threads_mixed_host_and_device_one_plan(tg, geo):
    """a host-buffer FDK and device forward projections interleaved on one plan"""
    s_host = rand((72, 80, 90), 70, -1, 1)
    vol = torch.from_numpy(rand((56, 60, 64), 71)).to(DEV)
    want_rec = tg.fdk_reconstruct(tg.Sinogram.cone_beam(72, geo.detector, data=s_host), geo,
                                  use_parker=False).data
    want_fp = tg.forward_project(tg.Image(geo.volume, vol), geo).data.clone()
    torch.cuda.synchronize()

    def call(i):
        if i == 0:
            return [tg.fdk_reconstruct(tg.Sinogram.cone_beam(72, geo.detector, data=s_host), geo,
                                       use_parker=False).data.copy() for _ in range(3)]
        st = torch.cuda.Stream(device=DEV)
        with torch.cuda.stream(st):
            r = [tg.forward_project(tg.Image(geo.volume, vol), geo).data for _ in range(6)]
        st.synchronize()
        return r

    outs = _run_threads(call, 2)
    for o in outs[0]:
        assert np.array_equal(o, want_rec)
    for o in outs[1]:
        assert torch.equal(o, want_fp)
