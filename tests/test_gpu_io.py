"""GPU: data read through the file formats (pinned host payload -> one DMA
to HBM) drives the device path identically to in-memory data; a calibrated
geometry file (explicit, non-circular projection matrices) runs the general
K1 / K2 paths and matches the oracle."""
import json
import math

import numpy as np
import pytest
import torch

import oracle as O
from _helpers import assert_close
from paper_1904_13342_b200 import io as tio

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def test_calibrated_geometry_file_drives_general_paths(tg, tmp_path):
    vol = tg.VolumeSpec.centered([40, 36, 32], [1.0] * 3)
    det = tg.Detector2D.centered(64, 56, 1.6, 1.6)
    circ = tg.make_cone(vol, det, 30, 2 * math.pi, 300.0, 600.0)
    m = np.asarray(circ.matrices).reshape(-1, 12).copy()
    rng = np.random.default_rng(7)
    m[:, [0, 1, 4, 5]] *= 1.0 + 1e-3 * rng.standard_normal((30, 4))  # detector tilt / skew
    m[:, 2] += 1e-2 * rng.standard_normal(30)                          # P[0][2] != 0
    m[:, 10] += 1e-4 * rng.standard_normal(30)                         # P[2][2] != 0
    j = {"type": "cone3d", "volume_shape": [40, 36, 32], "volume_spacing": [1.0] * 3,
         "detector_shape": [64, 56], "detector_spacing": [1.6, 1.6], "n_projections": 30,
         "angular_range_deg": 360.0, "sid": 300.0, "sdd": 600.0,
         "projection_matrices": m.tolist()}
    (tmp_path / "geo.json").write_text(json.dumps(j))
    geo = tio.load_geometry(str(tmp_path / "geo.json"))
    assert not geo.circular
    ov = O.make_volume(vol.shape, vol.spacing, vol.origin)
    od = O.or_det2(det.n_u, det.n_v, det.spacing_u, det.spacing_v, det.origin_u, det.origin_v)
    og = O.cone_from_matrices(ov, od, 2 * math.pi, 300.0, 600.0, m)
    assert np.array_equal(np.asarray(geo.matrices).reshape(-1, 12), og.mats)
    ph = tg.shepp_logan_3d(vol, device=DEV)
    sino = tg.forward_project(ph, geo)
    assert_close(sino.data.cpu().numpy(), O.cone_forward(og, ph.data.cpu().numpy()), what="FP")
    # write / read back (pinned, to the device) and back-project
    tio.write_sinogram(str(tmp_path / "p.json"), sino)
    back = tio.read_sinogram(str(tmp_path / "p.json"), geo, device=DEV)
    assert torch.equal(back.data, sino.data)
    bp = tg.back_project(back, geo)
    assert_close(bp.data.cpu().numpy(), O.cone_backproject(og, sino.data.cpu().numpy()), what="BP")


def test_image_read_to_device(tg, tmp_path):
    vol = tg.VolumeSpec.centered([32, 30, 28], [0.5] * 3)
    ph = tg.shepp_logan_3d(vol, device=DEV)
    tio.write_image(str(tmp_path / "ph.json"), ph)
    back = tio.read_image(str(tmp_path / "ph.json"), device=DEV)
    assert back.data.is_cuda and torch.equal(back.data, ph.data)
