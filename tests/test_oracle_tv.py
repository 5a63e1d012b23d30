"""CPU: the iterative-reconstruction restatement (oracle/tg_oracle_body.inc:
l2 / TV / descent loop, Gaussian noise) pinned bit-for-bit to the reference
itself (oracle/_ref: pipelines.hpp:273-299 tv_reconstruct and the same graph
over fan / cone geometry; pipelines.hpp:119-132 add_gaussian_noise), plus the
product's host noise generator against both."""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64
    assert O.mt19937_64(5489, 10000) == 9981545732273789042


def _planar(n_img, nb, n, rng, sid=0.0, sdd=0.0):
    v = O.make_volume([n_img, n_img - 4], [1.0, 1.0])
    d = O.det1_centered(nb, 1.0)
    return (O.make_planar(v, d, n, rng, sid, sdd),
            O.Ref.planar_geometry(v, d, n, rng, sid, sdd), v)


def test_tv_parallel_bitwise_vs_reference():
    # the reference's own iterative_tv parameters (configs/iterative_tv.json)
    g, gr, v = _planar(32, 45, 12, math.pi)
    sino = O.planar_forward(g, O.shepp_logan_2d(v, np.float64))
    x1, h1 = O.tv_reconstruct_planar(g, sino, 10, 1.5e-4, 3.0)
    x2, h2 = O.Ref.tv_reconstruct_planar(gr, sino, 10, 1.5e-4, 3.0)
    assert np.array_equal(x1, x2) and np.array_equal(h1, h2)
    assert h1[-1] < h1[0]


def test_tv_fan_bitwise_vs_reference_graph():
    g, gr, v = _planar(32, 45, 12, 2 * math.pi, 300.0, 600.0)
    sino = O.planar_forward(g, O.shepp_logan_2d(v, np.float64))
    x1, h1 = O.tv_reconstruct_planar(g, sino, 6, 1e-4, 0.7)
    x2, h2 = O.Ref.tv_reconstruct_planar(gr, sino, 6, 1e-4, 0.7)
    assert np.array_equal(x1, x2) and np.array_equal(h1, h2)


def test_tv_cone_bitwise_vs_reference_graph():
    v3 = O.make_volume([12, 10, 8], [1.0] * 3)
    gc = O.make_cone(v3, O.det2_centered(20, 16, 1.5, 1.5), 10, 2 * math.pi, 100.0, 200.0)
    sino = O.cone_forward(gc, O.shepp_logan_3d(v3, np.float64))
    x1, h1 = O.tv_reconstruct_cone(gc, sino, 4, 1e-4, 0.3)
    x2, h2 = O.Ref.tv_reconstruct_cone(gc, sino, 4, 1e-4, 0.3)
    assert np.array_equal(x1, x2) and np.array_equal(h1, h2)


def test_tv_divergence_message_matches_reference():
    g, gr, v = _planar(16, 23, 6, math.pi)
    sino = O.planar_forward(g, O.shepp_logan_2d(v, np.float64))
    msgs = []
    for fn, geo in ((O.tv_reconstruct_planar, g), (O.Ref.tv_reconstruct_planar, gr)):
        with pytest.raises(O.OracleError) as e:
            fn(geo, sino * 1e200, 50, 1e10, 0.0)
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]
    assert msgs[0].startswith("optimization diverged at iteration ")
    assert msgs[0].endswith(" (loss is not finite); lower the learning rate")


def test_tv_value_and_subgradient_known_answers():
    x = np.array([[0.0, 1.0, 1.0], [3.0, 1.0, 0.0]])
    # forward pairs: x-axis |1|+|0|+|-2|+|-1| = 4, y-axis |3|+|0|+|-1| = 4
    assert O.tv_value(x) == 8.0
    g = O.tv_subgrad(x, 1.0)
    # voxel (0,0): -sgn(1) (x) - sgn(3) (y) = -2 ; voxel (1,0): +sgn(3) - sgn(-2) = 2
    assert g[0, 0] == -2.0 and g[1, 0] == 2.0
    assert g.sum() == 0.0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_noise_bitwise_vs_reference(dtype):
    a = np.random.default_rng(3).uniform(0, 5, 4097).astype(dtype)
    assert np.array_equal(O.add_gaussian_noise(a, 0.02, 1337), O.Ref.add_gaussian_noise(a, 0.02, 1337))
    assert np.array_equal(O.add_gaussian_noise(a, 0.0, 1), a)


def test_product_host_noise_bitwise(tg):
    a = np.random.default_rng(4).uniform(0, 5, (12, 45)).astype(np.float32)
    s = tg.Sinogram.planar(12, tg.Detector1D.centered(45, 1.0), data=a.copy())
    out = tg.add_gaussian_noise(s, 0.02, 1337)
    assert np.array_equal(out.data, O.Ref.add_gaussian_noise(a, 0.02, 1337))
    with pytest.raises(tg.Error, match="noise level must be non-negative"):
        tg.add_gaussian_noise(s, -1.0, 1)
