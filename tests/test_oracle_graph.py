"""CPU: the graph-level restatements pinned to the reference itself
(oracle/_ref): experiment_learn_filter's graph (pipelines.hpp:196-261 —
fourier_filter forward and weight gradient, backproject and its registered
gradient, scale, l2) bit-for-bit in float64, and the reference glue that runs
the same graph on a given sinogram against the reference experiment."""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _learn_geometry(n_img=45, nb=64, n=60):
    # configs/learn_filter_geometry.json: 45^2 @ 1 mm, 64 bins @ 1 mm, 60 views / 180 deg
    v = O.make_volume([n_img, n_img], [1.0, 1.0])
    d = O.det1_centered(nb, 1.0)
    return O.make_planar(v, d, n, math.pi), O.Ref.planar_geometry(v, d, n, math.pi), v


def test_learn_filter_glue_equals_reference_experiment():
    g, gr, v = _learn_geometry()
    # noise-free run: the glue's sinogram is the reference's own FP of its phantom
    l1, d1, w1, r1 = O.Ref.experiment_learn_filter(gr, "shepp-logan", 0.0, 1337, 64, 1.5e-5, 6)
    sino = O.Ref.planar_forward(gr, O.Ref.shepp_logan_2d(v, np.float64))
    l2, d2, w2, r2 = O.Ref.learn_filter_graph(gr, sino, 64, 1.5e-5, 6)
    for a, b in ((l1, l2), (d1, d2), (w1, w2), (r1, r2)):
        assert np.array_equal(a, b)
    assert d1[-1] < d1[0]  # descent moves the ramp toward Ram-Lak


def test_learn_filter_restatement_bitwise_f64():
    g, gr, v = _learn_geometry()
    sino = O.planar_forward(g, O.shepp_logan_2d(v, np.float64))
    a = O.learn_filter_planar(g, sino, 64, 1.5e-5, 8)
    b = O.Ref.learn_filter_graph(gr, sino, 64, 1.5e-5, 8)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert a[0][-1] < a[0][0]


def test_learn_filter_restatement_bitwise_default_window():
    g, gr, v = _learn_geometry(24, 33, 16)
    sino = O.planar_forward(g, O.shepp_logan_2d(v, np.float64))
    P = O.filter_window(33)
    a = O.learn_filter_planar(g, sino, P, 1e-5, 3)
    b = O.Ref.learn_filter_graph(gr, sino, P, 1e-5, 3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_graph_probe_gradients_restated():
    """multiply_weights / tv / add / scale / forward_project gradients of the
    reference Graph against the restated pieces (graph.hpp:436-528)."""
    g, gr, v = _learn_geometry(20, 29, 9)
    rs = np.random.default_rng(7)
    x0 = rs.random(g.img_shape_yx)
    w0 = 0.5 + rs.random(29)
    sino = rs.random(g.sino_shape)
    lam = 0.7
    loss, gx, gw = O.Ref.graph_probe(gr, x0, w0, sino, lam)
    fp = O.planar_forward(g, x0)
    mw = fp * w0[None, :]
    d = mw - sino
    assert loss == pytest.approx(float(np.sum(d * d)) + lam * O.tv_value(x0), rel=1e-13)
    gmw = 2.0 * d
    np.testing.assert_allclose(gw, np.sum(gmw * fp, axis=0), rtol=1e-12)
    gfp = gmw * w0[None, :]
    want = O.planar_backproject(g, gfp) + O.tv_subgrad(x0, lam)
    np.testing.assert_allclose(gx, want, rtol=1e-11, atol=1e-11 * np.abs(want).max())
