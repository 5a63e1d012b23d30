"""CPU: the device graph's builders and feed checks mirror graph.hpp's
shape rules and exact messages (graph.hpp:104-216) — host logic only, no
kernel runs."""
import math

import numpy as np
import pytest
import torch

import paper_1904_13342_b200 as tg
from paper_1904_13342_b200.graph import Graph, OpKind, sino_shape, volume_shape


def _geo():
    vol = tg.VolumeSpec.centered([45, 40], [1.0, 1.0])
    return tg.make_parallel(vol, tg.Detector1D.centered(64, 1.0), 60, math.pi)


def _raises(msg, fn, *a):
    with pytest.raises(tg.Error) as e:
        fn(*a)
    assert str(e.value) == msg


def test_shapes_are_fastest_first():
    geo = _geo()
    assert volume_shape(geo) == [45, 40]
    assert sino_shape(geo) == [64, 60]
    cone = tg.make_cone(tg.VolumeSpec.centered([8, 7, 6], [1.0] * 3),
                        tg.Detector2D.centered(12, 10, 1.0, 1.0), 9, 2 * math.pi, 100.0, 200.0)
    assert sino_shape(cone) == [12, 10, 9]


def test_builder_checks_and_messages():
    geo = _geo()
    g = Graph()
    x = g.input([45, 40])
    p = g.input([64, 60])
    bad = g.input([40, 45])
    _raises("forward_project input shape does not match the geometry volume",
            g.forward_project, bad, geo)
    _raises("backproject input shape does not match the geometry sinogram", g.backproject, x, geo)
    fp = g.forward_project(x, geo)
    assert g.node(fp).shape == [64, 60] and g.node(fp).kind == OpKind.forward_project
    w_row = g.input([64])
    w_bad = g.input([60])
    assert g.node(g.multiply_weights(fp, w_row)).shape == [64, 60]
    _raises("weight shape must equal the input shape or a prefix of it", g.multiply_weights, fp,
            w_bad)
    k = g.input([128])
    _raises("filter window must be a power of two", g.fourier_filter, p, k, 96)
    _raises("filter window is smaller than the detector row", g.fourier_filter, p, k, 32)
    _raises("filter weight vector must have length padded_n", g.fourier_filter, p, k, 256)
    assert g.node(g.fourier_filter(p, k, 128)).padded_n == 128
    _raises("add expects matching shapes", g.add, x, p)
    _raises("l2_loss expects matching shapes", g.l2_loss, x, p)
    l2 = g.l2_loss(fp, p)
    assert g.node(l2).shape == []
    _raises("tv_loss needs a non-scalar input", g.tv_loss, l2)
    _raises("node id out of range", g.scale, 999, 2.0)
    assert g.node(g.scale(l2, 0.5)).factor == 0.5


def test_feed_checks_and_messages():
    geo = _geo()
    g = Graph()
    x = g.input([45, 40])
    fp = g.forward_project(x, geo)
    _raises("feed id does not name an input node", g.forward, {fp: torch.zeros(60, 64)})
    _raises("feed shape mismatch", g.forward, {x: torch.zeros(45, 40)})
    _raises("missing feed for input node", g.forward, {})
    _raises("run forward before backward", g.backward, fp)
    _raises("node has no value; run forward first", g.value, fp)


def test_trainable_parameters_listing():
    g = Graph()
    a = g.parameter(1.0, trainable=True)
    b = g.parameter(2.0, trainable=False)
    c = g.parameter(3.0)
    assert g.trainable_parameters() == [a, c]
    assert g.size() == 3 and not g.node(b).trainable


def test_scalar_graph_runs_on_host_values():
    """scalar-only graphs (losses) need no device: the reference's scalar
    arithmetic, forward and reverse (graph.hpp:318-353, 498-531)."""
    g = Graph()
    a = g.parameter(3.0)
    b = g.input([])
    loss = g.add(g.l2_loss(a, b), g.scale(a, 0.5))
    g.forward({b: 1.0})
    assert g.value(loss) == 4.0 + 1.5
    grads = g.backward(loss)
    assert grads[a] == 2.0 * (3.0 - 1.0) + 0.5
    tg.gradient_descent_step(g, grads, 0.1)
    assert g.node(a).value == pytest.approx(3.0 - 0.1 * 4.5)
