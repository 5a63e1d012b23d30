"""GPU parity of the device graph (graph.py over graph.cu / K1-K9, SURVEY
§8f row 1) and of the torch.autograd operators.

Oracles: the reference's own Graph (oracle/_ref: ref_graph_probe,
ref_learn_filter_graph, ref_experiment_learn_filter) and the C restatement of
the learn-filter loop (bitwise to the reference, tests/test_oracle_graph.py).

Tolerances (stated): single operators as SURVEY §8c (relRMSE 1e-5, max 1e-4;
the row filter FILTER_REL_RMSE); a one-pass graph of three operators (probe)
5e-5 / 5e-4; the weight gradient (a sum over rows of products of fp32 FFT
outputs) 1e-5 relRMSE.  The learn-filter loop is smooth (quadratic in K), so
the device loop is held to the FP64 reference at no more than 2x the
fp32-storage oracle's own drift (floors 1e-5 loss, 1e-5 weights)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from _helpers import FILTER_REL_RMSE, assert_close, planar_pair, rand

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(DEV)


@pytest.mark.parametrize("n,P", [(64, 128), (45, 64), (365, 1024), (1248, 4096), (20, 32)])
@pytest.mark.parametrize("sym", [True, False])
def test_fourier_filter_device_weights(tg, n, P, sym):
    rows = rand((37, n), 11, -1.0, 1.0)
    if sym:
        k = tg.ramlak_weights(P, 0.7)
    else:
        k = np.random.default_rng(5).uniform(0.0, 2.0, P)
    k32 = k.astype(np.float32)
    want = O.Ref.apply_filter(rows.astype(np.float64), 1.0, k32.astype(np.float64), P)
    out = tg.graph._fourier_filter(_t(rows), _t(k32), n, P)
    assert_close(out.cpu().numpy(), want, rel_rmse=FILTER_REL_RMSE, rel_max=10 * FILTER_REL_RMSE,
                 what=f"fourier_filter n={n} P={P} sym={sym}")


@pytest.mark.parametrize("n,P,rows", [(64, 64, 60), (365, 1024, 360), (33, 128, 1)])
def test_fourier_filter_weight_grad(tg, n, P, rows):
    x = rand((rows, n), 1, -1.0, 1.0)
    g = rand((rows, n), 2, -1.0, 1.0)
    X = np.fft.fft(x.astype(np.float64), P, axis=1)
    G = np.fft.fft(g.astype(np.float64), P, axis=1)
    want = np.sum(X.real * G.real + X.imag * G.imag, axis=0) / P
    gk = torch.full((P,), 0.25, dtype=torch.float32, device=DEV)  # accumulates
    dx, dg = _t(x), _t(g)
    tg._native.check(tg._native.lib().tg_fourier_filter_weight_grad(
        dx.data_ptr(), dg.data_ptr(), gk.data_ptr(), rows, n, P,
        torch.cuda.current_stream().cuda_stream))
    assert_close(gk.cpu().numpy() - 0.25, want, rel_rmse=1e-5, rel_max=1e-4, what="gk")
    assert np.allclose(gk.cpu().numpy()[1:], gk.cpu().numpy()[1:][::-1], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("fan", [False, True])
def test_graph_probe_vs_reference(tg, fan):
    """loss = l2(multiply_weights(forward_project(x), w), p) + scale(tv(x), lam):
    value and gradients of x and w against the reference's Graph."""
    kw = dict(sid=300.0, sdd=600.0) if fan else {}
    geo, og = planar_pair(tg, O, [20, 17], [1.0, 1.0], 29, 1.0, 9, 2 * math.pi if fan else math.pi,
                          **kw)
    x0 = rand((17, 20), 7)
    w0 = 0.5 + rand(29, 8)
    sino = rand((9, 29), 9)
    lam = 0.7
    ref_loss, ref_gx, ref_gw = O.Ref.graph_probe(og, x0, w0, sino, lam)
    g = tg.Graph()
    x = g.parameter(_t(x0))
    w = g.parameter(_t(w0))
    p = g.input([29, 9])
    mw = g.multiply_weights(g.forward_project(x, geo), w)
    loss = g.add(g.l2_loss(mw, p), g.scale(g.tv_loss(x), lam))
    g.forward({p: _t(sino)})
    assert g.value(loss) == pytest.approx(ref_loss, rel=2e-6)
    grads = g.backward(loss)
    assert_close(grads[x].cpu().numpy(), ref_gx, 5e-5, 5e-4, "grad x")
    assert_close(grads[w].cpu().numpy(), ref_gw, 5e-5, 5e-4, "grad w")
    # a second backward re-zeroes the gradients (graph.hpp:226-227)
    again = g.backward(loss)
    assert torch.equal(again[x], grads[x]) and torch.equal(again[w], grads[w])


def test_graph_backproject_node_and_its_gradient(tg):
    geo, og = planar_pair(tg, O, [24, 24], [1.0, 1.0], 35, 1.0, 12, math.pi)
    s0 = rand((12, 35), 3)
    t0 = rand((24, 24), 4)
    g = tg.Graph()
    s = g.parameter(_t(s0))
    t = g.input([24, 24])
    bp = g.backproject(s, geo)
    loss = g.l2_loss(bp, t)
    g.forward({t: _t(t0)})
    bp_ref = O.planar_backproject(og, s0.astype(np.float64))
    assert_close(g.value(bp).cpu().numpy(), bp_ref, what="bp node")
    grads = g.backward(loss)
    want = O.planar_forward(og, 2.0 * (bp_ref - t0.astype(np.float64)))
    assert_close(grads[s].cpu().numpy(), want, 5e-5, 5e-4, "registered gradient (FP)")


def _learn_setup(tg):
    geo, og = planar_pair(tg, O, [45, 45], [1.0, 1.0], 64, 1.0, 60, math.pi)
    ph = tg.shepp_logan_2d(geo.volume, torch.device(DEV))
    sino = tg.forward_project(ph, geo)
    return geo, og, sino


@pytest.mark.parametrize("via_graph", [False, True])
def test_learn_filter_vs_reference_graph(tg, via_graph):
    """configs/learn_filter.json geometry and rate, 40 steps, noise-free; the
    device-resident loop and the node-by-node device graph"""
    geo, og, sino = _learn_setup(tg)
    cfg = tg.ExperimentConfig(learning_rate=1.5e-5, iterations=40, filter_window=64)
    r = tg.learn_filter(sino, geo, cfg, via_graph=via_graph)
    s64 = sino.data.cpu().numpy().astype(np.float64)
    l_ref, d_ref, w_ref, rec_ref = O.Ref.learn_filter_graph(og, s64, 64, 1.5e-5, 40)
    l_or, d_or, w_or, _ = O.learn_filter_planar(og, s64, 64, 1.5e-5, 40)
    assert np.array_equal(l_or, l_ref) and np.array_equal(w_or, w_ref)
    l32, d32, w32, _ = O.learn_filter_planar(og, sino.data.cpu().numpy(), 64, 1.5e-5, 40)
    drift_l = np.max(np.abs(l32 - l_ref) / l_ref)
    drift_w = np.max(np.abs(w32 - w_ref)) / np.max(np.abs(w_ref))
    dev_l = np.max(np.abs(np.array(r.loss_history) - l_ref) / l_ref)
    dev_w = np.max(np.abs(r.learned_weights - w_ref)) / np.max(np.abs(w_ref))
    assert dev_l <= max(2 * drift_l, 1e-5), (dev_l, drift_l)
    assert dev_w <= max(2 * drift_w, 1e-5), (dev_w, drift_w)
    assert len(r.loss_history) == 41 and r.loss_history[-1] < r.loss_history[0]
    assert r.distance_history[-1] < r.distance_history[0]
    assert_close(r.reconstruction.data.cpu().numpy(), rec_ref, 1e-4, 1e-3, "learned FBP")


def test_learn_filter_loop_matches_graph(tg):
    """the fused device loop and the node-by-node graph run the same maths"""
    geo, og, sino = _learn_setup(tg)
    cfg = tg.ExperimentConfig(learning_rate=1.5e-5, iterations=12, filter_window=64)
    a = tg.learn_filter(sino, geo, cfg)
    b = tg.learn_filter(sino, geo, cfg, via_graph=True)
    # the loss is |recon - target|^2 with recon close to target: fp32 rounding
    # differences of the two summation orders are amplified by the
    # cancellation (measured up to 8.5e-6 relative once the FBP target moved
    # to the packed two-rows-per-FFT filter)
    np.testing.assert_allclose(a.loss_history, b.loss_history, rtol=2e-5)
    np.testing.assert_allclose(a.learned_weights, b.learned_weights, rtol=1e-6,
                               atol=1e-7 * np.abs(b.learned_weights).max())
    # run-to-run determinism of the captured loop
    c = tg.learn_filter(sino, geo, cfg)
    assert a.loss_history == c.loss_history
    assert np.array_equal(a.learned_weights, c.learned_weights)


def test_experiment_learn_filter_end_to_end(tg):
    """the reference experiment itself (phantom, FP, noise 0.3, seed 1337):
    the device phantom / FP feed the bit-exact noise, so the histories match
    to the fp32 projector tolerance"""
    geo, og, _ = _learn_setup(tg)
    cfg = tg.ExperimentConfig(noise_relative_std=0.3, learning_rate=1.5e-5, iterations=20,
                              filter_window=64)
    r = tg.experiment_learn_filter(geo, cfg, device=torch.device(DEV))
    l_ref, d_ref, w_ref, _ = O.Ref.experiment_learn_filter(og, "shepp-logan", 0.3, 1337, 64,
                                                           1.5e-5, 20)
    np.testing.assert_allclose(r.loss_history, l_ref, rtol=3e-4)
    np.testing.assert_allclose(r.distance_history, d_ref, rtol=3e-4, atol=1e-6)


def test_autograd_operators_register_each_other(tg):
    geo, og = planar_pair(tg, O, [30, 26], [1.0, 1.0], 41, 1.0, 16, math.pi)
    x = _t(rand((26, 30), 1)).requires_grad_(True)
    p = _t(rand((16, 41), 2))
    y = tg.forward_project_op(x, geo)
    loss = ((y - p) ** 2).sum()
    loss.backward()
    want = tg.back_project(tg.Sinogram.planar(16, geo.detector, data=(2 * (y - p)).detach()),
                           geo).data
    assert torch.equal(x.grad, want)
    s = _t(rand((16, 41), 3)).requires_grad_(True)
    b = tg.back_project_op(s, geo)
    b.sum().backward()
    ones = torch.ones(26, 30, device=DEV)
    assert torch.equal(s.grad, tg.forward_project(tg.Image(geo.volume, ones), geo).data)


def test_autograd_fourier_filter_matches_graph(tg):
    P = 128
    x0 = rand((12, 64), 4, -1.0, 1.0)
    k0 = tg.ramp_weights(P, 1.0).astype(np.float32)
    t0 = rand((12, 64), 5, -1.0, 1.0)
    k = _t(k0).requires_grad_(True)
    x = _t(x0).requires_grad_(True)
    y = tg.fourier_filter_op(x, k, P)
    ((y - _t(t0)) ** 2).sum().backward()
    g = tg.Graph()
    xn = g.parameter(_t(x0))
    kn = g.parameter(_t(k0))
    tn = g.input([64, 12])
    loss = g.l2_loss(g.fourier_filter(xn, kn, P), tn)
    g.forward({tn: _t(t0)})
    grads = g.backward(loss)
    assert torch.allclose(k.grad, grads[kn], rtol=1e-5, atol=1e-6 * k.grad.abs().max().item())
    assert torch.allclose(x.grad, grads[xn], rtol=1e-5, atol=1e-6 * x.grad.abs().max().item())


def test_nan_gradient_is_reported(tg):
    g = tg.Graph()
    a = g.parameter(_t(np.array([1.0, float("nan"), 2.0])))
    b = g.input([3])
    loss = g.l2_loss(a, b)
    g.forward({b: _t(np.zeros(3))})
    with pytest.raises(tg.Error) as e:
        g.backward(loss)
    # the reverse sweep meets the input b (its gradient -2(a - b)) before a
    assert str(e.value) == f"gradient of node {b} contains NaN"


def test_inf_gradient_is_not_nan(tg):
    """graph.hpp:389-393 tests std::isnan only: an overflowing (+-inf) gradient
    passes the check, as in the reference"""
    g = tg.Graph()
    a = g.parameter(_t(np.array([1.0, float("inf"), 2.0])))
    b = g.input([3])
    loss = g.l2_loss(a, b)
    g.forward({b: _t(np.zeros(3))})
    grads = g.backward(loss)
    assert torch.isinf(grads[a]).any() and not torch.isnan(grads[a]).any()


def test_graph_requires_device_values(tg):
    g = tg.Graph()
    x = g.input([4])
    with pytest.raises(Exception):
        # a CPU-only torch tensor is moved to CUDA; a non-tensor is rejected
        g.forward({x: "not a tensor"})
