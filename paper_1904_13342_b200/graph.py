"""The reference's reverse-mode computation graph (graph.hpp) on the device
path, plus the same operators as ``torch.autograd`` functions.

``Graph`` mirrors graph.hpp node for node — builders with the reference's
shape checks and messages (graph.hpp:104-190), ``forward(feeds)``
(graph.hpp:194-216), ``backward(loss)`` over the loss's ancestors in reverse
order (graph.hpp:219-246), ``gradient_descent_step`` (graph.hpp:533-546) — but
node values and gradients are fp32 CUDA tensors and every node runs a kernel
of libtomograd_b200.so:

    forward_project / backproject   K2/K5/K7 and K1/K4/K6 (each other's gradient,
                                    graph.hpp:408-434; the back-projection
                                    gradient accumulates in its epilogue)
    fourier_filter                  K3 with device weights + the packed-FFT
                                    weight-gradient kernel (graph.hpp:470-497)
    l2_loss, tv_loss                K8, K9 (value) and their gradient kernels
    multiply_weights, add, scale    graph.cu elementwise kernels

Shapes are listed fastest axis first, like the reference (a [ny][nx] image is
shape [nx, ny]); tensors carry the usual row-major torch shape (the reverse).
Scalar node values (losses) are Python floats, as the reference's
``scalar_value()``.  There is no CPU path: values must live on a CUDA device.

``ForwardProject`` / ``BackProject`` / ``FourierFilter`` (and the functional
``forward_project_op`` / ``back_project_op`` / ``fourier_filter_op``) expose
the same registered gradients to torch.autograd, so the projectors work as
layers of a PyTorch network — the known-operator use the reference's graph
exists for.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import torch

from . import _native as N
from .containers import Image, Sinogram, stream_of
from .geometry import ConeGeometry, FanGeometry, ParallelGeometry, check
from .projector import _dev, back_project, forward_project


class OpKind(enum.Enum):
    """graph.hpp:31-42"""
    input = 0
    parameter = 1
    forward_project = 2
    backproject = 3
    multiply_weights = 4
    fourier_filter = 5
    add = 6
    scale = 7
    l2_loss = 8
    tv_loss = 9


NodeId = int


def sino_shape(geo) -> List[int]:
    """graph.hpp:72-79 (fastest axis first)"""
    if isinstance(geo, ConeGeometry):
        return [geo.detector.n_u, geo.detector.n_v, geo.n_projections]
    return [geo.detector.n_bins, geo.n_projections]


def volume_shape(geo) -> List[int]:
    """graph.hpp:81-85"""
    return list(geo.volume.shape)


@dataclass
class Node:
    """graph.hpp:89-100"""
    kind: OpKind
    inputs: List[NodeId] = field(default_factory=list)
    shape: List[int] = field(default_factory=list)  # fastest first; [] = scalar
    trainable: bool = False
    factor: float = 1.0
    padded_n: int = 0
    geometry: object = None
    value: object = None  # torch.Tensor (fp32, CUDA) or float for scalars
    grad: object = None
    has_value: bool = False


def _torch_shape(shape: List[int]):
    return tuple(reversed([int(s) for s in shape]))


def _to_device(t, device) -> torch.Tensor:
    if isinstance(t, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32))
    check(isinstance(t, torch.Tensor), "graph values must be tensors or numpy arrays")
    if device is None:
        device = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
    return t.detach().to(device=device, dtype=torch.float32).contiguous()


def _axpby(a: torch.Tensor, b: Optional[torch.Tensor], out: torch.Tensor, alpha: float,
           beta: float) -> None:
    N.check(N.lib().tg_axpby(a.data_ptr(), b.data_ptr() if b is not None else None,
                             out.data_ptr(), out.numel(), float(alpha), float(beta),
                             stream_of(out)))


def _l2_value(a: torch.Tensor, b: torch.Tensor) -> float:
    s = torch.empty(1, dtype=torch.float64, device=a.device)
    N.check(N.lib().tg_l2_residual(a.data_ptr(), b.data_ptr(), None, a.numel(), s.data_ptr(),
                                   stream_of(a)))
    return float(s.item())


def _tv_dims(shape: List[int]):
    check(1 <= len(shape) <= 3, "tv_loss on the device supports 1 to 3 axes")
    d = [int(s) for s in shape] + [1] * (3 - len(shape))
    return d[0], d[1], d[2]


def _tv_value(x: torch.Tensor, shape: List[int]) -> float:
    nx, ny, nz = _tv_dims(shape)
    v = torch.empty(1, dtype=torch.float64, device=x.device)
    N.check(N.lib().tg_tv_step(x.data_ptr(), None, None, nx, ny, nz, 0, 0, 0.0, 0.0,
                               v.data_ptr(), stream_of(x)))
    return float(v.item())


def _fourier_filter(x: torch.Tensor, k: torch.Tensor, n: int, P: int,
                    out: torch.Tensor = None) -> torch.Tensor:
    out = torch.empty_like(x) if out is None else out
    N.check(N.lib().tg_fourier_filter(x.data_ptr(), k.data_ptr(), out.data_ptr(), x.numel() // n,
                                      n, P, stream_of(x)))
    return out


def _fp(x: torch.Tensor, geo) -> torch.Tensor:
    return forward_project(Image(geo.volume, x), geo).data


def _sino(data: torch.Tensor, geo) -> Sinogram:
    if isinstance(geo, ConeGeometry):
        return Sinogram.cone_beam(geo.n_projections, geo.detector, data=data)
    return Sinogram.planar(geo.n_projections, geo.detector, data=data)


def _bp(s: torch.Tensor, geo) -> torch.Tensor:
    return back_project(_sino(s, geo), geo).data


def _bp_accumulate(s: torch.Tensor, geo, into: torch.Tensor) -> None:
    """into += BP(s): the back-projection epilogue accumulates (no temporary)"""
    L = N.lib()
    if isinstance(geo, ConeGeometry):
        N.check(L.tg_cone_backproject(geo._plan(_dev(s)), s.data_ptr(), into.data_ptr(), 1.0, 1,
                                      stream_of(s)))
    else:
        N.check(L.tg_planar_backproject(geo._plan(_dev(s)), s.data_ptr(), into.data_ptr(), 1.0,
                                        1, stream_of(s)))


def _is_geometry(geo) -> bool:
    return isinstance(geo, (ParallelGeometry, FanGeometry, ConeGeometry))


class Graph:
    """graph.hpp:102-531 over device fp32 tensors."""

    def __init__(self, device=None):
        self._nodes: List[Node] = []
        self._nan_slots = None
        self.device = torch.device(device) if device is not None else None

    # --- builders (graph.hpp:104-190) ----------------------------------------

    def input(self, shape) -> NodeId:
        return self._push(Node(OpKind.input, [], [int(s) for s in shape]))

    def parameter(self, init, trainable: bool = True, shape=None) -> NodeId:
        """``init``: a tensor / array in torch layout (its reversed shape is the
        node's shape), or a float for a scalar; ``shape`` (fastest first)
        reinterprets a flat init like the reference's Tensor(shape, data)."""
        if isinstance(init, (int, float)):
            n = Node(OpKind.parameter, [], [], trainable, value=float(init), has_value=True)
            return self._push(n)
        t = _to_device(init, self.device)
        if shape is not None:
            t = t.reshape(_torch_shape(shape))
        if self.device is None:
            self.device = t.device
        n = Node(OpKind.parameter, [], list(reversed(t.shape)), trainable, value=t,
                 has_value=True)
        return self._push(n)

    def forward_project(self, x: NodeId, geo) -> NodeId:
        check(_is_geometry(geo), "projection node lost its geometry")
        n = Node(OpKind.forward_project, [self._valid(x)], sino_shape(geo), geometry=geo)
        check(self.node(x).shape == volume_shape(geo),
              "forward_project input shape does not match the geometry volume")
        return self._push(n)

    def backproject(self, x: NodeId, geo) -> NodeId:
        check(_is_geometry(geo), "projection node lost its geometry")
        n = Node(OpKind.backproject, [self._valid(x)], volume_shape(geo), geometry=geo)
        check(self.node(x).shape == sino_shape(geo),
              "backproject input shape does not match the geometry sinogram")
        return self._push(n)

    def multiply_weights(self, x: NodeId, w: NodeId) -> NodeId:
        xs = self.node(self._valid(x)).shape
        ws = self.node(self._valid(w)).shape
        full = ws == xs
        prefix = len(ws) < len(xs) and xs[: len(ws)] == ws
        check(full or prefix, "weight shape must equal the input shape or a prefix of it")
        return self._push(Node(OpKind.multiply_weights, [x, w], list(xs)))

    def fourier_filter(self, x: NodeId, k: NodeId, padded_n: int) -> NodeId:
        xs = self.node(self._valid(x)).shape
        ks = self.node(self._valid(k)).shape
        P = int(padded_n)
        check(len(xs) > 0, "fourier_filter input must have at least one axis")
        check(P > 0 and (P & (P - 1)) == 0, "filter window must be a power of two")
        check(P >= xs[0], "filter window is smaller than the detector row")
        check(len(ks) == 1 and ks[0] == P, "filter weight vector must have length padded_n")
        return self._push(Node(OpKind.fourier_filter, [x, k], list(xs), padded_n=P))

    def add(self, a: NodeId, b: NodeId) -> NodeId:
        check(self.node(self._valid(a)).shape == self.node(self._valid(b)).shape,
              "add expects matching shapes")
        return self._push(Node(OpKind.add, [a, b], list(self.node(a).shape)))

    def scale(self, x: NodeId, factor: float) -> NodeId:
        return self._push(Node(OpKind.scale, [self._valid(x)], list(self.node(x).shape),
                               factor=float(factor)))

    def l2_loss(self, a: NodeId, b: NodeId) -> NodeId:
        check(self.node(self._valid(a)).shape == self.node(self._valid(b)).shape,
              "l2_loss expects matching shapes")
        return self._push(Node(OpKind.l2_loss, [a, b], []))

    def tv_loss(self, x: NodeId) -> NodeId:
        check(len(self.node(self._valid(x)).shape) > 0, "tv_loss needs a non-scalar input")
        return self._push(Node(OpKind.tv_loss, [x], []))

    # --- execution (graph.hpp:194-246) -----------------------------------------

    def forward(self, feeds: Dict[NodeId, object]) -> None:
        for nid, t in feeds.items():
            check(0 <= nid < len(self._nodes) and self._nodes[nid].kind == OpKind.input,
                  "feed id does not name an input node")
            shape = [] if isinstance(t, (int, float)) else list(reversed(t.shape))
            check(shape == self._nodes[nid].shape, "feed shape mismatch")
        for nid, n in enumerate(self._nodes):
            if n.kind == OpKind.input:
                check(nid in feeds, "missing feed for input node")
                t = feeds[nid]
                n.value = float(t) if isinstance(t, (int, float)) else _to_device(t, self.device)
                if self.device is None and isinstance(n.value, torch.Tensor):
                    self.device = n.value.device
            elif n.kind != OpKind.parameter:
                n.value = self._evaluate(n)
            n.has_value = True

    def backward(self, loss: NodeId) -> Dict[NodeId, object]:
        self._valid(loss)
        check(self._nodes[loss].has_value, "run forward before backward")
        check(not isinstance(self._nodes[loss].value, torch.Tensor), "loss node must be scalar")
        for n in self._nodes:
            if isinstance(n.value, torch.Tensor):
                if isinstance(n.grad, torch.Tensor) and n.grad.shape == n.value.shape:
                    n.grad.zero_()
                else:
                    n.grad = torch.zeros_like(n.value)
            else:
                n.grad = 0.0
        self._nodes[loss].grad = 1.0
        active = [False] * len(self._nodes)
        stack = [loss]
        active[loss] = True
        while stack:
            nid = stack.pop()
            for i in self._nodes[nid].inputs:
                if not active[i]:
                    active[i] = True
                    stack.append(i)
        # graph.hpp:402-406 NaN checks: one device reduction per tensor
        # gradient into its own slot, read back once after the sweep (the
        # first offending node in sweep order is reported, as the reference)
        tensors = [i for i in range(loss + 1)
                   if active[i] and isinstance(self._nodes[i].grad, torch.Tensor)]
        if tensors:
            self._nan_slots = torch.zeros(len(self._nodes), dtype=torch.int64,
                                          device=self._nodes[tensors[0]].grad.device)
        try:
            for nid in range(loss, -1, -1):
                if active[nid]:
                    self._propagate(nid)
        finally:
            slots = self._nan_slots.cpu().numpy() if tensors else None
            self._nan_slots = None
        # the reference raises at the first NaN of its sweep (highest id first)
        for nid in sorted(tensors, reverse=True):
            if slots[nid] > 0:
                raise N.Error(f"gradient of node {nid} contains NaN")
        return {nid: n.grad for nid, n in enumerate(self._nodes) if n.kind == OpKind.parameter}

    def value(self, nid: NodeId):
        check(self._nodes[self._valid(nid)].has_value, "node has no value; run forward first")
        return self._nodes[nid].value

    def grad(self, nid: NodeId):
        return self._nodes[self._valid(nid)].grad

    def node(self, nid: NodeId) -> Node:
        return self._nodes[self._valid(nid)]

    def size(self) -> int:
        return len(self._nodes)

    def trainable_parameters(self) -> List[NodeId]:
        return [i for i, n in enumerate(self._nodes)
                if n.kind == OpKind.parameter and n.trainable]

    # --- internals ----------------------------------------------------------

    def _valid(self, nid: NodeId) -> NodeId:
        check(isinstance(nid, int) and 0 <= nid < len(self._nodes), "node id out of range")
        return nid

    def _push(self, n: Node) -> NodeId:
        self._nodes.append(n)
        return len(self._nodes) - 1

    def _in(self, n: Node, i: int):
        src = self._nodes[n.inputs[i]]
        check(src.has_value, "node evaluated before its input")
        return src.value

    def _evaluate(self, n: Node):
        k = n.kind
        if k == OpKind.forward_project:
            return _fp(self._in(n, 0), n.geometry)
        if k == OpKind.backproject:
            return _bp(self._in(n, 0), n.geometry)
        if k == OpKind.multiply_weights:
            x, w = self._in(n, 0), self._in(n, 1)
            if not isinstance(x, torch.Tensor):
                return x * w
            out = torch.empty_like(x)
            N.check(N.lib().tg_multiply_weights(x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                                x.numel(), w.numel(), stream_of(x)))
            return out
        if k == OpKind.fourier_filter:
            x, kk = self._in(n, 0), self._in(n, 1)
            return _fourier_filter(x, kk, n.shape[0], n.padded_n)
        if k == OpKind.add:
            a, b = self._in(n, 0), self._in(n, 1)
            if not isinstance(a, torch.Tensor):
                return a + b
            out = torch.empty_like(a)
            _axpby(a, b, out, 1.0, 1.0)
            return out
        if k == OpKind.scale:
            x = self._in(n, 0)
            if not isinstance(x, torch.Tensor):
                return x * n.factor
            out = torch.empty_like(x)
            _axpby(x, None, out, n.factor, 0.0)
            return out
        if k == OpKind.l2_loss:
            a, b = self._in(n, 0), self._in(n, 1)
            if not isinstance(a, torch.Tensor):
                return (a - b) * (a - b)
            return _l2_value(a, b)
        if k == OpKind.tv_loss:
            return _tv_value(self._in(n, 0), self._nodes[n.inputs[0]].shape)
        raise N.Error("node kind cannot be evaluated")

    def _check_grad_finite(self, nid: NodeId) -> None:
        """graph.hpp:389-393,402: tensor gradients count their NaN entries
        (std::isnan: +-inf passes) on the device into this node's slot, read
        back once per backward; a NaN scalar raises at once, unless a tensor
        node swept before it (higher id) already holds a NaN — the reference
        would have stopped there first."""
        g = self._nodes[nid].grad
        if not isinstance(g, torch.Tensor):
            if math.isnan(g):
                if self._nan_slots is not None:
                    slots = self._nan_slots.cpu().numpy()
                    earlier = [i for i in range(len(slots) - 1, nid, -1) if slots[i] > 0]
                    if earlier:
                        nid = earlier[0]
                raise N.Error(f"gradient of node {nid} contains NaN")
            return
        slot = self._nan_slots.data_ptr() + 8 * nid
        N.check(N.lib().tg_nan_count(g.data_ptr(), g.numel(), slot, stream_of(g)))

    def _add_grad(self, nid: NodeId, contrib, factor: float = 1.0) -> None:
        dst = self._nodes[nid]
        if isinstance(dst.grad, torch.Tensor):
            _axpby(dst.grad, contrib, dst.grad, 1.0, factor)
        else:
            dst.grad += factor * contrib

    def _propagate(self, nid: NodeId) -> None:
        n = self._nodes[nid]
        self._check_grad_finite(nid)
        g = n.grad
        k = n.kind
        if k in (OpKind.input, OpKind.parameter):
            return
        if k == OpKind.forward_project:
            _bp_accumulate(g, n.geometry, self._nodes[n.inputs[0]].grad)
        elif k == OpKind.backproject:
            self._add_grad(n.inputs[0], _fp(g, n.geometry))
        elif k == OpKind.multiply_weights:
            xn, wn = self._nodes[n.inputs[0]], self._nodes[n.inputs[1]]
            if not isinstance(g, torch.Tensor):
                xn.grad += g * wn.value
                wn.grad += g * xn.value
                return
            N.check(N.lib().tg_multiply_weights_grad(
                g.data_ptr(), xn.value.data_ptr(), wn.value.data_ptr(), xn.grad.data_ptr(),
                wn.grad.data_ptr(), g.numel(), wn.value.numel(), stream_of(g)))
        elif k == OpKind.fourier_filter:
            xn, kn = self._nodes[n.inputs[0]], self._nodes[n.inputs[1]]
            # the real filter matrix is symmetric: the input gradient is the same filter
            self._add_grad(n.inputs[0], _fourier_filter(g, kn.value, n.shape[0], n.padded_n))
            N.check(N.lib().tg_fourier_filter_weight_grad(
                xn.value.data_ptr(), g.data_ptr(), kn.grad.data_ptr(), g.numel() // n.shape[0],
                n.shape[0], n.padded_n, stream_of(g)))
        elif k == OpKind.add:
            self._add_grad(n.inputs[0], g)
            self._add_grad(n.inputs[1], g)
        elif k == OpKind.scale:
            self._add_grad(n.inputs[0], g, n.factor)
        elif k == OpKind.l2_loss:
            an, bn = self._nodes[n.inputs[0]], self._nodes[n.inputs[1]]
            if not isinstance(an.value, torch.Tensor):
                d = 2.0 * g * (an.value - bn.value)
                an.grad += d
                bn.grad -= d
                return
            N.check(N.lib().tg_l2_grad(an.value.data_ptr(), bn.value.data_ptr(),
                                       an.grad.data_ptr(), bn.grad.data_ptr(), an.value.numel(),
                                       float(g), stream_of(an.value)))
        elif k == OpKind.tv_loss:
            xn = self._nodes[n.inputs[0]]
            nx, ny, nz = _tv_dims(xn.shape)
            v = torch.empty(1, dtype=torch.float64, device=xn.value.device)
            N.check(N.lib().tg_tv_grad(xn.value.data_ptr(), xn.grad.data_ptr(), nx, ny, nz,
                                       float(g), v.data_ptr(), stream_of(xn.value)))


def gradient_descent_step(g: Graph, grads: Dict[NodeId, object], learning_rate: float) -> None:
    """graph.hpp:533-546: value -= lr * grad on the trainable parameters"""
    for nid in g.trainable_parameters():
        if nid not in grads:
            continue
        node = g.node(nid)
        grad = grads[nid]
        if not isinstance(node.value, torch.Tensor):
            node.value -= learning_rate * grad
            continue
        check(grad.numel() == node.value.numel(), "gradient shape mismatch")
        _axpby(node.value, grad, node.value, 1.0, -float(learning_rate))


# ---- torch.autograd: the same operators and registered gradients ----------


class ForwardProject(torch.autograd.Function):
    """y = A x (K2/K5/K7); dL/dx = BP(dL/dy) (graph.hpp:408-419)"""

    @staticmethod
    def forward(ctx, x, geo):
        ctx.geo = geo
        return _fp(x.detach().contiguous(), geo)

    @staticmethod
    def backward(ctx, g):
        return _bp(g.contiguous(), ctx.geo), None


class BackProject(torch.autograd.Function):
    """x = B p (K1/K4/K6); dL/dp = FP(dL/dx) (graph.hpp:420-432)"""

    @staticmethod
    def forward(ctx, s, geo):
        ctx.geo = geo
        return _bp(s.detach().contiguous(), geo)

    @staticmethod
    def backward(ctx, g):
        return _fp(g.contiguous(), ctx.geo), None


class FourierFilter(torch.autograd.Function):
    """rows of x filtered by the P frequency weights k (K3); gradients
    graph.hpp:470-497"""

    @staticmethod
    def forward(ctx, x, k, padded_n):
        x = x.detach().contiguous()
        k = k.detach().to(torch.float32).contiguous()
        ctx.save_for_backward(x, k)
        ctx.P = int(padded_n)
        return _fourier_filter(x, k, x.shape[-1], ctx.P)

    @staticmethod
    def backward(ctx, g):
        x, k = ctx.saved_tensors
        g = g.contiguous()
        n = x.shape[-1]
        gx = _fourier_filter(g, k, n, ctx.P) if ctx.needs_input_grad[0] else None
        gk = None
        if ctx.needs_input_grad[1]:
            gk = torch.zeros_like(k)
            N.check(N.lib().tg_fourier_filter_weight_grad(x.data_ptr(), g.data_ptr(),
                                                          gk.data_ptr(), x.numel() // n, n,
                                                          ctx.P, stream_of(g)))
        return gx, gk, None


def forward_project_op(x: torch.Tensor, geo) -> torch.Tensor:
    return ForwardProject.apply(x, geo)


def back_project_op(s: torch.Tensor, geo) -> torch.Tensor:
    return BackProject.apply(s, geo)


def fourier_filter_op(x: torch.Tensor, k: torch.Tensor, padded_n: int) -> torch.Tensor:
    return FourierFilter.apply(x, k, padded_n)
