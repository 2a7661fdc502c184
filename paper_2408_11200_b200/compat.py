"""Literal drop-in into the reference's own operator API (second half).

The reference (``ukan``, float64 NumPy) records one tape node per op through
``ukan.tensor.make_node(values, parents, backward_fn)`` with ``backward_fn(upstream, acc)``
(tensor.py:94-101), and its layers dispatch through the module-level functions
``ukan.layers.kan_forward`` (layers.py:304-318) and ``ukan.layers.ukan_forward`` (254-291)
(``KanLayer.forward`` / ``UkanLayer.forward`` / ``Model.forward`` look them up at call time).

``install(ukan)`` replaces those two functions with versions that keep the reference's tensors,
checks and exceptions but compute the layer on the B200 kernels (``libukan_b200.so``): NumPy
values are copied to the device as fp32 at the boundary, the forward runs the fused kernel, and
the recorded node's ``backward_fn`` runs the fused backward and hands float64 gradients to the
reference's ``acc`` — for x only when x is a recorded node (tensor.py:455-456), exactly as the
reference's own ops do.  The reference's ``Model``, ``train``, ``run_bench`` and tests then run
unchanged on the kernels, at the fp32 parity bar (|d| <= 1e-6 + 1e-5 |ref|; grid indices
bit-exact).  There is no CPU fallback: without a CUDA device the patched functions raise.

Tangent inputs (``pinn_loss``'s forward-over-reverse, tensor.py:411-424) are not routed
through this adapter; the B200 tangent path is ``kan_forward_tangent`` / ``ukan_forward_tangent``.
"""
from __future__ import annotations

import numpy as np
import torch

from . import layers as _L

_saved: dict = {}


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2408_11200_b200.compat needs a CUDA (sm_100a) device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, requires_grad=False):
    t = torch.as_tensor(np.asarray(a, dtype=np.float32), device=_dev())
    return t.requires_grad_(requires_grad)


def _check_tangent(ukan, *tensors):
    if ukan.tensor.tangent_active(*tensors):
        raise ukan.errors.ContractError("tangent inputs are not supported by the B200 compat path "
                                        "(use paper_2408_11200_b200.kan_forward_tangent)")


def _node(ukan, y, parents, leaves):
    """Record the fused op on the reference tape.  ``leaves`` pairs each reference parent with the
    device tensor standing for it (None when the parent needs no gradient)."""
    values = y.detach().double().cpu().numpy()
    live = [(p, t) for p, t in leaves if t is not None]

    def backward_fn(upstream, acc):
        g = torch.as_tensor(np.asarray(upstream, dtype=np.float32), device=y.device)
        grads = torch.autograd.grad(y, [t for _, t in live], g, allow_unused=True)
        for (p, t), gr in zip(live, grads):
            acc(p, np.zeros(t.shape) if gr is None else gr.double().cpu().numpy())

    return ukan.tensor.make_node(values, parents, backward_fn)


def kan_forward(layer, x):
    """Drop-in for ``ukan.layers.kan_forward`` (layers.py:304-318) on the B200 kernels."""
    ukan = _saved["ukan"]
    x = ukan.tensor.as_tensor(x)
    if x.values.ndim != 2 or x.shape[1] != layer.d_in:
        raise ukan.errors.DimensionError(f"expected [batch, {layer.d_in}] input, got {x.shape}")
    _check_tangent(ukan, x, layer.coeffs, layer.scale, layer.base_weight)
    xt = _to_dev(x.values, x.node_id is not None)
    C = _to_dev(layer.coeffs.values, layer.coeffs.node_id is not None)
    S = _to_dev(layer.scale.values, layer.scale.node_id is not None)
    bw = None if layer.base_weight is None else _to_dev(layer.base_weight.values,
                                                        layer.base_weight.node_id is not None)
    dl = _L.KanLayer(layer.d_in, layer.d_out, layer.k, float(layer.g_min), float(layer.g_max), int(layer.G), C, S, bw)
    with torch.enable_grad():
        y = _L.kan_forward(dl, xt)
    parents = [x, layer.coeffs, layer.scale] + ([layer.base_weight] if layer.base_weight is not None else [])
    leaves = [(x, xt if xt.requires_grad else None), (layer.coeffs, C if C.requires_grad else None),
              (layer.scale, S if S.requires_grad else None)]
    if bw is not None:
        leaves.append((layer.base_weight, bw if bw.requires_grad else None))
    return _node(ukan, y, parents, leaves)


_UKAN_PARAMS = ("feature_embedding", "cg_w1", "cg_b1", "cg_w2", "cg_b2", "scale")


def ukan_forward(layer, x, dedup: bool = True):
    """Drop-in for ``ukan.layers.ukan_forward`` (layers.py:254-291) on the B200 kernels.  The
    kernels always deduplicate the keys; the reference's ``dedup=False`` gives bitwise the same
    values (test_layers.py:147-152), so the flag is accepted and has no effect."""
    ukan = _saved["ukan"]
    x = ukan.tensor.as_tensor(x)
    if x.values.ndim != 2 or x.shape[1] != layer.d_in:
        raise ukan.errors.DimensionError(f"expected [batch, {layer.d_in}] input, got {x.shape}")
    if not np.isfinite(x.values).all():
        raise ukan.errors.DomainError("non-finite input")
    refs = [getattr(layer, n) for n in _UKAN_PARAMS]
    _check_tangent(ukan, x, *refs)
    xt = _to_dev(x.values, x.node_id is not None)
    dev_p = {n: _to_dev(r.values, r.node_id is not None) for n, r in zip(_UKAN_PARAMS, refs)}
    dl = _L.UkanLayer(layer.d_in, layer.d_out, layer.k, float(layer.delta_g), int(layer.d_pe), int(layer.d_femb),
                      **dev_p)
    with torch.enable_grad():
        y = _L.ukan_forward(dl, xt)
    leaves = [(x, xt if xt.requires_grad else None)]
    leaves += [(r, dev_p[n] if dev_p[n].requires_grad else None) for n, r in zip(_UKAN_PARAMS, refs)]
    return _node(ukan, y, [x] + refs, leaves)


def install(ukan_module) -> None:
    """Route the reference's layer ops through the B200 kernels (idempotent)."""
    import importlib
    layers = importlib.import_module(ukan_module.__name__ + ".layers")
    if "ukan" not in _saved:
        _saved.update(ukan=ukan_module, kan_forward=layers.kan_forward, ukan_forward=layers.ukan_forward)
    layers.kan_forward = kan_forward
    layers.ukan_forward = ukan_forward
    ukan_module.kan_forward = kan_forward
    ukan_module.ukan_forward = ukan_forward


def uninstall() -> None:
    """Restore the reference's own functions."""
    if "ukan" not in _saved:
        return
    import importlib
    ukan = _saved["ukan"]
    layers = importlib.import_module(ukan.__name__ + ".layers")
    layers.kan_forward = ukan.kan_forward = _saved["kan_forward"]
    layers.ukan_forward = ukan.ukan_forward = _saved["ukan_forward"]
    _saved.clear()
