"""Generate golden vectors for the spline hot path by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):
    python tests/golden/make_golden.py
It imports ``ukan`` from /root/reference/pkg/src (read-only), builds layers with the
reference's own ``init_layer`` / ``build_model``, rounds every parameter and input to fp32
(so the float64 reference and the fp32 GPU path see identical values), runs the reference
forward + tape backward (x wrapped in ``T.parameter`` so dx is produced, loss
``sum(y * g_up)``), and stores inputs and outputs as ``.npz`` fixtures next to this script.
The fixtures are committed; nothing at test time reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def run_kan(name, d_in, d_out, k, G, g_min, g_max, B, seed, xgen, base=False):
    from ukan import tensor as T
    from ukan.layers import init_layer, kan_forward
    layer = init_layer("kan", d_in, d_out, k, seed=seed, g_min=g_min, g_max=g_max, G=G, base=base)
    for p in layer.parameters().values():
        p.values[...] = f32(p.values)
    rng = np.random.default_rng(seed + 1)
    x = f32(xgen(rng, (B, d_in)))
    gup = f32(np.random.default_rng(seed + 2).normal(size=(B, d_out)))
    xt = T.parameter(x.copy())
    y = kan_forward(layer, xt)
    T.backward(T.sum_all(T.mul(y, T.as_tensor(gup))))
    dg = (g_max - g_min) / G
    xc = np.clip(x, g_min, np.nextafter(g_max, g_min))
    cell = np.clip(np.floor((xc - g_min) / dg), 0, G - 1).astype(np.int64)   # layers.py:299
    out = dict(kind="kan", d_in=d_in, d_out=d_out, k=k, G=G, g_min=g_min, g_max=g_max,
               x=x, g_up=gup, coeffs=layer.coeffs.values, scale=layer.scale.values,
               y=y.values, dx=xt.grad, dcoeffs=layer.coeffs.grad, dscale=layer.scale.grad, cell=cell)
    if base:
        out.update(base_weight=layer.base_weight.values, dbase_weight=layer.base_weight.grad)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k_: np.shape(v) for k_, v in out.items() if isinstance(v, np.ndarray)})


def run_ukan(name, d_in, d_out, k, delta_g, d_pe, d_femb, B, seed, xgen, d_hidden=None):
    from ukan import tensor as T
    from ukan.layers import init_layer, ukan_forward
    layer = init_layer("ukan", d_in, d_out, k, seed=seed, delta_g=delta_g, d_pe=d_pe, d_femb=d_femb,
                       d_hidden=d_hidden)
    for p in layer.parameters().values():
        p.values[...] = f32(p.values)
    rng = np.random.default_rng(seed + 1)
    x = f32(xgen(rng, (B, d_in)))
    gup = f32(np.random.default_rng(seed + 2).normal(size=(B, d_out)))
    xt = T.parameter(x.copy())
    y = ukan_forward(layer, xt)
    T.backward(T.sum_all(T.mul(y, T.as_tensor(gup))))
    g_id = np.floor(x * (1.0 / delta_g)).astype(np.int64)                      # layers.py:263
    K = k + 1
    group = g_id // K
    feat = np.broadcast_to(np.arange(d_in)[None, :], (B, d_in))
    keys = np.unique(np.concatenate([(group * d_in + feat).ravel(), ((group + 1) * d_in + feat).ravel()]))
    out = dict(kind="ukan", d_in=d_in, d_out=d_out, k=k, delta_g=delta_g, d_pe=d_pe, d_femb=d_femb,
               x=x, g_up=gup, y=y.values, dx=xt.grad, g_id=g_id, keys=keys)
    for n, p in layer.parameters().items():
        out[n] = p.values
        out["d" + n] = p.grad
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k_: np.shape(v) for k_, v in out.items() if isinstance(v, np.ndarray)})


def run_step(name, kind, widths, k, B, seed, loss_kind, layer_kw, lr=1e-2, wd=1e-5, steps=2):
    """Two full training steps of the reference harness semantics (train.py:142-150):
    loss -> T.backward -> adam_step (coupled L2)."""
    from ukan import tensor as T
    from ukan.layers import build_model
    from ukan.optim import AdamState, adam_step
    model = build_model(kind, widths, k, seed=seed, **layer_kw)
    params = list(model.parameters().values())
    for p in params:
        p.values[...] = f32(p.values)
    rng = np.random.default_rng(seed + 1)
    if kind == "kan":
        x = f32(rng.uniform(-1, 1, (B, widths[0])))
    else:
        x = f32(rng.normal(0, 3, (B, widths[0])))
    if loss_kind == "softmax_cross_entropy":
        target = np.random.default_rng(seed + 2).integers(0, widths[-1], B)
    else:
        target = f32(np.random.default_rng(seed + 2).normal(size=(B, widths[-1])))
    out = dict(kind=kind, widths=np.array(widths), k=k, x=x, target=target, loss_kind=loss_kind,
               lr=lr, wd=wd, steps=steps, **{f"kw_{a}": b for a, b in layer_kw.items()})
    names = list(model.parameters().keys())
    for n, p in zip(names, params):
        out["init." + n] = p.values.copy()
    state = AdamState()
    losses = []
    for s in range(steps):
        loss = T.reduce_loss(loss_kind, model(T.as_tensor(x)), target)
        losses.append(float(loss.values))
        T.backward(loss)
        grads = [p.grad for p in params]
        if s == 0:
            for n, g in zip(names, grads):
                out["grad0." + n] = g.copy()
        adam_step(params, grads, state, lr, weight_decay=wd)
    for n, p in zip(names, params):
        out["final." + n] = p.values.copy()
    out["losses"] = np.array(losses)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "losses", losses)


def run_tangent(name, kind, widths, k, B, seed, layer_kw, xgen):
    """Forward tangent through a spline stack (F2): x seeded with tx (tensor.py:411-424),
    L = sum(y * gup) + sum(y.tangent * gt), reference tape backward."""
    from ukan import tensor as T
    from ukan.layers import build_model
    model = build_model(kind, widths, k, seed=seed, **layer_kw)
    for p in model.parameters().values():
        p.values[...] = f32(p.values)
    rng = np.random.default_rng(seed + 1)
    x = f32(xgen(rng, (B, widths[0])))
    tx = f32(rng.normal(size=(B, widths[0])))
    r2 = np.random.default_rng(seed + 2)
    gup = f32(r2.normal(size=(B, widths[-1])))
    gt = f32(r2.normal(size=(B, widths[-1])))
    xp = T.parameter(x.copy())
    y = model(T.seed_tangent(xp, tx))
    ty = y.tangent
    T.backward(T.add(T.sum_all(T.mul(y, T.as_tensor(gup))), T.sum_all(T.mul(ty, T.as_tensor(gt)))))
    out = dict(kind=kind, widths=np.array(widths), k=k, x=x, tx=tx, g_up=gup, g_tan=gt, y=y.values,
               ty=ty.values, dx=xp.grad, **{f"kw_{a}": b for a, b in layer_kw.items()})
    for n, p in model.parameters().items():
        out[n] = p.values
        out["d" + n] = p.grad
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "ty", ty.values.shape)


def run_pinn(name, kind, k, seed, layer_kw, n_colloc=16):
    """pinn_loss (tasks.py:153-166) of a [1, 5, 1] stack and its parameter gradients."""
    from ukan import tensor as T
    from ukan.layers import build_model
    from ukan.tasks import PinnProblem, pinn_loss
    model = build_model(kind, [1, 5, 1], k, seed=seed, **layer_kw)
    for p in model.parameters().values():
        p.values[...] = f32(p.values)
    problem = PinnProblem(1.0, -5.0, 5.0, n_colloc)
    colloc = f32(problem.sample_collocation(np.random.default_rng(seed + 1)))
    loss = pinn_loss(model.forward, problem, colloc)
    T.backward(loss)
    out = dict(kind=kind, k=k, colloc=colloc, loss=float(loss.values), **{f"kw_{a}": b for a, b in layer_kw.items()})
    for n, p in model.parameters().items():
        out[n] = p.values
        out["d" + n] = p.grad
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "loss", float(loss.values))


def main():
    sys.path.insert(0, REF)
    import ukan
    assert ukan.__file__.startswith(REF), ukan.__file__

    unif = lambda lo, hi: (lambda r, s: r.uniform(lo, hi, s))

    def edges(r, s):
        x = r.uniform(-1.5, 1.5, s)
        flat = x.ravel()
        special = [np.inf, -np.inf, 1.0, -1.0, np.nextafter(1.0, 0.0), 0.0, 0.5, -0.5, 1e30, -1e30,
                   0.2, -0.6, 0.6000000238418579, 2.0 / 3.0]
        flat[:len(special)] = special
        return x

    run_kan("kan_small", 3, 4, 3, 5, -1.0, 1.0, 16, 11, unif(-1.3, 1.3))
    run_kan("kan_cfg1", 64, 64, 3, 10, -1.0, 1.0, 128, 0, unif(-1, 1))
    run_kan("kan_edges", 2, 3, 3, 8, -1.0, 1.0, 16, 5, edges)
    run_kan("kan_base", 4, 3, 3, 6, -2.0, 2.0, 24, 7, unif(-2.5, 2.5), base=True)
    for kk, G in ((0, 4), (1, 7), (2, 3), (5, 9), (10, 12)):
        run_kan(f"kan_k{kk}", 3, 5, kk, G, -2.0, 1.5, 20, 100 + kk, unif(-2.2, 1.7))
    run_kan("kan_odd", 5, 7, 3, 13, -0.7, 2.9, 33, 21, unif(-1.0, 3.2))

    def heavy(r, s):
        x = r.normal(0, 20.0, s)
        m = r.random(s) < 0.05
        x[m] = np.sign(r.normal(size=m.sum())) * 10 ** r.uniform(2, 5, m.sum())
        return x

    def knots(r, s):  # exact fp32 knot multiples of delta_g (SURVEY gotcha 1/2)
        m = r.integers(-2000, 2000, s)
        return (m * np.float32(0.3)).astype(np.float32)

    run_ukan("ukan_small", 3, 2, 3, 0.8, 8, 8, 32, 31, lambda r, s: r.normal(0, 5, s))
    run_ukan("ukan_heavy", 4, 3, 3, 0.5, 8, 8, 40, 32, heavy)
    run_ukan("ukan_k2", 3, 4, 2, 1.3, 6, 4, 24, 33, lambda r, s: r.uniform(-9, 9, s))
    run_ukan("ukan_knots", 2, 2, 3, 0.3, 8, 8, 64, 34, knots)
    run_ukan("ukan_hidden", 5, 3, 1, 0.4, 4, 6, 30, 35, lambda r, s: r.normal(0, 2, s), d_hidden=7)

    run_step("step_kan_ce", "kan", [6, 7, 3], 3, 48, 41, "softmax_cross_entropy",
             dict(g_min=-1.0, g_max=1.0, G=8))
    run_step("step_ukan_mse", "ukan", [3, 5, 2], 3, 32, 42, "mse", dict(delta_g=0.5, d_pe=8, d_femb=8))

    run_tangent("tan_kan", "kan", [4, 3], 3, 20, 51, dict(g_min=-1.0, g_max=1.0, G=7), unif(-1.3, 1.3))
    run_tangent("tan_kan_base", "kan", [3, 4], 3, 18, 52, dict(g_min=-2.0, g_max=2.0, G=5, base=True),
                unif(-2.5, 2.5))
    run_tangent("tan_kan_k1", "kan", [3, 2], 1, 16, 53, dict(g_min=-1.0, g_max=1.5, G=6), unif(-1.2, 1.7))
    run_tangent("tan_kan_stack", "kan", [2, 5, 3], 3, 24, 54, dict(g_min=-1.0, g_max=1.0, G=6), unif(-1, 1))
    run_tangent("tan_ukan", "ukan", [3, 2], 3, 20, 55, dict(delta_g=0.8, d_pe=8, d_femb=8),
                lambda r, s: r.normal(0, 4, s))
    run_tangent("tan_ukan_stack", "ukan", [2, 4, 2], 2, 16, 56, dict(delta_g=0.5, d_pe=6, d_femb=4),
                lambda r, s: r.normal(0, 2, s))
    run_pinn("pinn_kan", "kan", 3, 61, dict(g_min=-5.0, g_max=5.0, G=10))
    run_pinn("pinn_ukan", "ukan", 3, 62, dict(delta_g=0.5, d_pe=8, d_femb=8))


if __name__ == "__main__":
    main()


def make_checkpoint_golden():
    """A checkpoint written by the reference's own save_checkpoint (checkpoint.py:53-66)."""
    sys.path.insert(0, REF)
    from ukan.checkpoint import save_checkpoint
    from ukan.config import RunConfig
    from ukan.layers import build_model
    model = build_model("kan", [3, 4, 2], 3, seed=5, G=6)
    tensors = {n: f32(p.values) for n, p in model.parameters().items()}
    cfg = RunConfig(model="kan", widths=[3, 4, 2], grid_size=6)
    save_checkpoint(os.path.join(HERE, "ref_checkpoint.ukanckp"), cfg, tensors, {"epoch": 7, "adam_t": 3})
    print("ref_checkpoint.ukanckp written")


if __name__ == "__main__" and "--checkpoint" in sys.argv:
    make_checkpoint_golden()
