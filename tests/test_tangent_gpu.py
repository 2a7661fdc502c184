"""F2 parity on the GPU: the forward tangent (JVP) of the KAN / UKAN layers and the reverse pass
through it (forward-over-reverse, what pinn_loss needs: tasks.py:153-166), through the drop-in
API (kan_forward_tangent / ukan_forward_tangent / Model.forward_tangent / pinn_loss) against the
reference's golden vectors (tests/golden/tan_*, pinn_*) and the pinned CPU oracle.
Bar: rtol 1e-5 / atol 1e-6 (north star)."""
import numpy as np
import pytest
import torch

from conftest import assert_close, golden_names, load_golden

import oracle
import paper_2408_11200_b200 as P

pytestmark = pytest.mark.gpu
DEV = "cuda"
UKAN_P = ["feature_embedding", "cg_w1", "cg_b1", "cg_w2", "cg_b2", "scale"]


def _t(a, grad=False):
    return torch.tensor(np.asarray(a, dtype=np.float32), device=DEV, requires_grad=grad)


def model_from_golden(g, widths):
    kind, k = str(g["kind"]), int(g["k"])
    layers = []
    for li in range(len(widths) - 1):
        pre = f"layer{li}."
        if kind == "kan":
            bw = g.get(pre + "base_weight")
            layers.append(P.KanLayer(widths[li], widths[li + 1], k, float(g["kw_g_min"]), float(g["kw_g_max"]),
                                     int(g["kw_G"]), _t(g[pre + "coeffs"], True), _t(g[pre + "scale"], True),
                                     None if bw is None else _t(bw, True)))
        else:
            d_pe, d_femb = int(g["kw_d_pe"]), int(g["kw_d_femb"])
            layers.append(P.UkanLayer(widths[li], widths[li + 1], k, float(g["kw_delta_g"]), d_pe, d_femb,
                                      *[_t(g[pre + n], True) for n in UKAN_P]))
    return P.Model(kind=kind, layers=layers)


@pytest.mark.parametrize("name", golden_names("tan_"))
def test_tangent_golden(name):
    g = load_golden(name)
    widths = [int(w) for w in g["widths"]]
    model = model_from_golden(g, widths)
    x = _t(g["x"], True)
    y, ty = model.forward_tangent(x, _t(g["tx"]))
    ((y * _t(g["g_up"])).sum() + (ty * _t(g["g_tan"])).sum()).backward()
    assert_close(y.detach().cpu().numpy(), g["y"], what=f"{name}.y")
    assert_close(ty.detach().cpu().numpy(), g["ty"], what=f"{name}.ty")
    assert_close(x.grad.cpu().numpy(), g["dx"], what=f"{name}.dx")
    for n, p in model.parameters().items():
        assert_close(p.grad.cpu().numpy(), g["d" + n], what=f"{name}.d{n}")


@pytest.mark.parametrize("name", golden_names("pinn_"))
def test_pinn_loss_golden(name):
    g = load_golden(name)
    model = model_from_golden(g, [1, 5, 1])
    loss = P.pinn_loss(model.forward, P.PinnProblem(1.0, -5.0, 5.0, g["colloc"].shape[0]), g["colloc"])
    loss.backward()
    assert_close(loss.item(), float(g["loss"]), what=f"{name}.loss")
    for n, p in model.parameters().items():
        assert_close(p.grad.cpu().numpy(), g["d" + n], what=f"{name}.d{n}")


def _kan_case(B, d_in, d_out, k, G, seed, base=False, outliers=0.0):
    rng = np.random.default_rng(seed)
    layer = P.init_layer("kan", d_in, d_out, k, seed=seed, g_min=-1.0, g_max=1.5, G=G, base=base)
    with torch.no_grad():
        layer.scale.copy_(torch.tensor(rng.uniform(0.5, 1.5, (d_in, d_out)), dtype=torch.float32))
    x = rng.uniform(-1.0, 1.5, (B, d_in)).astype(np.float32)
    if outliers:
        m = rng.random(x.shape) < outliers
        x[m] = rng.uniform(-4, 4, m.sum())
    tx = rng.normal(size=(B, d_in)).astype(np.float32)
    gy = rng.normal(size=(B, d_out)).astype(np.float32)
    gt = rng.normal(size=(B, d_out)).astype(np.float32)
    return layer, x, tx, gy, gt


@pytest.mark.parametrize("B,d_in,d_out,k,G,base", [(64, 3, 5, 3, 7, False), (100, 4, 40, 0, 5, False),
                                                   (77, 5, 6, 1, 9, True), (50, 2, 33, 2, 12, False),
                                                   (40, 3, 4, 5, 6, True), (300, 6, 70, 3, 40, False)])
def test_kan_tangent_vs_oracle(B, d_in, d_out, k, G, base):
    layer, x, tx, gy, gt = _kan_case(B, d_in, d_out, k, G, seed=B + k, base=base, outliers=0.1)
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.kan_tangent_forward_backward(x, tx, p["coeffs"], p["scale"], gy.astype(np.float64),
                                               gt.astype(np.float64), k=k, g_min=-1.0, g_max=1.5, G=G,
                                               base_weight=p.get("base_weight"))
    xt, txt = _t(x, True), _t(tx, True)
    y, ty = P.kan_forward_tangent(layer, xt, txt)
    ((y * _t(gy)).sum() + (ty * _t(gt)).sum()).backward()
    got = dict(y=y, ty=ty, dx=xt.grad, dtx=txt.grad, dcoeffs=layer.coeffs.grad, dscale=layer.scale.grad)
    if base:
        got["dbase_weight"] = layer.base_weight.grad
    for key, v in got.items():
        assert_close(v.detach().cpu().numpy(), want[key], what=key)


@pytest.mark.parametrize("B,d_in,d_out,k,dg", [(40, 3, 2, 3, 0.8), (64, 2, 35, 2, 0.3), (33, 4, 5, 0, 1.7)])
def test_ukan_tangent_vs_oracle(B, d_in, d_out, k, dg):
    rng = np.random.default_rng(B)
    layer = P.init_layer("ukan", d_in, d_out, k, seed=B, delta_g=dg, d_pe=8, d_femb=6)
    x = rng.normal(0, 4, (B, d_in)).astype(np.float32)
    tx = rng.normal(size=(B, d_in)).astype(np.float32)
    gy = rng.normal(size=(B, d_out)).astype(np.float32)
    gt = rng.normal(size=(B, d_out)).astype(np.float32)
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.ukan_tangent_forward_backward(x, tx, p, gy.astype(np.float64), gt.astype(np.float64), k=k,
                                                delta_g=dg, d_pe=8)
    xt, txt = _t(x, True), _t(tx, True)
    y, ty = P.ukan_forward_tangent(layer, xt, txt)
    ((y * _t(gy)).sum() + (ty * _t(gt)).sum()).backward()
    got = dict(y=y, ty=ty, dx=xt.grad, dtx=txt.grad, **{"d" + n: t.grad for n, t in layer.parameters().items()})
    for key, v in got.items():
        assert_close(v.detach().cpu().numpy(), want[key], rtol=1e-5, atol=1e-5 if key.startswith("dcg") else 1e-6,
                     what=key)


def test_tangent_matches_finite_difference():   # test_layers.py:194-207
    layer = P.init_layer("ukan", 1, 1, 3, seed=8, delta_g=1.1)
    for tv in (-3.3, 0.21, 4.9):
        _, ty = P.ukan_forward_tangent(layer, [[tv]], [[1.0]])
        h = 1e-2
        fd = (P.ukan_forward(layer, [[tv + h]]) - P.ukan_forward(layer, [[tv - h]])).item() / (2 * h)
        assert abs(ty.item() - fd) < 2e-3 * max(1.0, abs(fd))


def test_tangent_deterministic_and_empty():
    layer, x, tx, gy, gt = _kan_case(500, 4, 36, 3, 300, seed=3)
    runs = []
    for _ in range(2):
        layer.coeffs.grad = None
        layer.scale.grad = None
        y, ty = P.kan_forward_tangent(layer, _t(x), _t(tx))
        (ty * _t(gt)).sum().backward()
        runs.append((ty.detach().cpu().numpy(), layer.coeffs.grad.cpu().numpy(), layer.scale.grad.cpu().numpy()))
    for a, b in zip(*runs):
        np.testing.assert_array_equal(a, b)
    y, ty = P.kan_forward_tangent(layer, torch.zeros((0, 4), device=DEV), torch.zeros((0, 4), device=DEV))
    assert ty.shape == (0, 36)


def test_tangent_seed_shape_error():
    layer, x, tx, _, _ = _kan_case(4, 3, 2, 3, 5, seed=1)
    with pytest.raises(P.DimensionError):
        P.kan_forward_tangent(layer, _t(x), _t(tx[:, :2]))
