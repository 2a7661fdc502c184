"""KAN parity on the GPU: the CUDA path (through the drop-in layer API / C ABI) against the
reference's golden vectors and the pinned CPU oracle.  Bar: grid cells bit-exact; outputs and
gradients within rtol 1e-5 / atol 1e-6 (north star)."""
import numpy as np
import pytest
import torch

from conftest import assert_close, golden_names, load_golden

import oracle
import paper_2408_11200_b200 as P
from paper_2408_11200_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _t(a, grad=False):
    return torch.tensor(np.asarray(a, dtype=np.float32), device=DEV, requires_grad=grad)


def make_layer(d_in, d_out, k, G, g_min, g_max, coeffs, scale, base_weight=None):
    return P.KanLayer(d_in, d_out, k, g_min, g_max, G, _t(coeffs, True), _t(scale, True),
                      None if base_weight is None else _t(base_weight, True))


def run_layer(layer, x, g_up, need_dx=True):
    xt = _t(x, need_dx)
    y = P.kan_forward(layer, xt)
    (y * _t(g_up)).sum().backward()
    out = dict(y=y.detach().cpu().numpy(), dcoeffs=layer.coeffs.grad.cpu().numpy(),
               dscale=layer.scale.grad.cpu().numpy())
    if need_dx:
        out["dx"] = xt.grad.cpu().numpy()
    if layer.base_weight is not None:
        out["dbase_weight"] = layer.base_weight.grad.cpu().numpy()
    return out


@pytest.mark.parametrize("name", golden_names("kan_"))
def test_kan_golden(name):
    g = load_golden(name)
    d_in, d_out, k, G = int(g["d_in"]), int(g["d_out"]), int(g["k"]), int(g["G"])
    layer = make_layer(d_in, d_out, k, G, float(g["g_min"]), float(g["g_max"]), g["coeffs"], g["scale"],
                       g.get("base_weight"))
    cell, _ = ops.kan_locate(_t(g["x"]), G, float(g["g_min"]), float(g["g_max"]))
    np.testing.assert_array_equal(cell.cpu().numpy(), g["cell"])
    r = run_layer(layer, g["x"], g["g_up"])
    for key in ("y", "dx", "dcoeffs", "dscale", "dbase_weight"):
        if key in g:
            assert_close(r[key], g[key], what=f"{name}.{key}")


def random_case(B, d_in, d_out, k, G, g_min=-1.0, g_max=1.0, seed=0, outliers=0.0, base=False):
    rng = np.random.default_rng(seed)
    layer = P.init_layer("kan", d_in, d_out, k, seed=seed, g_min=g_min, g_max=g_max, G=G, base=base)
    with torch.no_grad():
        layer.scale.copy_(torch.tensor(rng.uniform(0.5, 1.5, (d_in, d_out)), dtype=torch.float32))
    x = rng.uniform(g_min, g_max, (B, d_in)).astype(np.float32)
    if outliers:
        m = rng.random(x.shape) < outliers
        x[m] = rng.uniform(-3, 3, m.sum()) * (g_max - g_min)
    gup = rng.normal(size=(B, d_out)).astype(np.float32)
    return layer, x, gup


def check_against_oracle(layer, x, gup, need_dx=True):
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.kan_forward_backward(x.astype(np.float64), p["coeffs"], p["scale"], gup.astype(np.float64),
                                       k=layer.k, g_min=layer.g_min, g_max=layer.g_max, G=layer.G,
                                       base_weight=p.get("base_weight"), need_dx=need_dx)
    got = run_layer(layer, x, gup, need_dx)
    cell, _ = ops.kan_locate(_t(x), layer.G, layer.g_min, layer.g_max)
    np.testing.assert_array_equal(cell.cpu().numpy(), want["cell"])
    for key in got:
        assert_close(got[key], want[key], what=key)


def test_cfg1_full_batch():
    """configs[0]: KAN 64->64, G=10, k=3, B=1024 (the reference's CPU-runnable case)."""
    check_against_oracle(*random_case(1024, 64, 64, 3, 10, seed=1))


def test_cfg2_layer1_subbatch():
    """configs[1] first layer (784->256, G=32) on a 48-row slice (the oracle materialises
    [B, d_in, K, d_out] windows); the first layer needs no dx."""
    layer, x, gup = random_case(48, 784, 256, 3, 32, seed=2)
    check_against_oracle(layer, x, gup, need_dx=False)


def test_cfg2_layer2():
    check_against_oracle(*random_case(512, 256, 10, 3, 32, seed=3))


def test_cfg3_shaped_subbatch():
    """configs[2] shape on d_in (4096) and G (64) with a 1% clamp-exercising tail; d_out cut to
    256 and B to 4 so the float64 oracle fits in host memory."""
    check_against_oracle(*random_case(4, 4096, 256, 3, 64, seed=4, outliers=0.01))


@pytest.mark.parametrize("k", [0, 1, 2, 4, 5, 7, 10])
def test_degrees(k):
    check_against_oracle(*random_case(300, 9, 33, k, 11, g_min=-0.5, g_max=2.5, seed=10 + k, outliers=0.05))


def test_base_branch_and_odd_sizes():
    check_against_oracle(*random_case(257, 13, 19, 3, 7, seed=5, outliers=0.1, base=True))


def test_large_grid_global_accumulator():
    """G = 4096 (reference bench trend sweep) exercises the fp64 global-workspace path."""
    check_against_oracle(*random_case(700, 4, 32, 3, 4096, seed=6))


def test_deterministic_backward():
    layer, x, gup = random_case(3000, 64, 96, 3, 16, seed=7)
    a = run_layer(layer, x, gup)
    layer.coeffs.grad = None
    layer.scale.grad = None
    b = run_layer(layer, x, gup)
    for key in a:
        np.testing.assert_array_equal(a[key], b[key])


def test_nan_raises_index_error():
    layer, x, _ = random_case(8, 3, 4, 3, 5, seed=8)
    x[3, 1] = np.nan
    with pytest.raises(IndexError):
        P.kan_forward(layer, _t(x))


def test_empty_batch():
    layer, _, _ = random_case(1, 3, 4, 3, 5, seed=9)
    y = P.kan_forward(layer, torch.zeros((0, 3), device=DEV))
    assert y.shape == (0, 4)


def test_dimension_error():
    layer, _, _ = random_case(1, 3, 4, 3, 5, seed=9)
    with pytest.raises(P.DimensionError):
        P.kan_forward(layer, torch.zeros((2, 4), device=DEV))


def test_constant_coefficients_partition_of_unity():   # test_layers.py:211-216
    layer = P.init_layer("kan", 3, 2, 3, seed=0, g_min=-1, g_max=1, G=5)
    with torch.no_grad():
        layer.coeffs.fill_(1.5)
    x = torch.tensor(np.linspace(-1, 0.99, 7)[:, None].repeat(3, axis=1), dtype=torch.float32, device=DEV)
    np.testing.assert_allclose(P.kan_forward(layer, x).detach().cpu().numpy(), 4.5, rtol=1e-6)


@pytest.mark.parametrize("B,d_in,d_out,G", [(8192, 784, 256, 32), (65536, 256, 512, 64)])
def test_full_size_checksums(B, d_in, d_out, G):
    """Full-batch, size-independent identities (the oracle cannot run these sizes):
    sum_r dC[i,r,o] = scale[i,o] * sum_b g[b,o]  (partition of unity of the basis), and
    sum_i scale[i,o] * dscale[i,o] = sum_b g[b,o] * y[b,o]."""
    layer, x, gup = random_case(B, d_in, d_out, 3, G, seed=11)
    xt = _t(x)
    y = P.kan_forward(layer, xt)
    gy = _t(gup)
    (y * gy).sum().backward()
    g64 = gy.double()
    sc = layer.scale.detach().double()
    lhs = layer.coeffs.grad.double().sum(dim=1)
    rhs = sc * g64.sum(dim=0)[None, :]
    assert_close(lhs.cpu().numpy(), rhs.cpu().numpy(), rtol=1e-5, atol=1e-4, what="sum_r dC")
    lhs2 = (sc * layer.scale.grad.double()).sum(dim=0)
    rhs2 = (g64 * y.detach().double()).sum(dim=0)
    assert_close(lhs2.cpu().numpy(), rhs2.cpu().numpy(), rtol=1e-4, atol=1e-3, what="scale.dscale")


@pytest.mark.parametrize("B,d_in,d_out,k,G,base", [(1000, 6, 40, 3, 200, True), (513, 5, 70, 7, 150, False),
                                                   (300, 3, 10, 10, 90, True), (257, 2, 33, 0, 3000, False)])
def test_fine_grid_sorted_sweep(B, d_in, d_out, k, G, base):
    """Fine grids (R > 72 or K > 6) run the sorted-chunk sweep (kan_bwd_wide.cu)."""
    check_against_oracle(*random_case(B, d_in, d_out, k, G, seed=20 + k, outliers=0.05, base=base))


def test_fine_grid_clustered_cells():
    """Hundreds of samples per cell just below a 32-row tile boundary: the backward extension
    over cells r0-k..r0-1 must walk more than one 32-entry step, and chunk-crossing runs of one
    cell must accumulate in order."""
    layer, x, gup = random_case(1500, 3, 36, 3, 1000, seed=31)
    dg = 2.0 / 1000
    rng = np.random.default_rng(32)
    cells = rng.choice([30, 31, 62, 63, 64, 999], size=x.shape)
    x[:] = (-1.0 + (cells + rng.uniform(0.1, 0.9, x.shape)) * dg).astype(np.float32)
    check_against_oracle(layer, x, gup)
    layer.coeffs.grad = None
    layer.scale.grad = None
    a = run_layer(layer, x, gup)
    layer.coeffs.grad = None
    layer.scale.grad = None
    b = run_layer(layer, x, gup)
    for key in a:
        np.testing.assert_array_equal(a[key], b[key])


@pytest.mark.parametrize("G", [37, 48, 64])
def test_tmem_forward_fine_grid_variants(G):
    """TMEM-gather forward around its plan boundaries: G=37 (5-deep ring, two TMEM slabs), G=48
    (3-deep ring, one slab) and G=64 (one slab of 67 x 4 columns); d_out >= 128 takes that path."""
    check_against_oracle(*random_case(300, 5, 130, 3, G, seed=60 + G, outliers=0.05), need_dx=False)


@pytest.mark.parametrize("B,d_in,d_out,G,outliers", [(1, 1, 33, 3, 0.0), (37, 5, 100, 10, 0.2), (1024, 64, 64, 10, 0.05),
                                                     (1500, 16, 200, 40, 0.1), (6000, 16, 64, 10, 0.0),
                                                     (300, 2, 4096, 97, 0.0)])
def test_small_layer_path(B, d_in, d_out, G, outliers):
    """kan_small.cu (d_in * d_out <= 2^14, B * d_in * d_out <= 6 Mi, k = 3, no base): ragged output
    tiles (d_out not a multiple of 64), one sample, one feature, 375 samples per thread, the
    largest grid (R = 100 rows: 4 sample splits), outliers."""
    layer, x, gup = random_case(B, d_in, d_out, 3, G, seed=B + d_in, outliers=outliers)
    check_against_oracle(layer, x, gup)


def test_small_layer_prepared_records_and_determinism():
    """SplineTrainer builds the first layer's records on a side stream (ukan_kan_backward_prep ->
    kan_small_records); the step must equal the eager autograd step bitwise, twice."""
    x = np.random.default_rng(3).uniform(-1, 1, (1024, 64)).astype(np.float32)
    t = np.random.default_rng(4).normal(size=(1024, 64)).astype(np.float32)
    grads = []
    for _ in range(2):
        model = P.build_model("kan", [64, 64], 3, seed=0, device=DEV, g_min=-1.0, g_max=1.0, G=10)
        tr = P.SplineTrainer(model, "mse", 1e-3, "adam")
        tr.read_loss(tr.step(torch.tensor(x, device=DEV), torch.tensor(t, device=DEV)))
        grads.append(tr.flat.grad.cpu().numpy().copy())
    np.testing.assert_array_equal(grads[0], grads[1])
    layer = P.init_layer("kan", 64, 64, 3, seed=0, g_min=-1.0, g_max=1.0, G=10)
    p = {n: v.detach().double().cpu().numpy() for n, v in layer.parameters().items()}
    cfg = dict(k=3, g_min=-1.0, g_max=1.0, G=10)
    _, want, _, _, _ = oracle.model_step("kan", [p], [cfg], x.astype(np.float64), t.astype(np.float64), "mse", 1e-3)
    nC = p["coeffs"].size
    assert_close(grads[0][:nC].reshape(p["coeffs"].shape), want[0]["coeffs"], what="dcoeffs")
    assert_close(grads[0][nC:].reshape(p["scale"].shape), want[0]["scale"], what="dscale")
