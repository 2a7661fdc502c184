"""UKAN parity on the GPU: CUDA path vs the reference's golden vectors and the pinned oracle.
Bar: g_id and the unique key set bit-exact; outputs / gradients within rtol 1e-5 / atol 1e-6."""
import numpy as np
import pytest
import torch

from conftest import assert_close, golden_names, load_golden

import oracle
import paper_2408_11200_b200 as P
from paper_2408_11200_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"
NAMES = ["feature_embedding", "cg_w1", "cg_b1", "cg_w2", "cg_b2", "scale"]


def _t(a, grad=False):
    return torch.tensor(np.asarray(a, dtype=np.float32), device=DEV, requires_grad=grad)


def layer_from(params, d_in, d_out, k, delta_g, d_pe, d_femb):
    return P.UkanLayer(d_in, d_out, k, delta_g, d_pe, d_femb, **{n: _t(params[n], True) for n in NAMES})


def run(layer, x, gup):
    xt = _t(x, True)
    y = P.ukan_forward(layer, xt)
    (y * _t(gup)).sum().backward()
    out = dict(y=y.detach().cpu().numpy(), dx=xt.grad.cpu().numpy())
    for n, p in layer.parameters().items():
        out["d" + n] = p.grad.cpu().numpy()
    return out


def check_keys(x, k, delta_g, want_gid, want_keys):
    x_t = _t(x)
    keys = ops.ukan_build_keys(x_t, k, delta_g)
    d_in = x.shape[1]
    K = k + 1
    kf = keys.key_f.cpu().numpy().astype(np.int64)
    kg = keys.key_g.cpu().numpy()
    # same set as np.unique(group*d_in + f) (layers.py:275)
    np.testing.assert_array_equal(np.sort(kg * d_in + kf), want_keys)
    # feature-major, sorted within feature
    order = np.lexsort((kg, kf))
    np.testing.assert_array_equal(order, np.arange(len(kf)))
    # window rows reproduce g_id bit-exactly: base = idx(f, g_id div K)*K + g_id mod K
    base = keys.base_row.cpu().numpy().astype(np.int64)
    idx, off = base // K, base % K
    f = np.broadcast_to(np.arange(d_in)[None, :], x.shape)
    np.testing.assert_array_equal(kf[idx], f)
    np.testing.assert_array_equal(kg[idx] * K + off, want_gid)


@pytest.mark.parametrize("name", golden_names("ukan_"))
def test_ukan_golden(name):
    g = load_golden(name)
    d_in, d_out, k = int(g["d_in"]), int(g["d_out"]), int(g["k"])
    dg, d_pe, d_femb = float(g["delta_g"]), int(g["d_pe"]), int(g["d_femb"])
    check_keys(g["x"], k, dg, g["g_id"], g["keys"])
    layer = layer_from(g, d_in, d_out, k, dg, d_pe, d_femb)
    r = run(layer, g["x"], g["g_up"])
    for key in ["y", "dx"] + ["d" + n for n in NAMES]:
        assert_close(r[key], g[key], what=f"{name}.{key}")


def random_case(B, d_in, d_out, k, dg, d_pe, d_femb, seed, sigma=10.0, tails=0.0):
    rng = np.random.default_rng(seed)
    layer = P.init_layer("ukan", d_in, d_out, k, seed=seed, delta_g=dg, d_pe=d_pe, d_femb=d_femb)
    x = rng.normal(0, sigma, (B, d_in))
    if tails:
        m = rng.random(x.shape) < tails
        x[m] = np.sign(rng.normal(size=m.sum())) * 10 ** rng.uniform(2, 6, m.sum())
    x = x.astype(np.float32)
    gup = rng.normal(size=(B, d_out)).astype(np.float32)
    return layer, x, gup


def check_against_oracle(layer, x, gup):
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.ukan_forward_backward(x.astype(np.float64), p, gup.astype(np.float64), k=layer.k,
                                        delta_g=layer.delta_g, d_pe=layer.d_pe)
    got = run(layer, x, gup)
    for key in got:
        assert_close(got[key], want[key], what=key)


def test_ukan_256_medium():
    check_against_oracle(*random_case(256, 64, 64, 3, 1.0, 8, 8, seed=1))


def test_ukan_cfg4_shaped_subbatch():
    """cfg4 shape (d_pe = d_femb = 32, delta_g = 0.5, x ~ N(0, 20^2) with 0.1% heavy tails)
    on 64 x 128 -> 128 so the oracle stays small."""
    check_against_oracle(*random_case(64, 128, 128, 3, 0.5, 32, 32, seed=2, sigma=20.0, tails=0.001))


@pytest.mark.parametrize("k", [0, 1, 2, 5])
def test_ukan_degrees(k):
    check_against_oracle(*random_case(100, 5, 7, k, 0.7, 6, 4, seed=10 + k))


def test_nonfinite_raises_domain_error():
    layer, x, _ = random_case(4, 2, 2, 3, 1.0, 8, 8, seed=3)
    x[1, 1] = np.inf
    with pytest.raises(P.DomainError):
        P.ukan_forward(layer, _t(x))


def test_zero_generator_everywhere():   # test_layers.py:116-121
    layer = P.init_layer("ukan", 2, 2, 3, seed=0)
    with torch.no_grad():
        for p in (layer.cg_w1, layer.cg_b1, layer.cg_w2, layer.cg_b2):
            p.zero_()
    y = P.ukan_forward(layer, _t([[1e6, -1e6], [0.0, 0.3]]))
    assert torch.all(y == 0)


def test_constant_generator_partition_of_unity():   # test_layers.py:123-131
    layer = P.init_layer("ukan", 1, 1, 3, seed=0)
    with torch.no_grad():
        layer.cg_w1.zero_(); layer.cg_w2.zero_(); layer.cg_b1.zero_(); layer.cg_b2.fill_(2.75)
    x = _t(np.linspace(-100.0, 100.0, 31)[:, None])
    np.testing.assert_allclose(P.ukan_forward(layer, x).detach().cpu().numpy(), 2.75, rtol=1e-6)


def test_cg_coefficients_and_index_error():
    layer = P.init_layer("ukan", 2, 3, 3, seed=2)
    c = P.cg_coefficients(layer, 1, -2)
    assert tuple(c.shape) == (3, 4)
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want, _ = oracle.cg_forward(np.array([-2 * 2 + 1]), 2, p["feature_embedding"], p["cg_w1"], p["cg_b1"],
                                p["cg_w2"], p["cg_b2"], 8, 4, 3)
    assert_close(c.detach().cpu().numpy(), want[0].T, what="cg_coefficients")
    with pytest.raises(IndexError):
        P.cg_coefficients(layer, 2, 0)


def test_dedup_flag_transparent():
    layer, x, _ = random_case(50, 2, 3, 3, 1.0, 8, 8, seed=5, sigma=3.0)
    a = P.ukan_forward(layer, _t(x), dedup=True)
    b = P.ukan_forward(layer, _t(x), dedup=False)
    assert torch.equal(a, b)


def test_keys_at_scale_heavy_tails():
    """cfg4 batch/width (65536 x 1024, x ~ N(0, 20^2), 0.1% tails to 1e6): key set and window
    rows checked against NumPy's locate + np.unique at full size."""
    rng = np.random.default_rng(7)
    x = rng.normal(0, 20.0, (65536, 1024))
    m = rng.random(x.shape) < 0.001
    x[m] = np.sign(rng.normal(size=m.sum())) * 10 ** rng.uniform(2, 6, m.sum())
    x = x.astype(np.float32)
    g_id, _, group, _ = oracle.ukan_locate(x.astype(np.float64), 0.5, 3)
    f = np.broadcast_to(np.arange(1024)[None, :], x.shape)
    want_keys = np.unique(np.concatenate([(group * 1024 + f).ravel(), ((group + 1) * 1024 + f).ravel()]))
    check_keys(x, 3, 0.5, g_id, want_keys)


@pytest.mark.parametrize("d_out,sigma", [(40, 2.0), (37, 30.0)])
def test_ukan_segmented_sweep_multi_chunk(d_out, sigma):
    """B = 1000 spans four 256-sample chunks (partial last one).  sigma = 2 packs every sample
    of a feature into one 32-row tile (> 256 staged samples -> several batches); sigma = 30
    spreads them over many tiles; d_out = 37 takes the 4-byte staging path."""
    layer, x, gup = random_case(1000, 3, d_out, 3, 1.0, 8, 8, seed=40 + d_out, sigma=sigma)
    check_against_oracle(layer, x, gup)
    for p in layer.parameters().values():
        p.grad = None
    a = run(layer, x, gup)
    for p in layer.parameters().values():
        p.grad = None
    b = run(layer, x, gup)
    for key in a:
        np.testing.assert_array_equal(a[key], b[key])


@pytest.mark.parametrize("B,d_in,d_out,dg,sigma", [(1500, 12, 64, 0.4, 1.0), (700, 9, 100, 1.0, 7.0), (257, 33, 256, 0.5, 2.0),
                                                  (2000, 16, 64, 0.4, 0.3), (1, 5, 64, 0.4, 1.0), (5, 7, 68, 0.4, 1.0),
                                                  (300, 6, 128, 0.4, 1.0)])
def test_ukan_dense_layer_on_tensor_cores(B, d_in, d_out, dg, sigma):
    """Dense UKAN layers (every feature's virtual table <= 67 rows, the cfg5 regime) take the KAN
    FP64 tensor-core backward (ukan_ukan_backward_dense): multi-chunk, ragged output tiles
    (d_out = 100), 8- and 16-row-block plans, few-row segments (sample-split sweep), and for
    d_out >= 128 the TMEM-gather forward over the segments; oracle parity and bitwise determinism."""
    from paper_2408_11200_b200 import _lib
    layer, x, gup = random_case(B, d_in, d_out, 3, dg, 8, 8, seed=B + d_out, sigma=sigma)
    keys = ops.ukan_build_keys(_t(x), 3, dg)
    assert 0 < keys.max_rows <= 67
    lib = _lib.load()
    assert lib.ukan_ukan_backward_dense_workspace_size(B, d_in, d_out, keys.n_u, keys.max_rows, 3) > 0
    if d_out >= 128 and keys.max_rows >= 4:  # the TMEM-gather forward over the segments too
        assert lib.ukan_ukan_forward_dense_workspace_size(B, d_in, d_out, keys.max_rows, 3) > 0
    check_against_oracle(layer, x, gup)
    for p in layer.parameters().values():
        p.grad = None
    a = run(layer, x, gup)
    for p in layer.parameters().values():
        p.grad = None
    b = run(layer, x, gup)
    for key in a:
        np.testing.assert_array_equal(a[key], b[key])


def test_ukan_dense_stack_training_step():
    """A cfg5-shaped (scaled-down) UKAN stack through SplineTrainer: layers 1 and 2 are dense and
    need dx; the step's gradients match oracle.model_step."""
    widths, dg = [8, 64, 64], 0.4
    kw = dict(delta_g=dg, d_pe=8, d_femb=8)
    rng = np.random.default_rng(9)
    x = rng.normal(size=(700, widths[0])).astype(np.float32)
    t = rng.normal(size=(700, widths[-1])).astype(np.float32)
    model = P.build_model("ukan", widths, 3, seed=0, device=DEV, **kw)
    params = [{n: v.detach().double().cpu().numpy() for n, v in L.parameters().items()} for L in model.layers]
    tr = P.SplineTrainer(model, "mse", 1e-3, "adam")
    tr.read_loss(tr.step(torch.tensor(x, device=DEV), torch.tensor(t, device=DEV)))
    grad = tr.flat.grad.cpu().numpy()
    cfgs = [dict(k=3, delta_g=dg, d_pe=8) for _ in model.layers]
    _, want, _, _, _ = oracle.model_step("ukan", params, cfgs, x.astype(np.float64), t.astype(np.float64), "mse", 1e-3)
    off = 0
    for li, L in enumerate(model.layers):
        for n, v in L.parameters().items():
            g = grad[off:off + v.numel()].reshape(v.shape)
            off += v.numel()
            assert_close(g, want[li][n], what=f"layer{li}.{n}")


def test_ukan_large_batch_sorted_sweep_with_row_hint():
    """B = 8192 > 6144: the 2*B*K bound used to keep the batch off the per-feature sorted sweep;
    with the key build's max_rows (ukan_ukan_backward2) it takes that sweep.  Sparse segments
    (> 67 rows, not the dense path), a d_out that is not a multiple of 8."""
    layer, x, gup = random_case(8192, 4, 40, 3, 0.5, 8, 8, seed=77, sigma=30.0)
    keys = ops.ukan_build_keys(_t(x), 3, 0.5)
    assert 67 < keys.max_rows < 2 * 8192 * 4
    check_against_oracle(layer, x, gup)
