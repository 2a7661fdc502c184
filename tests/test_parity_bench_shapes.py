"""Parity at the shapes bench.py times (VERDICT r1 "pin parity at the benchmarked
shapes").  The GPU runs the SAME kernel launches as the bench (full batch, full widths); the
float64 oracle checks them on what it can afford:
  * y / dx of a few sample rows (a row depends only on its own sample: ``oracle.kan_rows``);
  * dcoeffs / dscale of a few features over the WHOLE batch (a feature's gradient depends only
    on its own x column and all of g: ``oracle.kan_feature_grads``).
Bar: grid cells bit-exact, everything else |got - want| <= 1e-6 + 1e-5 |want| (north star).
Reference being replaced: layers.py:57-105 (span_gather / edge_combine), 294-318 (kan_forward),
232-291 (UKAN)."""
import ctypes

import numpy as np
import pytest
import torch

from conftest import assert_close

import oracle
import paper_2408_11200_b200 as P
from paper_2408_11200_b200 import _lib, ops
from paper_2408_11200_b200._lib import check, ptr, stream_ptr

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _layer(d_in, d_out, G, seed, scale_rng=True):
    layer = P.init_layer("kan", d_in, d_out, 3, seed=seed, g_min=-1.0, g_max=1.0, G=G, device=DEV)
    if scale_rng:
        g = torch.Generator(device=DEV).manual_seed(seed + 100)
        with torch.no_grad():
            layer.scale.copy_(torch.rand(layer.scale.shape, device=DEV, generator=g) + 0.5)
    return layer


def _inputs(B, d_in, d_out, seed, tail=0.0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.rand((B, d_in), device=DEV, generator=g) * 2 - 1
    if tail:
        m = torch.rand((B, d_in), device=DEV, generator=g) < tail
        x = torch.where(m, x * 3, x)  # clamp-exercising tail (|x| up to 3)
    gy = torch.randn((B, d_out), device=DEV, generator=g)
    return x, gy


def _check_rows_and_features(layer, x, gy, y, dx, rows, feats):
    """Oracle checks of y/dx rows and dcoeffs/dscale features of one full-batch GPU run."""
    kw = dict(k=layer.k, g_min=layer.g_min, g_max=layer.g_max, G=layer.G)
    coeffs = layer.coeffs.detach().double().cpu().numpy()
    scale = layer.scale.detach().double().cpu().numpy()
    want = oracle.kan_rows(x[rows].double().cpu().numpy(), coeffs, scale, gy[rows].double().cpu().numpy(), **kw)
    cell, _ = ops.kan_locate(x[rows].contiguous(), layer.G, layer.g_min, layer.g_max)
    np.testing.assert_array_equal(cell.cpu().numpy(), want["cell"])
    assert_close(y[rows].cpu().numpy(), want["y"], what="y rows")
    if dx is not None:
        assert_close(dx[rows].cpu().numpy(), want["dx"], what="dx rows")
    g64 = gy.double().cpu().numpy()
    for i in feats:
        wf = oracle.kan_feature_grads(x[:, i].double().cpu().numpy(), coeffs[i], scale[i], g64, **kw)
        assert_close(layer.coeffs.grad[i].cpu().numpy(), wf["dcoeffs"], what=f"dcoeffs[{i}]")
        assert_close(layer.scale.grad[i].cpu().numpy(), wf["dscale"], what=f"dscale[{i}]")


def _full_layer(layer, x, gy, need_dx):
    xt = x.clone().requires_grad_(need_dx)
    y = P.kan_forward(layer, xt)
    (y * gy).sum().backward()
    torch.cuda.synchronize()
    return y.detach(), (xt.grad if need_dx else None)


def test_cfg2_layer0_slice_multichunk():
    """tc2 sweep <8,8,4,4> over 8 chunks of 256 samples (B = 2048) on a 16-feature slice of the
    cfg2 first layer (784 -> 256, G = 32) against the full oracle."""
    layer = _layer(16, 256, 32, seed=1)
    x, gy = _inputs(2048, 16, 256, seed=2)
    xn, gn = x.double().cpu().numpy(), gy.double().cpu().numpy()
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    for need_dx in (False, True):
        for t in layer.parameters().values():
            t.grad = None
        y, dx = _full_layer(layer, x, gy, need_dx)
        want = oracle.kan_forward_backward(xn, p["coeffs"], p["scale"], gn, k=3, g_min=-1.0, g_max=1.0, G=32,
                                           need_dx=need_dx)
        assert_close(y.cpu().numpy(), want["y"], what="y")
        assert_close(layer.coeffs.grad.cpu().numpy(), want["dcoeffs"], what="dcoeffs")
        assert_close(layer.scale.grad.cpu().numpy(), want["dscale"], what="dscale")
        if need_dx:
            assert_close(dx.cpu().numpy(), want["dx"], what="dx")


def test_prep_on_side_stream_then_ws2():
    """The trainer's split backward: ukan_kan_backward_prep on a side stream, then
    ukan_kan_backward_ws2(flags = 1) reusing its records == flags = 0, bitwise, and == oracle."""
    lib = _lib.load()
    B, d_in, d_out, G = 2048, 16, 256, 32
    layer = _layer(d_in, d_out, G, seed=3)
    x, gy = _inputs(B, d_in, d_out, seed=4)
    C, sc = layer.coeffs.detach(), layer.scale.detach()
    nb = lib.ukan_kan_backward_workspace_size(B, d_in, d_out, G, 3)
    outs = []
    for flags in (0, 1):
        ws = torch.full((nb,), 0xAB, device=DEV, dtype=torch.uint8)
        dC, ds = torch.empty_like(C), torch.empty_like(sc)
        if flags:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            prepared = ctypes.c_int32(0)
            with torch.cuda.stream(side):
                check(lib.ukan_kan_backward_prep(ptr(x), None, B, d_in, d_out, G, 3, -1.0, 1.0, ptr(ws), nb,
                                                 ctypes.byref(prepared), stream_ptr()), "prep")
            assert prepared.value == 1
            torch.cuda.current_stream().wait_stream(side)
        check(lib.ukan_kan_backward_ws2(ptr(x), ptr(C), ptr(sc), None, ptr(gy), None, ptr(dC), ptr(ds), None, B, d_in,
                                        d_out, G, 3, -1.0, 1.0, ptr(ws), nb, flags, stream_ptr()), "ws2")
        torch.cuda.synchronize()
        outs.append((dC.cpu().numpy(), ds.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    want = oracle.kan_forward_backward(x.double().cpu().numpy(), C.double().cpu().numpy(), sc.double().cpu().numpy(),
                                       gy.double().cpu().numpy(), k=3, g_min=-1.0, g_max=1.0, G=G, need_dx=False)
    assert_close(outs[1][0], want["dcoeffs"], what="dcoeffs")
    assert_close(outs[1][1], want["dscale"], what="dscale")


def test_cfg2_layer0_full_batch():
    """cfg2 first layer at the bench batch (B = 8192, 784 -> 256, G = 32): the bench's launch
    plan (32 chunks, tc2 sweep <8,8,4,4>, TMEM forward); rows and features vs the oracle."""
    layer = _layer(784, 256, 32, seed=5)
    x, gy = _inputs(8192, 784, 256, seed=6)
    y, _ = _full_layer(layer, x, gy, need_dx=False)
    _check_rows_and_features(layer, x, gy, y, None, rows=[0, 4095, 8191], feats=[0, 391, 783])


def test_cfg3_full_batch_with_dx():
    """configs[2] exactly as benched: KAN 4096 -> 4096, G = 64, B = 65536, 1% clamp tail,
    forward + backward INCLUDING dx; rows (y, dx) and features (dcoeffs, dscale) vs the oracle."""
    layer = _layer(4096, 4096, 64, seed=7)
    x, gy = _inputs(65536, 4096, 4096, seed=8, tail=0.01)
    y, dx = _full_layer(layer, x, gy, need_dx=True)
    # every row holds ~40 clamped entries (1% tail over 4096 features): dx = 0 there (mask)
    _check_rows_and_features(layer, x, gy, y, dx, rows=[0, 32768, 65535], feats=[0, 2047, 4095])


def test_trainer_cfg2_step_matches_oracle_model_step():
    """A cfg2-shaped SplineTrainer.step (KAN [784, 256, 10], G = 32, softmax-CE, Adam) at B = 128
    against oracle.model_step: loss, every gradient and the Adam-updated parameters.  The first
    layer's records come from the side-stream prep (ukan_kan_backward_prep + ws2 flags = 1)."""
    B = 128
    model = P.build_model("kan", [784, 256, 10], 3, seed=0, g_min=-1.0, g_max=1.0, G=32, device=DEV)
    tr = P.SplineTrainer(model, "softmax_cross_entropy", 1e-3, "adam")
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (B, 784)).astype(np.float32)
    y = rng.integers(0, 10, B)
    params = [{n.split(".", 1)[1]: tr.flat.views[n].double().cpu().numpy() for n in tr.flat.names
               if n.startswith(f"layer{i}.")} for i in range(2)]
    cfgs = [dict(k=3, g_min=-1.0, g_max=1.0, G=32)] * 2
    loss_w, grads_w, new_w, _, _ = oracle.model_step("kan", params, cfgs, x.astype(np.float64), y,
                                                     "softmax_cross_entropy", 1e-3)
    loss = tr.read_loss(tr.step(torch.tensor(x, device=DEV), torch.tensor(y, device=DEV)))
    assert abs(loss - loss_w) <= 1e-6 + 1e-5 * abs(loss_w)
    for i in range(2):
        for n in ("coeffs", "scale"):
            assert_close(tr.flat.gviews[f"layer{i}.{n}"].cpu().numpy(), grads_w[i][n], what=f"grad layer{i}.{n}")
    # Adam on the GPU's own gradients (float64 restatement, optim.py:31-54).  Comparing against
    # the oracle's parameters instead would be ill-posed: on step 1 the update is
    # lr * g / (|g| + eps), so a gradient near 0 that is within the 1e-6 atol can move a parameter
    # by up to lr.
    flat_names = [f"layer{i}.{n}" for i in range(2) for n in params[i]]
    p0 = [params[i][n] for i in range(2) for n in params[i]]
    g_gpu = [tr.flat.gviews[name].double().cpu().numpy() for name in flat_names]
    new_p = [a.copy() for a in p0]
    oracle.adam_step(new_p, g_gpu, [np.zeros_like(a) for a in p0], [np.zeros_like(a) for a in p0], 1, 1e-3)
    for name, want in zip(flat_names, new_p):
        assert_close(tr.flat.views[name].cpu().numpy(), want, what=f"updated {name}")


def test_ukan_bench_scale_key_count():
    """UKAN at a bench-scale key count: B = 64, 1024 -> 256, delta_g = 0.5, d_pe = d_femb = 32,
    x ~ N(0, 20^2) with 0.1% tails (n_u ~ 1e5, the regime of the bench's 72.8k-key layer), every
    output and gradient against the full oracle (CG reductions over all n_u rows)."""
    rng = np.random.default_rng(10)
    B, d_in, d_out = 64, 1024, 256
    layer = P.init_layer("ukan", d_in, d_out, 3, seed=11, delta_g=0.5, d_pe=32, d_femb=32, device=DEV)
    x = rng.normal(0, 20.0, (B, d_in))
    m = rng.random(x.shape) < 0.001
    x[m] = np.sign(rng.normal(size=m.sum())) * 10 ** rng.uniform(2, 6, m.sum())
    x = x.astype(np.float32)
    gup = rng.normal(size=(B, d_out)).astype(np.float32)
    n_u = ops.ukan_build_keys(torch.tensor(x, device=DEV), 3, 0.5).n_u
    print(f"n_u = {n_u}")
    assert n_u > 40_000, n_u
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.ukan_forward_backward(x.astype(np.float64), p, gup.astype(np.float64), k=3, delta_g=0.5, d_pe=32)
    xt = torch.tensor(x, device=DEV, requires_grad=True)
    y = P.ukan_forward(layer, xt)
    (y * torch.tensor(gup, device=DEV)).sum().backward()
    assert_close(y.detach().cpu().numpy(), want["y"], what="y")
    assert_close(xt.grad.cpu().numpy(), want["dx"], what="dx")
    for n, t in layer.parameters().items():
        assert_close(t.grad.cpu().numpy(), want["d" + n], what="d" + n)


@pytest.mark.parametrize("n_u", [72_809, 219_922])
def test_cg_gemms_at_bench_key_counts(n_u):
    """The CG GEMMs at the bench / cfg4 key counts (M or K = n_u) against float64 torch:
    table GEMM (tcgen05 tf32 pieces, fwd), dW2 = H^T dT and dH = dT W2^T (FP64 DMMA split-K)."""
    lib = _lib.load()
    g = torch.Generator(device=DEV).manual_seed(n_u)
    d_h, n_out = 128, 4 * 1024
    pre = torch.randn(n_u, d_h, device=DEV, generator=g)
    H = pre * torch.sigmoid(pre)
    W2 = torch.randn(d_h, n_out, device=DEV, generator=g) * (0.1 / d_h ** 0.5)
    b2 = torch.zeros(n_out, device=DEV)
    dT = torch.randn(n_u, n_out, device=DEV, generator=g) * 0.05
    T = torch.empty(n_u, n_out, device=DEV)
    check(lib.ukan_gemm_bias_act(ptr(H), ptr(W2), ptr(b2), ptr(T), None, n_u, n_out, d_h, 0, stream_ptr()), "tab")
    dW2 = torch.empty(d_h, n_out, device=DEV)
    db2 = torch.empty(n_out, device=DEV)
    check(lib.ukan_gemm_tn(ptr(H), ptr(dT), ptr(dW2), ptr(db2), d_h, n_out, n_u, stream_ptr()), "tn")
    dH = torch.empty(n_u, d_h, device=DEV)
    check(lib.ukan_gemm_nt(ptr(dT), ptr(W2), ptr(dH), n_u, d_h, n_out, stream_ptr()), "nt")
    torch.cuda.synchronize()
    H64, W64, dT64 = H.double(), W2.double(), dT.double()
    # the table feeds the fp32 forward: checked at the rtol/atol bar on the forward's scale
    # (fp32-exact products, sums over d_h = 128)
    assert_close(T.cpu().numpy(), (H64 @ W64).cpu().numpy(), rtol=1e-5, atol=1e-6, what="table")
    assert_close(dW2.cpu().numpy(), (H64.T @ dT64).cpu().numpy(), what="dW2")
    assert_close(db2.cpu().numpy(), dT64.sum(0).cpu().numpy(), what="db2")
    assert_close(dH.cpu().numpy(), (dT64 @ W64.T).cpu().numpy(), what="dH")


def test_backward_part_slices_equal_whole_layer_bitwise():
    """ukan_kan_backward_part over uneven feature slices (the DP trainer's bucketed backward)
    reproduces ukan_kan_backward_ws2 bitwise: dcoeffs, dscale and dx."""
    lib = _lib.load()
    B, d_in, d_out, G = 3000, 70, 256, 64
    assert lib.ukan_kan_backward_part_supported(B, d_in, d_out, G, 3) == 1
    layer = _layer(d_in, d_out, G, seed=12)
    x, gy = _inputs(B, d_in, d_out, seed=13, tail=0.02)
    C, sc = layer.coeffs.detach(), layer.scale.detach()
    nb = lib.ukan_kan_backward_workspace_size(B, d_in, d_out, G, 3)
    ws = torch.empty(nb, device=DEV, dtype=torch.uint8)
    dC0, ds0, dx0 = torch.empty_like(C), torch.empty_like(sc), torch.empty_like(x)
    check(lib.ukan_kan_backward_ws2(ptr(x), ptr(C), ptr(sc), None, ptr(gy), ptr(dx0), ptr(dC0), ptr(ds0), None, B, d_in,
                                    d_out, G, 3, -1.0, 1.0, ptr(ws), nb, 0, stream_ptr()), "ws2")
    dC1, ds1, dx1 = torch.full_like(C, float("nan")), torch.full_like(sc, float("nan")), torch.full_like(x, float("nan"))
    prepared = ctypes.c_int32(0)
    check(lib.ukan_kan_backward_prep(ptr(x), None, B, d_in, d_out, G, 3, -1.0, 1.0, ptr(ws), nb,
                                     ctypes.byref(prepared), stream_ptr()), "prep")
    assert prepared.value == 1
    check(lib.ukan_kan_backward_part(ptr(C), ptr(sc), ptr(gy), ptr(dx1), None, None, B, d_in, d_out, G, 3, -1.0, 1.0,
                                     ptr(ws), nb, 0, d_in, 2, stream_ptr()), "dx part")
    for lo, hi in ((0, 13), (13, 64), (64, 70)):
        check(lib.ukan_kan_backward_part(ptr(C), ptr(sc), ptr(gy), None, ptr(dC1), ptr(ds1), B, d_in, d_out, G, 3, -1.0,
                                         1.0, ptr(ws), nb, lo, hi, 1, stream_ptr()), "table part")
    torch.cuda.synchronize()
    assert torch.equal(dC0, dC1) and torch.equal(ds0, ds1) and torch.equal(dx0, dx1)
    want = oracle.kan_forward_backward(x.double().cpu().numpy(), C.double().cpu().numpy(), sc.double().cpu().numpy(),
                                       gy.double().cpu().numpy(), k=3, g_min=-1.0, g_max=1.0, G=G)
    assert_close(dx1.cpu().numpy(), want["dx"], what="dx")
    assert_close(dC1.cpu().numpy(), want["dcoeffs"], what="dcoeffs")
