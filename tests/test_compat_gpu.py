"""The literal drop-in: the UNMODIFIED reference package (``ukan``, installed into
the git-ignored ``baseline/_ref`` by ``__graft_entry__.build()`` from /root/reference) runs its own
layer API, tape (``ukan.tensor.backward``), ``Model`` and ``train`` loop with
``paper_2408_11200_b200.compat.install(ukan)`` routing ``kan_forward`` / ``ukan_forward`` through
the C ABI.  Results are compared with the reference's own float64 path on the same
fp32-representable inputs at the north-star bar (rtol 1e-5 / atol 1e-6); the reference's tests
at 1e-10 (test_layers.py:225-234) are restated at that fp32 bar."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, assert_close

pytestmark = pytest.mark.gpu
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ukan():
    if not os.path.isdir(os.path.join(REF, "ukan")):
        pytest.fail("baseline/_ref/ukan is missing: run __graft_entry__.build() where /root/reference exists")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ukan as U
    yield U
    from paper_2408_11200_b200 import compat
    compat.uninstall()


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def _round_params(layer):
    for p in layer.parameters().values():
        p.values[...] = _f32(p.values)


def _run(U, layer, x, gup):
    """y and every gradient through the reference's tape with x as a recorded node."""
    T = U.tensor
    xt = T.parameter(x.copy())
    for p in layer.parameters().values():
        p.grad = None
    y = layer(xt)
    T.backward(T.sum_all(T.mul(y, T.as_tensor(gup))))
    out = {"y": y.values.copy(), "dx": xt.grad.copy()}
    out.update({"d" + n: p.grad.copy() for n, p in layer.parameters().items()})
    return out


def _both(U, layer, x, gup):
    from paper_2408_11200_b200 import compat
    compat.uninstall()
    want = _run(U, layer, x, gup)
    compat.install(U)
    got = _run(U, layer, x, gup)
    compat.uninstall()
    return got, want


def test_kan_layer_through_reference_tape(ukan):
    rng = np.random.default_rng(1)
    layer = ukan.init_layer("kan", 24, 40, 3, seed=1, g_min=-1.0, g_max=1.0, G=16)
    _round_params(layer)
    layer.scale.values[...] = _f32(rng.uniform(0.5, 1.5, layer.scale.shape))
    x = _f32(rng.uniform(-1.2, 1.2, (300, 24)))
    gup = _f32(rng.normal(size=(300, 40)))
    got, want = _both(ukan, layer, x, gup)
    for key in want:
        assert_close(got[key], want[key], what="compat kan " + key)


def test_kan_base_branch_and_degrees(ukan):
    rng = np.random.default_rng(2)
    for k, base in ((1, True), (5, False)):
        layer = ukan.init_layer("kan", 5, 7, k, seed=k, g_min=-2.0, g_max=2.0, G=9, base=base)
        _round_params(layer)
        x = _f32(rng.uniform(-3, 3, (50, 5)))
        gup = _f32(rng.normal(size=(50, 7)))
        got, want = _both(ukan, layer, x, gup)
        for key in want:
            assert_close(got[key], want[key], what=f"compat kan k={k} {key}")


def test_ukan_layer_through_reference_tape(ukan):
    rng = np.random.default_rng(3)
    layer = ukan.init_layer("ukan", 16, 12, 3, seed=3, delta_g=0.5, d_pe=16, d_femb=8)
    _round_params(layer)
    x = _f32(rng.normal(0, 10.0, (128, 16)))
    gup = _f32(rng.normal(size=(128, 12)))
    got, want = _both(ukan, layer, x, gup)
    for key in want:
        assert_close(got[key], want[key], what="compat ukan " + key)


def test_matches_naive_random_at_fp32_bar(ukan):
    """test_layers.py:225-234 restated: the (patched) matrix form against the reference's naive
    full-grid layer on 30 random shapes."""
    from paper_2408_11200_b200 import compat
    T = ukan.tensor
    rng = np.random.default_rng(4)
    compat.install(ukan)
    try:
        for _ in range(30):
            k = int(rng.integers(0, 6))
            G = int(rng.integers(1, 24))
            d_in, d_out = int(rng.integers(1, 5)), int(rng.integers(1, 5))
            layer = ukan.init_layer("kan", d_in, d_out, k, rng=rng, g_min=-2, g_max=2, G=G)
            _round_params(layer)
            x = T.as_tensor(_f32(rng.uniform(-3, 3, (6, d_in))))
            a = ukan.layers.kan_forward(layer, x).values
            b = ukan.naive_kan_forward(layer, x).values
            assert_close(a, b, what=f"k={k} G={G}")
    finally:
        compat.uninstall()


def test_reference_errors_and_index_rules(ukan):
    from paper_2408_11200_b200 import compat
    T = ukan.tensor
    compat.install(ukan)
    try:
        kl = ukan.init_layer("kan", 3, 2, 3, seed=0, G=5)
        with pytest.raises(ukan.errors.DimensionError):
            ukan.kan_forward(kl, T.as_tensor(np.zeros((2, 4))))
        ul = ukan.init_layer("ukan", 2, 2, 3, seed=0)
        with pytest.raises(ukan.errors.DomainError):
            ukan.ukan_forward(ul, T.as_tensor([[np.inf, 0.0]]))
        # clamp rule (test_layers.py:218-223): far outside == just inside, bitwise on the kernels
        layer = ukan.init_layer("kan", 2, 2, 3, seed=1, g_min=-1, g_max=1, G=8)
        _round_params(layer)
        inside = ukan.kan_forward(layer, T.as_tensor([[1.0 - 1e-12, -1.0]])).values
        beyond = ukan.kan_forward(layer, T.as_tensor([[50.0, -77.0]])).values
        np.testing.assert_array_equal(beyond, inside)
    finally:
        compat.uninstall()


def test_reference_model_and_train_loop_run_on_the_kernels(ukan):
    """The reference's Model (2-layer stack) gradients through compat at the bar, then its own
    training loop (train.train, train.py:118-190) end to end with every layer call on the GPU."""
    from paper_2408_11200_b200 import compat
    T = ukan.tensor
    rng = np.random.default_rng(5)
    model = ukan.build_model("kan", [6, 9, 3], 3, seed=0, g_min=-1.0, g_max=1.0, G=7)
    for layer in model.layers:
        _round_params(layer)
    x = _f32(rng.uniform(-1, 1, (64, 6)))
    y = rng.integers(0, 3, 64)

    def grads():
        for p in model.parameters().values():
            p.grad = None
        loss = T.reduce_loss("softmax_cross_entropy", model(T.as_tensor(x)), y)
        T.backward(loss)
        return float(loss.values), {n: p.grad.copy() for n, p in model.parameters().items()}

    compat.uninstall()
    l0, g0 = grads()
    compat.install(ukan)
    calls = {"n": 0}
    orig = compat.kan_forward

    def counting(layer, xx):
        calls["n"] += 1
        return orig(layer, xx)

    ukan.layers.kan_forward = counting
    try:
        l1, g1 = grads()
        assert abs(l1 - l0) <= 1e-6 + 1e-5 * abs(l0)
        for n in g0:
            assert_close(g1[n], g0[n], what="model grad " + n)
        from ukan.config import RunConfig
        from ukan.train import train
        cfg = RunConfig(task="regression_II", model="kan", widths=[2, 5, 1], epochs=3, eval_every=1, seed=0)
        res = train(cfg)
        assert res.epochs_run == 3 and np.isfinite(res.final_train) and np.isfinite(res.final_val)
        assert calls["n"] >= 2 + 3 * 2, calls  # the stack above plus every training / eval forward
    finally:
        compat.uninstall()
