"""The memory-bounded oracle forms used for parity at the benchmarked shapes
(oracle.kan_rows / oracle.kan_feature_grads) equal the full restatement (which is pinned to the
reference's golden vectors in test_oracle_golden.py) on every row and feature.  CPU only."""
import numpy as np

import oracle


def test_rows_and_features_equal_full_oracle():
    rng = np.random.default_rng(0)
    B, f, o, G, k = 400, 7, 9, 13, 3
    x = rng.uniform(-1.3, 1.3, (B, f))
    C = rng.normal(size=(f, G + k, o))
    s = rng.uniform(0.5, 1.5, (f, o))
    g = rng.normal(size=(B, o))
    kw = dict(k=k, g_min=-1.0, g_max=1.0, G=G)
    full = oracle.kan_forward_backward(x, C, s, g, **kw)
    rows = [0, 5, 399]
    r = oracle.kan_rows(x[rows], C, s, g[rows], feat_block=3, **kw)
    np.testing.assert_array_equal(r["cell"], full["cell"][rows])
    np.testing.assert_allclose(r["y"], full["y"][rows], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(r["dx"], full["dx"][rows], rtol=1e-13, atol=1e-13)
    for i in range(f):
        q = oracle.kan_feature_grads(x[:, i], C[i], s[i], g, **kw)
        np.testing.assert_allclose(q["dcoeffs"], full["dcoeffs"][i], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(q["dscale"], full["dscale"][i], rtol=1e-12, atol=1e-12)


def test_other_degrees():
    rng = np.random.default_rng(1)
    for k in (0, 1, 2, 5):
        B, f, o, G = 120, 3, 4, 6
        x = rng.uniform(-1.2, 1.2, (B, f))
        C = rng.normal(size=(f, G + k, o))
        s = np.ones((f, o))
        g = rng.normal(size=(B, o))
        kw = dict(k=k, g_min=-1.0, g_max=1.0, G=G)
        full = oracle.kan_forward_backward(x, C, s, g, **kw)
        r = oracle.kan_rows(x, C, s, g, **kw)
        np.testing.assert_allclose(r["dx"], full["dx"], rtol=1e-12, atol=1e-12)
        q = oracle.kan_feature_grads(x[:, 1], C[1], s[1], g, **kw)
        np.testing.assert_allclose(q["dcoeffs"], full["dcoeffs"][1], rtol=1e-12, atol=1e-12)
