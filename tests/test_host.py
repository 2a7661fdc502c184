"""Host-side logic of the drop-in API (no GPU): init parity with the reference's draws,
exception types, window helpers, positional encoding, DP shard bounds."""
import numpy as np
import pytest

from conftest import load_golden

import paper_2408_11200_b200 as P
from paper_2408_11200_b200 import errors, layers
from paper_2408_11200_b200.train import shard_bounds


def test_exception_hierarchy_matches_reference():
    for cls in (errors.DimensionError, errors.DomainError, errors.ContractError, errors.ConfigError,
                errors.FormatError):
        assert issubclass(cls, errors.UkanError) and issubclass(cls, ValueError)


def test_init_matches_reference_draws():
    g = load_golden("kan_small")     # reference init_layer("kan", 3, 4, 3, seed=11, G=5) rounded to fp32
    layer = P.init_layer("kan", 3, 4, 3, seed=11, g_min=-1.0, g_max=1.0, G=5, device="cpu")
    np.testing.assert_array_equal(layer.coeffs.detach().numpy(), g["coeffs"].astype(np.float32))
    np.testing.assert_array_equal(layer.scale.detach().numpy(), g["scale"].astype(np.float32))
    u = load_golden("ukan_small")
    ul = P.init_layer("ukan", 3, 2, 3, seed=31, delta_g=0.8, d_pe=8, d_femb=8, device="cpu")
    for n, p in ul.parameters().items():
        np.testing.assert_array_equal(p.detach().numpy(), u[n].astype(np.float32), err_msg=n)


def test_build_model_shared_rng_and_names():
    m = P.build_model("kan", [2, 4, 3], seed=0, device="cpu")
    assert list(m.parameters()) == ["layer0.coeffs", "layer0.scale", "layer1.coeffs", "layer1.scale"]
    m2 = P.build_model("ukan", [2, 4, 3], seed=0, device="cpu")
    assert list(m2.parameters())[:6] == ["layer0.feature_embedding", "layer0.cg_w1", "layer0.cg_b1",
                                         "layer0.cg_w2", "layer0.cg_b2", "layer0.scale"]


def test_config_errors():
    with pytest.raises(errors.ConfigError):
        P.init_layer("kan", 0, 3, 3, seed=0, device="cpu")
    with pytest.raises(errors.ConfigError):
        P.init_layer("nope", 2, 3, 3, seed=0, device="cpu")
    with pytest.raises(errors.ConfigError):
        P.init_layer("kan", 2, 3, 3, seed=0, g_min=1.0, g_max=-1.0, device="cpu")
    with pytest.raises(errors.ConfigError):
        P.init_layer("ukan", 2, 3, 3, seed=0, d_pe=5, device="cpu")
    with pytest.raises(errors.ConfigError):
        P.init_layer("ukan", 2, 3, 3, seed=0, delta_g=0.0, device="cpu")
    with pytest.raises(errors.ConfigError):
        P.build_model("kan", [3], device="cpu")


def test_select_window_cases():      # test_layers.py:37-57
    prev, nxt = np.arange(4.0), np.arange(10.0, 14.0)
    np.testing.assert_array_equal(P.select_window(prev, nxt, 5, 4), [1, 2, 3, 10])
    np.testing.assert_array_equal(P.select_window(prev, nxt, 8, 4), prev)
    np.testing.assert_array_equal(P.select_window(prev, nxt, -1, 4), [3, 10, 11, 12])


def test_positional_encoding_values():   # test_layers.py:14-33
    np.testing.assert_array_equal(P.positional_encoding(0, 8).numpy(), [0, 1, 0, 1, 0, 1, 0, 1])
    pe = P.positional_encoding(1, 4).numpy()
    np.testing.assert_allclose(pe, [np.sin(1), np.cos(1), np.sin(0.01), np.cos(0.01)], rtol=1e-12)
    for g in (1, 5, 123):
        a, b = P.positional_encoding(g, 8).numpy(), P.positional_encoding(-g, 8).numpy()
        np.testing.assert_allclose(b[0::2], -a[0::2], rtol=1e-15)
        np.testing.assert_allclose(b[1::2], a[1::2], rtol=1e-15)
    with pytest.raises(errors.ConfigError):
        P.positional_encoding(0, 5)


def test_basis_matrix_api():
    bm = P.basis_matrix(3)
    assert bm.K == 4 and bm.rational[0][1] == 4 * bm.rational[0][0]
    with pytest.raises(errors.DomainError):
        P.basis_matrix(11)


@pytest.mark.parametrize("n,world", [(10, 3), (8192, 8), (7, 2), (0, 4), (3, 4)])
def test_shard_bounds_partition(n, world):
    spans = [shard_bounds(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and b >= a
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_lr_schedule():
    s = P.LrSchedule(1e-2, 0.5, 1e-3)
    assert P.lr_at(s, 0) == 1e-2 and P.lr_at(s, 1) == 5e-3 and P.lr_at(s, 10) == 1e-3
    with pytest.raises(errors.ContractError):
        P.LrSchedule(1e-2, 0.0)
