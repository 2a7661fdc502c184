"""The naive comparison arm (naive_kan_forward, layers.py:321-370) on the GPU: same contract as
kan_forward (test_layers.py:225-234 checks the reference's two arms agree), parameter gradients
against the pinned oracle, and the CSV benchmark's schema (bench.py:15-96)."""
import numpy as np
import pytest
import torch

from conftest import assert_close

import oracle
import paper_2408_11200_b200 as P
from paper_2408_11200_b200 import bench_arms

pytestmark = pytest.mark.gpu


def test_matches_matrix_arm_random():
    rng = np.random.default_rng(0)
    for _ in range(40):
        k = int(rng.integers(0, 6))
        G = int(rng.integers(1, 24))
        d_in, d_out = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        layer = P.init_layer("kan", d_in, d_out, k, rng=rng, g_min=-2, g_max=2, G=G)
        x = torch.tensor(rng.uniform(-3, 3, (6, d_in)), dtype=torch.float32, device="cuda")
        a = P.kan_forward(layer, x).detach().double().cpu().numpy()
        b = P.naive_kan_forward(layer, x).detach().double().cpu().numpy()
        assert_close(b, a, what=f"k={k} G={G}")


@pytest.mark.parametrize("G,k", [(10, 3), (64, 2), (300, 3)])
def test_parameter_gradients_vs_oracle(G, k):
    rng = np.random.default_rng(G)
    B, d_in, d_out = 128, 7, 5
    layer = P.init_layer("kan", d_in, d_out, k, seed=G, g_min=-1.0, g_max=1.0, G=G)
    x = rng.uniform(-1.1, 1.1, (B, d_in)).astype(np.float32)
    gup = rng.normal(size=(B, d_out)).astype(np.float32)
    y = P.naive_kan_forward(layer, torch.tensor(x, device="cuda"))
    (y * torch.tensor(gup, device="cuda")).sum().backward()
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.kan_forward_backward(x.astype(np.float64), p["coeffs"], p["scale"], gup.astype(np.float64), k=k,
                                       g_min=-1.0, g_max=1.0, G=G)
    assert_close(y.detach().cpu().numpy(), want["y"], what="y")
    assert_close(layer.coeffs.grad.cpu().numpy(), want["dcoeffs"], what="dcoeffs")
    assert_close(layer.scale.grad.cpu().numpy(), want["dscale"], what="dscale")


def test_bench_csv_schema():
    rows = bench_arms.run_bench([3], [16, 64], batch=256, reps=2)
    assert [r.impl for r in rows] == ["matrix", "naive", "matrix", "naive"]
    for r in rows:
        fields = r.csv().split(",")
        assert len(fields) == len(bench_arms.BENCH_HEADER.split(","))
        assert r.total_s > 0 and r.peak_mem_bytes >= 0
