"""SplineTrainer.step with world size 2 (reference step: train.py:142-150): two
ranks over gloo sharing cuda:0 (this run has one GPU; the bench's N > 1 path is the same code
over NCCL), UNEVEN contiguous shards, n_global NOT passed (the trainer all-reduces the shard
sizes).  The summed gradients, the all-reduced loss and the Adam-updated parameters of rank 0
must equal a single-process step over the whole batch (rtol 1e-5 / atol 1e-6: the all-reduce
order changes fp32 rounding)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import assert_close

pytestmark = pytest.mark.gpu

CASES = {
    "kan": dict(widths=[16, 24, 5], kw=dict(g_min=-1.0, g_max=1.0, G=8), loss="softmax_cross_entropy"),
    "ukan": dict(widths=[6, 8, 3], kw=dict(delta_g=0.5, d_pe=8, d_femb=8), loss="mse"),
}
B = 37  # shards 19 + 18


def _data(kind):
    rng = np.random.default_rng(5)
    c = CASES[kind]
    x = (rng.uniform(-1.2, 1.2, (B, c["widths"][0])) if kind == "kan"
         else rng.normal(0, 3.0, (B, c["widths"][0]))).astype(np.float32)
    if c["loss"] == "mse":
        t = rng.normal(size=(B, c["widths"][-1])).astype(np.float32)
    else:
        t = rng.integers(0, c["widths"][-1], B)
    return x, t


def _run(kind, x, t, group_world=1, rank=0):
    import paper_2408_11200_b200 as P
    from paper_2408_11200_b200.train import shard_bounds
    c = CASES[kind]
    model = P.build_model(kind, c["widths"], 3, seed=0, device="cuda", **c["kw"])
    tr = P.SplineTrainer(model, c["loss"], 1e-2, "adam")
    lo, hi = shard_bounds(B, rank, group_world)
    xs = torch.tensor(x[lo:hi], device="cuda")
    ts = torch.tensor(t[lo:hi], device="cuda")
    loss = tr.read_loss(tr.step(xs, ts))
    return loss, tr.flat.grad.cpu().numpy().copy(), tr.flat.data.cpu().numpy().copy()


def _worker(rank, world, port, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, t = _data(kind)
        out = _run(kind, x, t, world, rank)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind", ["kan", "ukan"])
def test_two_ranks_uneven_shards_match_single_process(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, t = _data(kind)
    loss1, grad1, data1 = _run(kind, x, t)
    for r in (0, 1):
        loss2, grad2, data2 = res[r]
        assert abs(loss2 - loss1) <= 1e-6 + 1e-5 * abs(loss1)
        assert_close(grad2, grad1, what=f"rank{r} summed gradient")
        assert_close(data2, data1, what=f"rank{r} updated parameters")
    # both ranks hold identical replicas after the step
    np.testing.assert_array_equal(res[0][2], res[1][2])


def _layer_run(x, gy, world=1, rank=0, buckets=3, d_out=64):
    import paper_2408_11200_b200 as P
    from paper_2408_11200_b200.train import shard_bounds
    layer = P.init_layer("kan", 24, d_out, 3, seed=3, g_min=-1.0, g_max=1.0, G=16, device="cuda")
    tr = P.LayerTrainer(layer, 1e-2, buckets=buckets)
    lo, hi = shard_bounds(x.shape[0], rank, world)
    y, dx = tr.step(torch.tensor(x[lo:hi], device="cuda"), torch.tensor(gy[lo:hi], device="cuda"))
    torch.cuda.synchronize()
    return (y.cpu().numpy(), dx.cpu().numpy(), tr.flat.grad.cpu().numpy().copy(), tr.flat.data.cpu().numpy().copy())


def _layer_data(d_out=64):
    rng = np.random.default_rng(8)
    x = rng.uniform(-1.2, 1.2, (301, 24)).astype(np.float32)
    gy = (rng.normal(size=(301, d_out)) / 301).astype(np.float32)  # dL/dy of a global mean loss
    return x, gy


def _layer_worker(rank, world, port, q, d_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, gy = _layer_data(d_out)
        q.put((rank, _layer_run(x, gy, world, rank, d_out=d_out)))
    finally:
        dist.destroy_process_group()


# d_out 704: the bucketed ukan_kan_backward_part path; d_out 64 (d_in * d_out <= 2^14): the small-
# layer path (kan_small.cu) through ukan_kan_backward_ws2 and one all-reduce of the whole gradient.
LAYER_D_OUT = [704, 64]


@pytest.mark.parametrize("d_out", LAYER_D_OUT)
def test_layer_trainer_matches_autograd_and_oracle(d_out):
    """LayerTrainer (the bench's cfg3 unit: dx first, then the table gradient in feature buckets
    via ukan_kan_backward_part) against the oracle; bucketing changes no bit."""
    import oracle
    import paper_2408_11200_b200 as P
    from paper_2408_11200_b200 import _lib
    assert _lib.load().ukan_kan_backward_part_supported(301, 24, d_out, 16, 3) == (1 if d_out == 704 else 0)
    x, gy = _layer_data(d_out)
    y, dx, grad, _ = _layer_run(x, gy, buckets=3, d_out=d_out)
    layer = P.init_layer("kan", 24, d_out, 3, seed=3, g_min=-1.0, g_max=1.0, G=16, device="cuda")
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.kan_forward_backward(x.astype(np.float64), p["coeffs"], p["scale"], gy.astype(np.float64), k=3,
                                       g_min=-1.0, g_max=1.0, G=16)
    assert_close(y, want["y"], what="y")
    assert_close(dx, want["dx"], what="dx")
    nC = p["coeffs"].size
    assert_close(grad[:nC].reshape(p["coeffs"].shape), want["dcoeffs"], what="dcoeffs")
    assert_close(grad[nC:].reshape(p["scale"].shape), want["dscale"], what="dscale")
    _, _, grad1, _ = _layer_run(x, gy, buckets=1, d_out=d_out)
    np.testing.assert_array_equal(grad, grad1)  # bucketing does not change a bit


@pytest.mark.parametrize("d_out", LAYER_D_OUT)
def test_layer_trainer_two_ranks_match_single_process(d_out):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_layer_worker, args=(r, 2, port, q, d_out)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, gy = _layer_data(d_out)
    y1, dx1, grad1, data1 = _layer_run(x, gy, d_out=d_out)
    from paper_2408_11200_b200.train import shard_bounds
    for r in (0, 1):
        lo, hi = shard_bounds(x.shape[0], r, 2)
        y2, dx2, grad2, data2 = res[r]
        np.testing.assert_array_equal(y2, y1[lo:hi])  # forward / dx are per sample: bitwise
        np.testing.assert_array_equal(dx2, dx1[lo:hi])
        assert_close(grad2, grad1, what=f"rank{r} summed gradient")
    np.testing.assert_array_equal(res[0][3], res[1][3])
