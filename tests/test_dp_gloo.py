"""Data-parallel host logic on CPU with world_size 2 over gloo: contiguous batch shards
(shard_bounds), loss / gradients normalised by the GLOBAL batch, one all-reduce(sum) of the
flat gradient buffer in model.parameters() order (GradSync).  The per-shard gradients come
from the CPU oracle (the GPU kernels are covered by the -m gpu tests); the reduced result must
equal the single-process full-batch gradient."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2408_11200_b200.train import GradSync, shard_bounds

WIDTHS = [5, 6, 3]
CFG = dict(k=3, g_min=-1.0, g_max=1.0, G=6)


def _problem():
    rng = np.random.default_rng(0)
    params = []
    for i in range(len(WIDTHS) - 1):
        params.append({"coeffs": rng.normal(0, 0.3, (WIDTHS[i], CFG["G"] + CFG["k"], WIDTHS[i + 1])),
                       "scale": rng.uniform(0.5, 1.5, (WIDTHS[i], WIDTHS[i + 1]))})
    x = rng.uniform(-1.2, 1.2, (37, WIDTHS[0]))
    y = rng.integers(0, WIDTHS[-1], 37)
    return params, x, y


def _shard_grads(params, x, y, n_global):
    """fwd + CE (sum over the shard / n_global) + bwd, flattened in parameters() order."""
    hs = [x]
    for lp in params:
        hs.append(oracle.kan_forward_backward(hs[-1], lp["coeffs"], lp["scale"], None, **CFG)["y"])
    loss_mean, g = oracle.softmax_xent(hs[-1], y)
    n = x.shape[0]
    loss = loss_mean * n / n_global
    g = g * n / n_global
    flat = [None] * len(params)
    for li in range(len(params) - 1, -1, -1):
        r = oracle.kan_forward_backward(hs[li], params[li]["coeffs"], params[li]["scale"], g, need_dx=li > 0, **CFG)
        flat[li] = [r["dcoeffs"].ravel(), r["dscale"].ravel()]
        g = r.get("dx")
    return loss, np.concatenate([a for pair in flat for a in pair])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params, x, y = _problem()
        lo, hi = shard_bounds(x.shape[0], rank, world)
        loss, grad = _shard_grads(params, x[lo:hi], y[lo:hi], x.shape[0])
        sync = GradSync()
        assert sync.enabled and sync.world == world and sync.rank == rank
        buf = torch.tensor(np.concatenate([[loss], grad]))
        sync.allreduce_async(buf[:1])
        sync.allreduce_async(buf[1:])
        sync.wait()
        if rank == 0:
            q.put(buf.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_allreduce_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    params, x, y = _problem()
    loss, grad = _shard_grads(params, x, y, x.shape[0])
    np.testing.assert_allclose(got[0], loss, rtol=1e-12)
    np.testing.assert_allclose(got[1:], grad, rtol=1e-10, atol=1e-14)


def test_grad_sync_is_noop_without_group():
    s = GradSync()
    t = torch.ones(3)
    s.allreduce_async(t)
    s.wait()
    assert not s.enabled and s.world == 1 and torch.equal(t, torch.ones(3))
