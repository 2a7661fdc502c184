"""The DP training step on one GPU against the reference's own training step (golden:
train.py:142-150 semantics - loss, tape backward, Adam with coupled L2, two steps)."""
import numpy as np
import pytest
import torch

from conftest import assert_close, golden_names, load_golden

import paper_2408_11200_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", golden_names("step_"))
def test_two_steps_match_reference(name):
    g = load_golden(name)
    kind = str(g["kind"])
    widths = [int(w) for w in g["widths"]]
    k = int(g["k"])
    kw = {n[3:]: (float(v) if n[3:] != "G" and n[3:] not in ("d_pe", "d_femb") else int(v))
          for n, v in g.items() if n.startswith("kw_")}
    model = P.build_model(kind, widths, k, seed=0, **kw)
    with torch.no_grad():
        for n, p in model.parameters().items():
            p.copy_(torch.tensor(g["init." + n], dtype=torch.float32))
    loss_kind = str(g["loss_kind"])
    tr = P.SplineTrainer(model, loss_kind, float(g["lr"]), "adam", weight_decay=float(g["wd"]))
    x = torch.tensor(g["x"], dtype=torch.float32, device="cuda")
    if loss_kind == "softmax_cross_entropy":
        tgt = torch.tensor(g["target"], dtype=torch.int64, device="cuda")
    else:
        tgt = torch.tensor(g["target"], dtype=torch.float32, device="cuda")
    for s in range(int(g["steps"])):
        loss = tr.read_loss(tr.step(x, tgt))
        assert abs(loss - g["losses"][s]) <= 1e-6 + 1e-5 * abs(g["losses"][s])
        if s == 0:
            for n in model.parameters():
                assert_close(tr.flat.gviews[n].cpu().numpy(), g["grad0." + n], what="grad0." + n)
    for n in model.parameters():
        assert_close(tr.flat.views[n].cpu().numpy(), g["final." + n], what="final." + n)


def test_diverged_loss_skips_update_and_raises():
    model = P.build_model("kan", [3, 2], seed=0, G=4)
    tr = P.SplineTrainer(model, "mse", 1e-2)
    before = tr.flat.data.clone()
    x = torch.zeros((4, 3), device="cuda")
    tgt = torch.full((4, 2), float("inf"), device="cuda")
    with pytest.raises(P.DivergedError):
        tr.read_loss(tr.step(x, tgt))
    assert torch.equal(before, tr.flat.data)


def test_device_prefetcher_yields_every_batch():
    """Each batch arrives intact on the device (checked at its iteration: buffers are reused)."""
    host = [(torch.full((64, 3), float(i)).pin_memory(), torch.arange(64) + i) for i in range(5)]
    n = 0
    for i, (x, y) in enumerate(P.DevicePrefetcher(iter(host), "cuda")):
        assert x.is_cuda and y.is_cuda
        assert torch.equal(x.cpu(), host[i][0]) and torch.equal(y.cpu(), host[i][1])
        torch.cuda._sleep(1000000)  # a slow consumer must not see the next copy land early
        assert torch.equal(x.cpu(), host[i][0])
        n += 1
    assert n == 5


def test_capture_rejects_ukan():
    model = P.build_model("ukan", [3, 2], 3, seed=1, delta_g=0.5, d_pe=8, d_femb=8)
    tr = P.SplineTrainer(model, "mse", 1e-2)
    x = torch.zeros((4, 3), device="cuda")
    with pytest.raises(P.ConfigError):
        tr.capture(x, torch.zeros((4, 2), device="cuda"))


@pytest.mark.parametrize("kind", ["kan"])
def test_captured_step_matches_eager(kind):
    """CapturedStep (the step as one CUDA graph, device-side Adam counter) reproduces eager steps."""
    kw = dict(G=8) if kind == "kan" else dict(delta_g=0.5, d_pe=8, d_femb=8)
    rng = np.random.default_rng(3)
    xs = [torch.tensor(rng.uniform(-1, 1, (64, 6)), dtype=torch.float32, device="cuda") for _ in range(4)]
    ys = [torch.tensor(rng.integers(0, 3, 64), device="cuda") for _ in range(4)]
    runs = []
    for use_graph in (False, True):
        model = P.build_model(kind, [6, 7, 3], 3, seed=5, **kw)
        tr = P.SplineTrainer(model, "softmax_cross_entropy", 1e-2, "adam", weight_decay=1e-5)
        losses = [tr.read_loss(tr.step(xs[0], ys[0]))]
        if use_graph:
            cap = tr.capture(xs[0], ys[0])
            losses += [tr.read_loss(cap.replay(xs[s], ys[s])) for s in range(1, 4)]
            assert cap.sync_step_count() == 4
        else:
            losses += [tr.read_loss(tr.step(xs[s], ys[s])) for s in range(1, 4)]
        runs.append((losses, {n: p.detach().cpu().numpy().copy() for n, p in model.parameters().items()}))
    (la, pa), (lb, pb) = runs
    np.testing.assert_allclose(lb, la, rtol=1e-6)
    for n in pa:
        np.testing.assert_allclose(pb[n], pa[n], rtol=1e-5, atol=1e-7, err_msg=n)


def test_captured_step_learning_rate_change():
    """CapturedStep.set_lr changes the device-side rate the graph reads (the reference changes the
    rate per epoch, train.py:153)."""
    rng = np.random.default_rng(4)
    xs = [torch.tensor(rng.uniform(-1, 1, (32, 5)), dtype=torch.float32, device="cuda") for _ in range(3)]
    ys = [torch.tensor(rng.integers(0, 2, 32), device="cuda") for _ in range(3)]
    runs = []
    for use_graph in (False, True):
        model = P.build_model("kan", [5, 2], 3, seed=9, G=6)
        tr = P.SplineTrainer(model, "softmax_cross_entropy", 1e-2, "adam")
        tr.read_loss(tr.step(xs[0], ys[0]))
        if use_graph:
            cap = tr.capture(xs[0], ys[0])
            cap.set_lr(5e-3)
            tr.read_loss(cap.replay(xs[1], ys[1]))
            cap.set_lr(1e-3)
            tr.read_loss(cap.replay(xs[2], ys[2]))
        else:
            tr.read_loss(tr.step(xs[1], ys[1], lr=5e-3))
            tr.read_loss(tr.step(xs[2], ys[2], lr=1e-3))
        runs.append({n: p.detach().cpu().numpy().copy() for n, p in model.parameters().items()})
    for n in runs[0]:
        np.testing.assert_allclose(runs[1][n], runs[0][n], rtol=1e-5, atol=1e-7, err_msg=n)


def test_step_input_checks_like_the_reference():
    """SplineTrainer.step validates its inputs the way the reference's losses do (tensor.py:368-400):
    float64 / non-contiguous x are converted (same loss as fp32 x), a wrong width or label count is
    a DimensionError, a label outside [0, c) an IndexError at the host read, never an OOB read."""
    model = P.build_model("kan", [5, 7, 3], 3, seed=0, G=6)
    tr = P.SplineTrainer(model, "softmax_cross_entropy", 0.0, "sgd")
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (16, 5))
    y = rng.integers(0, 3, 16)
    l32 = tr.read_loss(tr.step(torch.tensor(x, dtype=torch.float32, device="cuda"), torch.tensor(y, device="cuda")))
    x64 = torch.tensor(x, dtype=torch.float64, device="cuda")
    l64 = tr.read_loss(tr.step(x64, torch.tensor(y, dtype=torch.int32, device="cuda")))
    assert l32 == l64
    xt = torch.tensor(x.T.copy(), dtype=torch.float32, device="cuda").T  # non-contiguous view
    assert tr.read_loss(tr.step(xt, torch.tensor(y, device="cuda"))) == l32
    with pytest.raises(P.DimensionError):
        tr.step(torch.zeros((16, 4), device="cuda"), torch.tensor(y, device="cuda"))
    with pytest.raises(P.DimensionError):
        tr.step(torch.tensor(x, dtype=torch.float32, device="cuda"), torch.tensor(y[:15], device="cuda"))
    bad = y.copy()
    bad[3] = 3
    with pytest.raises(IndexError):
        tr.read_loss(tr.step(torch.tensor(x, dtype=torch.float32, device="cuda"), torch.tensor(bad, device="cuda")))


def test_skipped_step_does_not_advance_adam_counter():
    """The reference raises DivergedError before adam_step bumps state.t (train.py:143-144)."""
    model = P.build_model("kan", [3, 2], seed=0, G=4)
    tr = P.SplineTrainer(model, "mse", 1e-2)
    x = torch.zeros((4, 3), device="cuda")
    ok = torch.zeros((4, 2), device="cuda")
    tr.read_loss(tr.step(x, ok))
    assert tr.t == 1
    with pytest.raises(P.DivergedError):
        tr.read_loss(tr.step(x, torch.full((4, 2), float("inf"), device="cuda")))
    assert tr.t == 1
    tr.read_loss(tr.step(x, ok))
    assert tr.t == 2
