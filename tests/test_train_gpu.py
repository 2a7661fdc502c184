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
