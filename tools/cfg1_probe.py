"""cfg1 (KAN 64 -> 64, G = 10, B = 1024) as a captured training step: per-kernel launch list tool.
python tools/cfg1_probe.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11200_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = torch.Generator(device=dev)
g.manual_seed(3)
x = torch.rand((1024, 64), device=dev, generator=g) * 2 - 1
t = torch.randn((1024, 64), device=dev, generator=g)
model = P.build_model("kan", [64, 64], 3, seed=0, device=dev, g_min=-1.0, g_max=1.0, G=10)
tr = P.SplineTrainer(model, "mse", 1e-3, "adam")
for _ in range(3):
    tr.read_loss(tr.step(x, t))
cap = tr.capture(x, t)
for _ in range(steps):
    loss = cap.replay()
tr.read_loss(loss)
torch.cuda.synchronize()
print("ok")
