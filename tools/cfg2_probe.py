"""cfg2 (KAN [784,256,10], G = 32, B = 8192, softmax-CE + Adam) captured training steps for a
launch list: python tools/cfg2_probe.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11200_b200 as P  # noqa: E402
from paper_2408_11200_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
model = P.build_model("kan", [784, 256, 10], 3, seed=0, device=dev, g_min=-1.0, g_max=1.0, G=32)
tr = P.SplineTrainer(model, "softmax_cross_entropy", 1e-3, "adam")
ops.set_check_mode("deferred")
g = torch.Generator(device=dev)
g.manual_seed(99)
x = torch.rand((8192, 784), device=dev, generator=g) * 2 - 1
y = torch.randint(0, 10, (8192,), device=dev, generator=g)
for _ in range(3):
    tr.step(x, y)
tr.read_loss(tr.step(x, y))
cap = tr.capture(x, y)
for _ in range(steps):
    loss = cap.replay(x, y)
tr.read_loss(loss)
print("ok")
