"""cfg5 (UKAN [64,512,512,64], delta_g 0.4, d_pe = d_femb = 24, B = 65536) training steps for a
launch list: python tools/cfg5_probe.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11200_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
model = P.build_model("ukan", [64, 512, 512, 64], 3, seed=0, device=dev, delta_g=0.4, d_pe=24, d_femb=24)
tr = P.SplineTrainer(model, "mse", 1e-3, "adam")
g = torch.Generator(device=dev)
g.manual_seed(5)
x = torch.randn((65536, 64), device=dev, generator=g)
t = torch.randn((65536, 64), device=dev, generator=g)
tr.read_loss(tr.step(x, t))
for _ in range(steps):
    loss = tr.step(x, t)
print(tr.read_loss(loss), [L.d_in for L in model.layers])
