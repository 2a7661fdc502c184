"""Rows per feature of the UKAN virtual tables of the cfg5 stack (and the cfg4 layer):
python tools/ukan_density.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11200_b200 as P  # noqa: E402
from paper_2408_11200_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
model = P.build_model("ukan", [64, 512, 512, 64], 3, seed=0, device=dev, delta_g=0.4, d_pe=24, d_femb=24)
g = torch.Generator(device=dev)
g.manual_seed(5)
h = torch.randn((65536, 64), device=dev, generator=g)
with torch.no_grad():
    for li, L in enumerate(model.layers):
        keys = ops.ukan_build_keys(h, L.k, float(L.delta_g))
        ss = keys.seg_start.long()
        rows = (ss[1:] - ss[:-1]) * (L.k + 1)
        print(f"cfg5 layer {li}: d_in {L.d_in} n_u {keys.n_u} rows/feature max {int(rows.max())} mean {float(rows.float().mean()):.1f} "
              f"h std {float(h.std()):.3f} absmax {float(h.abs().max()):.2f}")
        h = P.ukan_forward(L, h)
L = P.init_layer("ukan", 1024, 1024, 3, seed=0, delta_g=0.5, d_pe=32, d_femb=32, device=dev)
x = torch.randn((4096, 1024), device=dev, generator=g) * 20
keys = ops.ukan_build_keys(x, 3, 0.5)
ss = keys.seg_start.long()
rows = (ss[1:] - ss[:-1]) * 4
print(f"cfg4-shaped: n_u {keys.n_u} rows/feature max {int(rows.max())} mean {float(rows.float().mean()):.1f}")
