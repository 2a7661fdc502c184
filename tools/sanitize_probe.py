"""Small invocations of every async-proxy kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): the TMEM forward (G <= 37 five-deep ring and G = 64 three-deep ring),
the FP64 DMMA table-gradient sweep and dx kernels, the feature-sliced backward, and a UKAN layer
(key build, tcgen05 table GEMM, fp64 CG GEMMs, sorted table-gradient sweep, dx).
python tools/sanitize_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11200_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
for (B, d_in, d_out, G) in ((600, 12, 256, 32), (300, 8, 256, 64)):
    layer = P.init_layer("kan", d_in, d_out, 3, seed=0, G=G, device=dev)
    x = (torch.rand((B, d_in), device=dev, generator=g) * 2.4 - 1.2).requires_grad_(True)
    gy = torch.randn((B, d_out), device=dev, generator=g)
    y = P.kan_forward(layer, x)
    torch.autograd.grad(y, [x, layer.coeffs, layer.scale], gy)
    tr = P.LayerTrainer(layer, 1e-3, buckets=3)
    tr.step(x.detach(), gy)
ul = P.init_layer("ukan", 16, 64, 3, seed=1, delta_g=0.5, d_pe=8, d_femb=8, device=dev)
xu = (torch.randn((256, 16), device=dev, generator=g) * 10).requires_grad_(True)
yu = P.ukan_forward(ul, xu)
torch.autograd.grad(yu, [xu] + list(ul.parameters().values()), torch.randn_like(yu))
torch.cuda.synchronize()
print("sanitize probe done")
