"""Small invocations of every async-proxy kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): the TMEM forward (G <= 37 five-deep ring and G = 64 three-deep ring),
the FP64 DMMA table-gradient sweeps (tc3: tensor-map TMA + mbarrier ring) and dx kernels, the
feature-sliced backward, a UKAN layer (key build, pre-split bulk-copy tcgen05 table GEMM, fp64 CG
GEMMs, sorted table-gradient sweep, dx), dense UKAN layers (per-feature segments on the DMMA
sweep, block-split and sample-split, and the DMMA dx), and the small-layer kernels (cluster +
distributed-shared-memory table gradient).
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
for sigma, dg in ((1.0, 0.4), (0.3, 0.4)):  # dense UKAN: ~28-row segments (tc3) and <= 12 rows (sample split)
    ud = P.init_layer("ukan", 12, 64, 3, seed=2, delta_g=dg, d_pe=8, d_femb=8, device=dev)
    xd = (torch.randn((700, 12), device=dev, generator=g) * sigma).requires_grad_(True)
    yd = P.ukan_forward(ud, xd)
    torch.autograd.grad(yd, [xd] + list(ud.parameters().values()), torch.randn_like(yd))
small = P.build_model("kan", [64, 64], 3, seed=0, device=dev, g_min=-1.0, g_max=1.0, G=10)  # cfg1 small path
trs = P.SplineTrainer(small, "mse", 1e-3, "adam")
xs = torch.rand((1024, 64), device=dev, generator=g) * 2 - 1
trs.read_loss(trs.step(xs, torch.randn((1024, 64), device=dev, generator=g)))
torch.cuda.synchronize()
print("sanitize probe done")
