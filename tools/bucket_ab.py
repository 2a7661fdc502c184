"""LayerTrainer step time at cfg3 by bucket count: python tools/bucket_ab.py BUCKETS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11200_b200 as P  # noqa: E402

nb = int(sys.argv[1])
dev = torch.device("cuda", 0)
layer = P.init_layer("kan", 4096, 4096, 3, seed=0, g_min=-1.0, g_max=1.0, G=64, device=dev)
tr = P.LayerTrainer(layer, 1e-3, buckets=nb)
g = torch.Generator(device=dev)
g.manual_seed(1)
x = torch.rand((65536, 4096), device=dev, generator=g) * 2 - 1
gy = torch.randn((65536, 4096), device=dev, generator=g) / 65536
for _ in range(2):
    tr.step(x, gy)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    tr.step(x, gy)
b.record()
torch.cuda.synchronize()
print({"buckets": nb, "ms_per_step": a.elapsed_time(b) / 3})
