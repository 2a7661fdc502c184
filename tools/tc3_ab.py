"""Bitwise A/B of the table-gradient sweep variants: python tools/tc3_ab.py OUT.npz [B d_in d_out G]
(run once with UKAN_TC3=0 and once without, then compare the two files)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_11200_b200 import _lib  # noqa: E402
from paper_2408_11200_b200._lib import check, ptr, stream_ptr  # noqa: E402

out = sys.argv[1]
B, d_in, d_out, G = (int(a) for a in (sys.argv[2:6] if len(sys.argv) > 5 else (5000, 70, 256, 64)))
lib = _lib.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(7)
x = torch.rand((B, d_in), device=dev, generator=g) * 2.2 - 1.1
C = torch.randn((d_in, G + 3, d_out), device=dev, generator=g)
sc = torch.rand((d_in, d_out), device=dev, generator=g) + 0.5
gy = torch.randn((B, d_out), device=dev, generator=g)
dC, ds = torch.empty_like(C), torch.empty_like(sc)
nb = lib.ukan_kan_backward_workspace_size(B, d_in, d_out, G, 3)
ws = torch.empty(nb, device=dev, dtype=torch.uint8)
check(lib.ukan_kan_backward_ws2(ptr(x), ptr(C), ptr(sc), None, ptr(gy), None, ptr(dC), ptr(ds), None, B, d_in, d_out, G,
                                3, -1.0, 1.0, ptr(ws), nb, 0, stream_ptr()), "ws2")
torch.cuda.synchronize()
np.savez(out, dC=dC.cpu().numpy(), ds=ds.cpu().numpy())
print("saved", out, float(dC.abs().sum()))
