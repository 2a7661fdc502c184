"""Forward A/B between two builds of the library: python tools/fwd_ab.py OUT.npy B d_in d_out G
(UKAN_B200_LIB selects the build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_11200_b200 import _lib  # noqa: E402
from paper_2408_11200_b200._lib import check, ptr, stream_ptr  # noqa: E402

out = sys.argv[1]
if sys.argv[2] == "ukan":  # UKAN layer forward: python tools/fwd_ab.py OUT.npy ukan B d_in d_out
    import paper_2408_11200_b200 as P
    B, d_in, d_out = (int(a) for a in sys.argv[3:6])
    dev = torch.device("cuda", 0)
    layer = P.init_layer("ukan", d_in, d_out, 3, seed=0, delta_g=0.5, d_pe=32, d_femb=32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    x = torch.randn((B, d_in), device=dev, generator=g) * 20
    with torch.no_grad():
        y = P.ukan_forward(layer, x)
    np.save(out, y.cpu().numpy())
    print("saved", out)
    sys.exit(0)
B, d_in, d_out, G = (int(a) for a in sys.argv[2:6])
lib = _lib.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(11)
x = torch.rand((B, d_in), device=dev, generator=g) * 2.2 - 1.1
C = torch.randn((d_in, G + 3, d_out), device=dev, generator=g)
sc = torch.rand((d_in, d_out), device=dev, generator=g) + 0.5
y = torch.empty((B, d_out), device=dev)
nb = lib.ukan_kan_forward_workspace_size(B, d_in, d_out, G, 3)
ws = torch.empty(max(nb, 8), device=dev, dtype=torch.uint8)
err = torch.zeros(1, device=dev, dtype=torch.int32)
check(lib.ukan_kan_forward_ws(ptr(x), ptr(C), ptr(sc), None, ptr(y), B, d_in, d_out, G, 3, -1.0, 1.0, ptr(err), ptr(ws),
                              nb, stream_ptr()), "fwd")
torch.cuda.synchronize()
np.save(out, y.cpu().numpy())
print("saved", out)
