"""cfg3 single KAN layer (4096->4096, G=64, B=65536) fwd + parameter grads — profiling tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_11200_b200 as P
dev = torch.device("cuda", 0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
layer = P.init_layer("kan", 4096, 4096, 3, seed=0, g_min=-1.0, g_max=1.0, G=64, device=dev)
x = torch.rand((B, 4096), device=dev) * 2 - 1
gy = torch.randn((B, 4096), device=dev)
for _ in range(2):
    torch.autograd.grad(P.kan_forward(layer, x), [layer.coeffs, layer.scale], gy)
torch.cuda.synchronize()
