"""UKAN layer fwd+bwd timing through the drop-in API (profiling tool, not the bench).

python tools/ukbench.py B d_in d_out delta_g d_pe d_femb [x_std]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11200_b200 as P  # noqa: E402


def main():
    B, d_in, d_out = (int(a) for a in sys.argv[1:4])
    dg = float(sys.argv[4])
    d_pe, d_femb = int(sys.argv[5]), int(sys.argv[6])
    std = float(sys.argv[7]) if len(sys.argv) > 7 else 20.0
    dev = torch.device("cuda", 0)
    layer = P.init_layer("ukan", d_in, d_out, 3, seed=0, delta_g=dg, d_pe=d_pe, d_femb=d_femb, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    x = (torch.randn((B, d_in), device=dev, generator=g) * std).requires_grad_(True)
    gy = torch.randn((B, d_out), device=dev, generator=g)
    params = list(layer.parameters().values())

    def step():
        y = P.ukan_forward(layer, x)
        grads = torch.autograd.grad(y, [x] + params, gy)
        return grads

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    keys = P.ops.ukan_build_keys(x.detach(), 3, dg)
    print(json.dumps({"shape": [B, d_in, d_out], "delta_g": dg, "d_pe": d_pe, "d_femb": d_femb, "x_std": std,
                      "n_u": keys.n_u, "ms": ts[len(ts) // 2],
                      "samples_per_s": B / (ts[len(ts) // 2] * 1e-3)}))


if __name__ == "__main__":
    main()
