"""Per-kernel timing of the KAN layer C-ABI calls (profiling tool, not the bench).

python tools/kbench.py B d_in d_out G k [dx]   -> JSON {fwd_ms, bwd_ms, fwd_tflops, bwd_tflops}
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_11200_b200 import _lib  # noqa: E402
from paper_2408_11200_b200._lib import ptr, stream_ptr  # noqa: E402


def main():
    B, d_in, d_out, G, k = (int(a) for a in sys.argv[1:6])
    want_dx = len(sys.argv) > 6 and sys.argv[6] == "dx"
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    R = G + k
    x = torch.rand((B, d_in), device=dev, generator=g) * 2 - 1
    C = torch.randn((d_in, R, d_out), device=dev, generator=g) * 0.01
    sc = torch.ones((d_in, d_out), device=dev)
    y = torch.empty((B, d_out), device=dev)
    gy = torch.randn((B, d_out), device=dev, generator=g)
    dx = torch.empty_like(x) if want_dx else None
    dC = torch.empty_like(C)
    ds = torch.empty_like(sc)
    err = torch.zeros(1, device=dev, dtype=torch.int32)
    nb = lib.ukan_kan_backward_workspace_size(B, d_in, d_out, G, k)
    ws = torch.empty(max(nb, 8), device=dev, dtype=torch.uint8)
    flush = torch.empty(64 << 20, device=dev, dtype=torch.float32)

    nf = lib.ukan_kan_forward_workspace_size(B, d_in, d_out, G, k)
    wsf = torch.empty(max(nf, 8), device=dev, dtype=torch.uint8)

    def fwd():
        assert lib.ukan_kan_forward_ws(ptr(x), ptr(C), ptr(sc), None, ptr(y), B, d_in, d_out, G, k, -1.0, 1.0,
                                       ptr(err), ptr(wsf), nf, stream_ptr()) == 0

    def bwd():
        assert lib.ukan_kan_backward_ws(ptr(x), ptr(C), ptr(sc), None, ptr(gy), ptr(dx), ptr(dC), ptr(ds), None,
                                        B, d_in, d_out, G, k, -1.0, 1.0, ptr(ws), nb, stream_ptr()) == 0

    out = {"shape": [B, d_in, d_out, G, k], "dx": want_dx, "env": {k_: v for k_, v in os.environ.items() if k_.startswith("UKAN")}}
    for name, fn in (("fwd", fwd), ("bwd", bwd)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        ms = ts[len(ts) // 2]
        fl = 2.0 * (k + 1) * B * d_in * d_out * (2 if (name == "bwd" and want_dx) else 1)
        out[name + "_ms"] = ms
        out[name + "_tflops"] = fl / ms / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
