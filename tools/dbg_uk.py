import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import test_parity_ukan as T
import oracle
for args in [(256, 64, 64, 3, 1.0, 8, 8), (64, 128, 128, 3, 0.5, 32, 32)]:
    layer, x, gup = T.random_case(*args, seed=1 if args[0] == 256 else 2, **({} if args[0] == 256 else dict(sigma=20.0, tails=0.001)))
    got = T.run(layer, x, gup)
    p = {n: t.detach().double().cpu().numpy() for n, t in layer.parameters().items()}
    want = oracle.ukan_forward_backward(x.astype(np.float64), p, gup.astype(np.float64), k=args[3], delta_g=args[4], d_pe=args[5])
    for key in got:
        g, w = np.asarray(got[key], np.float64), np.asarray(want[key], np.float64)
        err = np.abs(g - w); tol = 1e-6 + 1e-5 * np.abs(w)
        print(args[:3], key, "max ratio %.3g" % float((err / tol).max()), "max rel %.3g" % float((err / np.maximum(np.abs(w), 1e-30)).max()))
