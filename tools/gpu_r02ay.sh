#!/bin/bash
# sample-blocked pair order in spline_dx64: bitwise A/B vs the previous build + cfg4 timings
O=gpurun_out/ay; mkdir -p $O
cat > $O/dx_ab.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2408_11200_b200 as P
dev = torch.device("cuda", 0)
B = int(sys.argv[2])
layer = P.init_layer("ukan", 64, 256, 3, seed=0, delta_g=0.5, d_pe=8, d_femb=8, device=dev)
g = torch.Generator(device=dev); g.manual_seed(3)
x = (torch.randn((B, 64), device=dev, generator=g) * 20).requires_grad_(True)
gy = torch.randn((B, 256), device=dev, generator=g)
y = P.ukan_forward(layer, x)
dx, = torch.autograd.grad(y, [x], gy)
np.save(sys.argv[1], dx.cpu().numpy())
PY
for Bv in 5000 9000; do
  UKAN_B200_LIB=abtmp/lib_pre.so timeout 300 python $O/dx_ab.py $O/old_$Bv.npy $Bv > $O/e1.txt 2>&1
  timeout 300 python $O/dx_ab.py $O/new_$Bv.npy $Bv > $O/e2.txt 2>&1
  python -c "
import numpy as np
a=np.load('$O/old_$Bv.npy'); b=np.load('$O/new_$Bv.npy'); print('B=$Bv dx bitwise', np.array_equal(a,b))"
done
tail -2 $O/e1.txt $O/e2.txt
rm -f $O/*.npy
timeout 900 python -c "
import bench, torch, json; r = bench.cfg4_rate(torch.device('cuda', 0)); print(json.dumps({'ms': r['ms_per_step'], 'sps': r['samples_per_s']}))" 2>&1 | tail -1
timeout 600 python tools/ukbench.py 4096 1024 1024 0.5 32 32 | cut -c1-200
timeout 900 python -m pytest tests/test_parity_ukan.py -x -q -m gpu 2>&1 | tail -1
