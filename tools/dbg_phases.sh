for d in 0 1 2 3; do echo "UKAN_DBG=$d"; UKAN_DBG=$d python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernel_ms'])"; done
UKAN_NO_DMMA=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nodmma', d['kernel_ms'])"
