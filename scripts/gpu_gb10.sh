timeout 300 python -m pytest tests/test_gb_gpu.py -x -q 2>&1 | tail -1
for st in 4; do for r in 1 2; do timeout 100 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['kernel_ms'], d['kernel'])"; done; done
