timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in c4 c3; do python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$c', d['kernel_ms'], d['roofline']['frac'])"; done
