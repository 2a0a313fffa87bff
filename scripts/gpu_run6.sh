timeout 900 python -m pytest tests/test_fast_path_gpu.py tests/test_parity_gpu.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'], d['roofline']['frac'])"
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['kernel_ms'], d['roofline']['frac'])"
bash scripts/gpu_prof.sh
