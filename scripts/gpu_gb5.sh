timeout 180 python -m pytest tests/test_gb_gpu.py -x -q > gpurun_out/gb_pytest.log 2>&1; echo pytest_gb=$?
for r in 1 2; do for sw in 0 1; do DTB_GB_SWAP=$sw timeout 100 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('swap=$sw', d['kernel_ms'], d['roofline']['frac'])"; done; done
DTB_GB_SWAP=1 timeout 180 python -m pytest tests/test_gb_gpu.py -x -q > gpurun_out/gb_pytest_swap.log 2>&1; echo pytest_gb_swap=$?
