# gb_kernel first check: parity tests, then C4 kernel time gb vs ws
timeout 600 python -m pytest tests/test_gb_gpu.py -x -q > gpurun_out/gb_pytest.log 2>&1; echo pytest_gb=$?
tail -5 gpurun_out/gb_pytest.log
for m in 2 0; do DTB_GB=$m DTB_PRINT_PLAN=1 timeout 300 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>gpurun_out/gb_plan_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('DTB_GB=$m', d['kernel_ms'], d['roofline']['frac'])"; tail -2 gpurun_out/gb_plan_$m.log; done
