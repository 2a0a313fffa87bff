timeout 180 python -m pytest tests/test_gb_gpu.py -x -q > gpurun_out/gb_pytest.log 2>&1; echo pytest_gb=$?; tail -1 gpurun_out/gb_pytest.log
timeout 600 python scripts/config_table.py --reps 10 > gpurun_out/config_table_gb.json 2> gpurun_out/config_table_gb.err; echo table=$?
for r in 1 2; do timeout 100 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'], d['roofline']['frac'])"; done
