timeout 180 python -m pytest tests/test_gb_gpu.py -x -q > gpurun_out/gb_pytest.log 2>&1; echo pytest_gb=$?
for bs in 1 1.5 2 2.5 3; do DTB_BAND_SCALE=$bs timeout 100 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bs=$bs', d['kernel_ms'], d['roofline']['frac'])"; done
