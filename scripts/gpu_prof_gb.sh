# ncu full capture of gb_kernel on C4 (bench), plus the test file
timeout 600 python -m pytest tests/test_gb_gpu.py -x -q > gpurun_out/gb_pytest.log 2>&1; echo pytest_gb=$?
tail -3 gpurun_out/gb_pytest.log
python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gb_kernel -s 2 -c 1 -o gpurun_out/prof_gb python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
