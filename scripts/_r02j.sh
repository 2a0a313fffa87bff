timeout 300 python -m pytest tests/test_bb_gpu.py -x -q > gpurun_out/bb_tests.log 2>&1; echo bbtests=$?
timeout 200 python scripts/bb_sweep.py 124 160 248 > gpurun_out/sweep.log 2>&1
timeout 120 python scripts/bb_times.py > gpurun_out/times133.log 2>&1
