set -x
timeout 120 python -m pytest tests/test_bb_gpu.py -x -q -k "c4_crop" > gpurun_out/bb_first.log 2>&1; echo first=$?
timeout 600 python -m pytest tests/test_bb_gpu.py -x -q > gpurun_out/bb_tests.log 2>&1; echo bbtests=$?
DTB_PRINT_PLAN=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_bb.log 2>&1; echo bench=$?
