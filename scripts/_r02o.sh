timeout 600 python -m pytest tests/test_bench_multirank_gpu.py -x -q > gpurun_out/multirank.log 2>&1; echo multirank=$?
timeout 300 python bench.py --emulate-bands 8 --steps 10 --warmup 3 > gpurun_out/emul8.log 2>&1; echo emul=$?
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
