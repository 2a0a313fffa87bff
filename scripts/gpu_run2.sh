set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
