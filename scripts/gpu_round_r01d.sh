# round-1 measurement bundle (gb_kernel default on C4): smoke, tests, bench (contract line), ncu launch list + full capture
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
timeout 900 python scripts/config_table.py --reps 10 > gpurun_out/config_table.json 2> gpurun_out/config_table.err; echo table=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gb_kernel" -s 2 -c 1 -o gpurun_out/prof_gb_r01d python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
