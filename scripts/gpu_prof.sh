python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:slide_kernel -s 2 -c 1 -o gpurun_out/prof_slide python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu.log 2>&1; echo ncu=$?
