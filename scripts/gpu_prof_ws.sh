export DTB_WS=1
python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ws_kernel -s 2 -c 1 -o gpurun_out/prof_ws python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
