timeout 900 python -m pytest tests/test_fast_path_gpu.py tests/test_parity_gpu.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
DTB_SLIDE_V=32 timeout 900 python -m pytest tests/test_fast_path_gpu.py -m gpu -x -q > gpurun_out/pytest_gpu32.log 2>&1; echo pytest32=$?
for v in 16 32; do
  echo "V=$v"
  DTB_SLIDE_V=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'], d['roofline']['frac'])"
  DTB_SLIDE_V=$v python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['kernel_ms'], d['roofline']['frac'])"
done
python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:slide_kernel -s 2 -c 1 -o gpurun_out/prof_slide python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
