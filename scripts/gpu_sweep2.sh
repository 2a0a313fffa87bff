for R in 168 200 232 255; do
  DTB_NVCC_EXTRA="-DDTB_SLIDE_MAXREG(V)=$R" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
  for H in 0 1; do
    echo -n "R=$R hint=$H  "
    DTB_L2HINT=$H python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'], d['roofline']['frac'])"
  done
done
python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_fast_path_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -1
