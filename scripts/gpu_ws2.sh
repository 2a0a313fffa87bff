for R in 128 168; do
  DTB_NVCC_EXTRA="-DDTB_WS_MAXREG=$R" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
  for VO in 16 32; do
    echo -n "maxreg=$R VO=$VO  "
    DTB_WS=1 DTB_WS_VO=$VO timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'])"
    echo -n "                   "
    DTB_WS=1 DTB_WS_VO=$VO timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['kernel_ms'])"
  done
done
python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
DTB_WS=1 timeout 600 python -m pytest tests/test_fast_path_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -2
