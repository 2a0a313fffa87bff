for AB in 0 1; do
  DTB_NVCC_EXTRA="-DDTB_ALU_BALANCE=$AB" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
  echo -n "alu_balance=$AB  "
  python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'])"
  echo -n "                 "
  python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['kernel_ms'])"
done
timeout 600 python -m pytest tests/test_fast_path_gpu.py -m gpu -x -q 2>&1 | tail -1
