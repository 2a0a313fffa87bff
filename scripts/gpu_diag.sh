for D in 0 1 2 3; do
  DTB_NVCC_EXTRA="-DDTB_DIAG_SKIP=$D" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
  echo -n "skip=$D  "
  python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'])"
done
