for m in 1 2 3; do
  DTB_NVCC_EXTRA="-DDTB_SLIDE_MINB=$m" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
  echo "minb=$m"
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'], d['roofline']['frac'])"
  python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['kernel_ms'], d['roofline']['frac'])"
done
