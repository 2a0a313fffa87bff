for Q in 0 1; do for P in 0 1; do for H in 0 1; do
  DTB_NVCC_EXTRA="-DDTB_PREFIX_QUARTERS=$Q -DDTB_PAR_PRODUCER=$P" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
  echo -n "quarters=$Q par_producer=$P l2hint=$H  "
  DTB_L2HINT=$H python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'])"
done; done; done
