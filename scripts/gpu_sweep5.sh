for NS in 3 4 6; do
  DTB_NVCC_EXTRA="-DSLIDE_STAGES=$NS" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
  for V in 16 32; do
    echo -n "NS=$NS V=$V  "
    DTB_SLIDE_V=$V python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c4', d['kernel_ms'])"
    echo -n "             "
    DTB_SLIDE_V=$V python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['kernel_ms'])"
  done
done
