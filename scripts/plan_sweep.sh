# Band-count / kernel-choice sweep on the smaller configs (kernel ms from bench.py)
for cfgw in "c2 15" "c2 63" "c3 31" "c5 3" "c5 35" "c5 131" "c5 243" "c4 127"; do
  set -- $cfgw
  for ws in 2 1; do
    for bs in 1 0.5 0.25; do
      ms=$(DTB_WS=$ws DTB_BAND_SCALE=$bs timeout 120 python bench.py --config $1 --window $2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['kernel_ms'])")
      echo "$1 W=$2 ws=$ws bs=$bs -> $ms"
    done
  done
  DTB_PRINT_PLAN=1 timeout 60 python bench.py --config $1 --window $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "dtb plan" | head -1
done
