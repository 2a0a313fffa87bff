for cfgw in "c2 15" "c3 31" "c5 3" "c5 35" "c5 131" "c4 127"; do
  set -- $cfgw
  for bs in 1 1.5 2 4; do
    ms=$(DTB_BAND_SCALE=$bs timeout 120 python bench.py --config $1 --window $2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['kernel_ms'])")
    echo "$1 W=$2 bs=$bs -> $ms"
  done
done
