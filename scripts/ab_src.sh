# A/B two source trees on the C4 bench: bash scripts/ab_src.sh DIR_A DIR_B ... ("" = in-tree csrc)
for d in "$@"; do
  DTB_CSRC_DIR="$d" timeout 300 python -c "from paper_1210_3165_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $d"; continue; }
  for r in 1 2; do
    DTB_AB_ALLOW_MISSING=1 timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('[$d]', d['kernel_ms'], d['value'], d['clocks']['sm_mhz'])"
  done
done
