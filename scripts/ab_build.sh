# A/B compile-time variants on the C4 bench (on the GPU box; the in-tree .so is rebuilt per variant)
# usage: bash scripts/ab_build.sh "FLAGS_A" "FLAGS_B" ... (each a quoted -D list; "" = default)
for flags in "$@"; do
  DTB_NVCC_EXTRA="$flags" timeout 300 python -c "from paper_1210_3165_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  for r in 1 2; do
    timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('[$flags]', d['kernel_ms'], d['value'], d['clocks']['sm_mhz'])"
  done
done
