# A/B a kernel env knob on the C4 bench: bash scripts/ab_env.sh VAR "v1 v2 ..." [reps]
VAR=$1; VALS=$2; REPS=${3:-3}
for r in $(seq 1 $REPS); do
  for v in $VALS; do
    env $VAR=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$VAR=$v', d['kernel_ms'], d['value'], d['clocks']['sm_mhz'])"
  done
done
