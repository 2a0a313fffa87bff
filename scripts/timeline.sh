# Timeline of one C4 launch with the strip/band mapping read from the launch plan itself.
PLAN=$(DTB_PRINT_PLAN=1 python scripts/bb_probe.py ${1:-c4} ${2:-127} 2>&1 | grep -m1 "dtb plan")
echo "$PLAN"
NS=$(echo "$PLAN" | sed -n 's/.*strips=\([0-9]*\).*/\1/p'); NP=$(echo "$PLAN" | sed -n 's/.* pairs=\([0-9]*\).*edge.*/\1/p'); NE=$(echo "$PLAN" | sed -n 's/.*edge TH=[0-9]* pairs=\([0-9]*\).*/\1/p')
DTB_PLAN="$NS $NP $NE" python scripts/bb_times.py page 8 2>&1 | grep -E "kernel|span|duration|main|strip  0|strip  1 |strip  9|strip 18|octile|^cta"
