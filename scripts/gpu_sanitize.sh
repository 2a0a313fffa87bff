TOOL=${TOOL:-memcheck}
for WS in 0 1; do
  DTB_WS=$WS timeout 600 compute-sanitizer --tool $TOOL --print-limit 20 python scripts/sanitize_case.py > gpurun_out/sanitize_${TOOL}_ws$WS.log 2>&1; echo "$TOOL ws=$WS rc=$?"
done
