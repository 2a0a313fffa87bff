# correctness across build variants: bash scripts/ab_correct.sh "FLAGS_A" "FLAGS_B" ... -- script args
for flags in "$@"; do
  DTB_NVCC_EXTRA="$flags" timeout 300 python -c "from paper_1210_3165_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  echo "[$flags] $(DTB_WS=1 timeout 120 python scripts/bisect_c5.py 195 211 243 2>&1 | tail -1)"
done
