# A/B compile-time variants over the per-config table: bash scripts/ab_table.sh TAG "FLAGS" [TAG "FLAGS" ...]
while [ $# -ge 2 ]; do
  tag=$1; flags=$2; shift 2
  DTB_NVCC_EXTRA="$flags" timeout 400 python -c "from paper_1210_3165_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  timeout 600 python scripts/config_table.py --reps 10 > gpurun_out/table_$tag.json 2> gpurun_out/table_$tag.err; echo "$tag table=$?"
done
