# A/B of compile-time variants: bash scripts/ab_build_probe.sh "-DBB_STAGES=4" "-DBB_STAGES=5" ...
# builds each variant into /tmp and runs the C4 probe (bb_kernel time, exact-path groups) on it.
set -u
i=0
for FLAGS in "$@"; do
  i=$((i+1))
  ( DTB_LIB_OUT=/tmp/lib_ab$i.so DTB_NVCC_EXTRA="$FLAGS" python paper_1210_3165_b200/build.py --force > gpurun_out/ab_build$i.log 2>&1 ) &
done
wait
i=0
for FLAGS in "$@"; do
  i=$((i+1))
  echo "== $FLAGS"
  DTB_LIB_PATH=/tmp/lib_ab$i.so timeout 120 python scripts/bb_probe.py c4 127 2>&1 | tail -2
  DTB_LIB_PATH=/tmp/lib_ab$i.so timeout 300 python bench.py --emulate-bands 8 --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('band8', d['ms_per_band'], 'page', d['ms_whole_page'])"
done
