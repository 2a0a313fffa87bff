# A/B of compile-time variants: bash scripts/ab_build_probe.sh "-DBB_STAGES=4" "-DBB_STAGES=5" ...
# Builds each variant into /tmp, then per variant: the C4 probe (kernel time, exact-path groups,
# golden hash), the 8-band emulation, and (AB_NCU=1) one ncu pass for DRAM bytes / L2 hit rate.
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
  DTB_LIB_PATH=/tmp/lib_ab$i.so timeout 120 python scripts/bb_probe.py ${AB_CFG:-c4} ${AB_WIN:-127} 2>&1 | tail -1
  if [ "${AB_EMUL:-1}" = 1 ]; then
    DTB_LIB_PATH=/tmp/lib_ab$i.so timeout 300 python bench.py --emulate-bands 8 --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('band8', d['ms_per_band'], 'page', d['ms_whole_page'])"
  fi
  if [ "${AB_NCU:-0}" = 1 ]; then
    DTB_LIB_PATH=/tmp/lib_ab$i.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --clock-control none -k regex:bb_kernel -c 1 python scripts/bb_probe.py ${AB_CFG:-c4} ${AB_WIN:-127} 2>&1 | grep -E "duration|bytes|hit_rate|inst_exec" | awk '{print "   ", $1, $(NF-1), $NF}'
  fi
done
