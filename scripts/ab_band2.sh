# A/B of compile-time variants on the half-page band launch (ncu metrics + plan)
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
  DTB_LIB_PATH=/tmp/lib_ab$i.so python bench.py --emulate-bands ${AB_BANDS:-2} --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('band', d['ms_per_band'], 'page', d['ms_whole_page'])"
  DTB_LIB_PATH=/tmp/lib_ab$i.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --clock-control none -k regex:bb_kernel -s 6 -c 1 python bench.py --emulate-bands ${AB_BANDS:-2} --steps 3 --warmup 3 2>&1 | grep -E "duration|bytes|hit_rate|inst_exec" | awk '{print "   ", $1, $(NF-1), $NF}'
done
