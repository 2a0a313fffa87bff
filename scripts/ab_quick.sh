# One GPU call: bb parity tests on the in-tree build, then A/B of compile-time variants
#   bash scripts/ab_quick.sh "-DX=1" "-DY=2" ...   (AB_NCU=1 adds DRAM bytes / L2 hit rate)
set -u
timeout 900 python -m pytest tests/test_bb_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -3
echo "== in-tree"
timeout 120 python scripts/bb_probe.py c4 127 2>&1 | tail -1
timeout 300 python bench.py --emulate-bands 8 --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('band8', d['ms_per_band'], 'page', d['ms_whole_page'])"
if [ "${AB_NCU:-0}" = 1 ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:bb_kernel -c 1 python scripts/bb_probe.py c4 127 2>&1 | grep -E "duration|bytes|hit_rate|inst_exec|issue_active" | awk '{print "   ", $1, $(NF-1), $NF}'
fi
if [ $# -gt 0 ]; then bash scripts/ab_build_probe.sh "$@"; fi
