# One GPU call: full ncu captures (with SASS source page) of the C3 per-pixel kernel and the
# C4 binary+tmap kernel, after plain runs of both probes (scripts/, analysis only).
set -u
O=gpurun_out
TAG=${1:-prof}
DTB_PRINT_PLAN=1 timeout 300 python scripts/c3_probe.py > $O/${TAG}_c3_probe.log 2>&1; echo c3=$?
DTB_PRINT_PLAN=1 timeout 300 python scripts/tmap_probe.py > $O/${TAG}_tmap_probe.log 2>&1; echo tmap=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"slide_kernel" -s 2 -c 1 -f -o $O/${TAG}_prof_c3 \
  python scripts/c3_probe.py > $O/${TAG}_ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"slide_kernel" -s 1 -c 1 -f -o $O/${TAG}_prof_tmap \
  python scripts/tmap_probe.py > $O/${TAG}_ncu_tmap.log 2>&1; echo ncu_tmap=$?
for k in c3 tmap; do
  ncu -i $O/${TAG}_prof_$k.ncu-rep --page source --csv --print-source sass > $O/${TAG}_${k}_sass.csv 2>/dev/null
done
ls -la $O | tail -12
