# GPU call: edge-padded single-strip layout (DTB_PAD) A/B on C3 / C2 / C5, then the parity suites
# that exercise slide_kernel (scripts/, analysis only).
set -u
O=gpurun_out
TAG=${1:-pad}
for m in 0 2; do
  echo "== DTB_PAD=$m"
  DTB_PAD=$m DTB_PRINT_PLAN=1 timeout 300 python scripts/c3_probe.py 2>&1 | grep -v Warn | tail -2
  DTB_PAD=$m DTB_PRINT_PLAN=1 timeout 300 python scripts/c5_probe.py --windows 3,19,35,51,67 --reps 8 2>&1 | grep -v Warn | sort -u | tail -30
done > $O/${TAG}_ab.log 2>&1
timeout 1500 python -m pytest tests/test_fast_path_gpu.py tests/test_tmap_gpu.py tests/test_parity_gpu.py tests/test_bb_gpu.py -x -q > $O/${TAG}_pytest.log 2>&1; echo pytest=$?
tail -5 $O/${TAG}_pytest.log
cat $O/${TAG}_ab.log
