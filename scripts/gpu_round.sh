# Measurement bundle for one GPU call (writes gpurun_out/):
#   bash scripts/gpu_round.sh TAG         smoke, GPU tests, bench (+ reference arm), config
#                                          table, ncu launch list and one full capture of the
#                                          C4 hot kernel
set -u
TAG=${1:-run}
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > $O/${TAG}_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_ref.log 2>&1; echo ref=$?
timeout 600 python bench.py --emulate-bands 8 --steps 10 --warmup 3 > $O/${TAG}_emul8.log 2>&1; echo emul=$?
timeout 300 python scripts/tmap_probe.py > $O/${TAG}_tmap_probe.log 2>&1; echo tmap=$?
timeout 300 python scripts/c3_probe.py > $O/${TAG}_c3_probe.log 2>&1; echo c3=$?
timeout 900 python scripts/config_table.py --reps 10 > $O/${TAG}_config_table.json 2> $O/${TAG}_config_table.err; echo table=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bb_kernel" -s 2 -c 1 -o $O/${TAG}_prof_bb \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bb_kernel" -s 6 -c 1 -o $O/${TAG}_prof_band \
  python bench.py --emulate-bands 8 --steps 3 --warmup 3 > $O/${TAG}_ncu_band.log 2>&1; echo ncu_band=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"slide_kernel" -s 2 -c 1 -f -o $O/${TAG}_prof_c3 \
  python scripts/c3_probe.py > $O/${TAG}_ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 300 python scripts/pad_probe.py > $O/${TAG}_pad_probe.log 2>&1; echo pad=$?
timeout 1800 bash scripts/safety_checks.sh > $O/${TAG}_safety_checks.txt 2>&1; echo safety=$?
