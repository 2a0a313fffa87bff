timeout 120 python scripts/bb_probe.py c4 127 > gpurun_out/probe.log 2>&1; echo probe=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"bb_kernel" -s 1 -c 1 -o gpurun_out/prof_bb_v1 python scripts/bb_probe.py c4 127 > gpurun_out/ncu_bb.log 2>&1; echo ncu=$?
