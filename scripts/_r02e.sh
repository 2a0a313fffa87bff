timeout 300 python -m pytest tests/test_bb_gpu.py -x -q > gpurun_out/bb_tests.log 2>&1; echo bbtests=$?
DTB_PRINT_PLAN=1 timeout 120 python scripts/bb_probe.py c4 127 > gpurun_out/probe.log 2>&1; echo probe=$?
DTB_BB_MINB=12 DTB_PRINT_PLAN=1 timeout 120 python scripts/bb_probe.py c4 127 > gpurun_out/probe12.log 2>&1; echo probe=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"bb_kernel" -s 1 -c 1 -o gpurun_out/prof_bb_v5 python scripts/bb_probe.py c4 127 > gpurun_out/ncu_bb.log 2>&1; echo ncu=$?
