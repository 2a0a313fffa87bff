timeout 300 python -m pytest tests/test_bb_gpu.py -x -q > gpurun_out/bb_tests.log 2>&1; echo bbtests=$?
timeout 400 python scripts/bb_sweep.py 96 124 160 248 > gpurun_out/sweep.log 2>&1
DTB_BB_MINB=12 timeout 200 python scripts/bb_sweep.py 124 248 > gpurun_out/sweep12.log 2>&1
DTB_BB_BANDS=248 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"bb_kernel" -s 1 -c 1 -o gpurun_out/prof_bb_v6 python scripts/bb_probe.py c4 127 > gpurun_out/ncu_bb.log 2>&1; echo ncu=$?
