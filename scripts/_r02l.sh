DTB_PRINT_PLAN=1 timeout 120 python scripts/bb_probe.py c4 127 > gpurun_out/probe.log 2>&1
timeout 200 python scripts/bb_sweep.py 100 110 118 236 > gpurun_out/sweep.log 2>&1
timeout 120 python scripts/bb_times.py 20 > gpurun_out/times.log 2>&1
