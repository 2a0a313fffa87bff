# per-config table with the group-bound kernel on (default) and off
timeout 600 python scripts/config_table.py --reps 10 > gpurun_out/config_table_gb.json 2> gpurun_out/config_table_gb.err; echo gb=$?
DTB_GB=0 timeout 600 python scripts/config_table.py --reps 10 > gpurun_out/config_table_ws.json 2> gpurun_out/config_table_ws.err; echo ws=$?
