DTB_NVCC_EXTRA="-DDTB_DEBUG_BOUNDS=1" python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
for WS in 0 1 2; do DTB_WS=$WS timeout 900 python -m pytest tests/test_fast_path_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -1 | sed "s/^/ws=$WS: /"; done
python paper_1210_3165_b200/build.py --force > /dev/null 2>&1
