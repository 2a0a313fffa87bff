# Race / bounds evidence for the asynchronous kernels (compute-sanitizer is closed on this pool):
# a library built with DTB_DEBUG_BOUNDS=1 (trap on any out-of-range shared-memory index) and
# DTB_PERTURB=1 (pseudo-random per-lane sleeps at every lane-to-lane / TMA hand-off in
# bb_kernel) runs the bit-exact parity suites of the hot kernels.
set -u
OUT=/tmp/libdocthresh_b200_safety.so
DTB_LIB_OUT=$OUT DTB_NVCC_EXTRA="-DDTB_DEBUG_BOUNDS=1 -DDTB_PERTURB=1" python paper_1210_3165_b200/build.py --force > gpurun_out/safety_build.log 2>&1; echo build=$?
for T in tests/test_bb_gpu.py tests/test_fast_path_gpu.py tests/test_parity_gpu.py tests/test_tmap_gpu.py; do
  DTB_LIB_PATH=$OUT timeout 1200 python -m pytest $T -m gpu -x -q 2>&1 | tail -1 | sed "s#^#$T: #"
done
