timeout 600 python -m pytest tests/test_tmap_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/tmap_tests.log 2>&1; echo t=$?
cat > /tmp/tm.py <<'PY'
import torch, sys, statistics
sys.path.insert(0, '.')
from paper_1210_3165_b200 import engine, workloads, _lib
import paper_1210_3165_b200 as dt
img = torch.from_numpy(workloads.c4_image()).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for want in (True, False):
    ts = []
    for i in range(6):
        flush.zero_(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); engine.binarize(img, 127, "sauvola", 0.34, 128.0, want_tmap=want); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print("tmap" if want else "binary", _lib.lib().dtb_last_kernel().decode(), "ms", statistics.median(ts[1:]))
PY
timeout 300 python /tmp/tm.py > gpurun_out/tmap_time.log 2>&1; echo tm=$?
