"""bench.py's N>1 code path (torchrun, p2p halo mapping, max-over-ranks timing, one JSON line
from rank 0) exercised with 2 ranks on this box's single GPU through the test-only
DTB_BENCH_SAME_DEVICE / DTB_BENCH_BACKEND=gloo switches.  Kernels only read each other's
bands after a barrier; the numbers are not measurements."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, extra_env):
    env = dict(os.environ, DTB_BENCH_SAME_DEVICE="1", DTB_BENCH_BACKEND="gloo", **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           "2", "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", *args]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg", ["c1", "c5"])
def test_bench_two_ranks_p2p(cfg):
    d = _torchrun(["--config", cfg, "--steps", "2", "--warmup", "3", "--no-cpu-baseline"], {})
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert "CUDA IPC" in d["config"]["halo"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] == 2


def test_bench_two_ranks_fresh_bands_event_ordering():
    d = _torchrun(["--config", "c5", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                   "--fresh-bands"], {})
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert "interprocess CUDA events" in d["config"]["halo"]


def test_bench_reference_arm_two_ranks():
    d = _torchrun(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3"], {})
    assert d["impl"] == "reference" and d["value"] > 0


def test_bench_self_launches_n_ranks():
    # `bench.py --gpus 2` without torchrun re-launches itself under torch.distributed.run
    env = dict(os.environ, DTB_BENCH_SAME_DEVICE="1", DTB_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c1",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["halo_bytes_per_step"] == 2 * 7 * 512  # 2 boundaries' worth, r = 7


def test_bench_world_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--config", "c1", "--steps", "1", "--warmup", "1"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT, env=env)
    assert res.returncode != 0 and "WORLD_SIZE" in (res.stdout + res.stderr)


def test_band_emulation_mode():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5",
                          "--window", "131", "--emulate-bands", "4", "--steps", "3",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    d = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][0])
    assert d["mode"] == "band_emulation" and d["band_equals_page_rows"]
    assert d["ms_per_band"] > 0 and d["halo_bytes_per_band"] == 2 * 65 * 4096
