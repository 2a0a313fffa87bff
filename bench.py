#!/usr/bin/env python
"""Benchmark: Sauvola binarization Mpixel/s on 1..8 B200 (+ % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c4|c3|c5|c2|c1] [--scaling weak|strong]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (default): BASELINE config 4 -- a 16384x16384 synthetic gray page,
Sauvola W=127 k=0.34 R=128, split in row bands across ranks with the 63-row
halos read in place from the neighbouring GPUs' HBM over NVLink (CUDA IPC mappings,
fused into the kernel's row staging; ``--halo nccl`` copies them with NCCL send/recv
every step instead).
``--scaling weak`` (default): every rank owns one full 16384x16384 band of a
(16384*N)-row page, so per-GPU work is fixed; ``strong`` splits the one
16384x16384 page N ways.  One step = one pass of the fused sliding-sum
binarization kernel over the rank's band (plus the NCCL halo copy with --halo nccl).

Prints ONE JSON line (rank 0).  ``value`` is whole-job Mpixel/s with inputs
resident in HBM, timed with CUDA events (max over ranks); ``e2e`` is the
same metric through the public API with pinned host buffers and the H2D/D2H
copies inside the timed region; ``roofline`` is the kernel's achieved
algorithmic bandwidth (2 B/px) vs the measured HBM copy peak; ``cpu_baseline``
is the CPU oracle port (oracle/, a C restatement of the reference's integral
engine) on the box's host cores on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Sauvola binarization Mpixel/s"
UNIT = "Mpixel/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c4", "c3", "c5", "c2", "c1"], default="c4")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong")
    ap.add_argument("--emulate-bands", type=int, default=0,
                    help="one GPU: time one middle band of an N-way row-band split (C4/N) "
                         "through dtb_binarize_segments; prints its own JSON line")
    ap.add_argument("--window", type=int, default=None, help="override W (c5 sweep point)")
    ap.add_argument("--halo", choices=["p2p", "nccl"], default="p2p",
                    help="row-band halos: read in place from the neighbours' HBM (CUDA IPC, "
                         "fused into the kernel's row staging) or copied with NCCL send/recv")
    ap.add_argument("--fresh-bands", action="store_true",
                    help="N > 1, p2p halos: refill every band inside the step (device copy) and order "
                         "the ranks with interprocess CUDA events (PeerHalos publish / retire) "
                         "instead of timing constant bands")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def build_id() -> str:
    """Hash of the kernel sources (csrc + the C-ABI header): ties a committed ncu traffic number
    to the build it was measured on."""
    import glob
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_1210_3165_b200", "csrc", "*.cu*")) +
                   glob.glob(os.path.join(ROOT, "include", "*.h")))
    for f in files:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + fh.read())
    return h.hexdigest()[:16]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


DTYPE = ("u8 in/out; exact uint32 window sums; decision from certified fp32 bounds "
         "(8-pixel groups, then per pixel), fp64 reference replay of undecided pixels")
# the per-pixel kernels (slide_kernel / ws_kernel: Niblack, small windows, small pages)
DTYPE_PIXEL = ("u8 in/out; exact uint32 window sums; per-pixel decision from a certified fp32 "
               "threshold, fp64 reference replay of pixels within the certified tolerance")


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid: str | None):
        self.lines = []
        cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
               "-lms", "50"]
        if uuid:
            cmd += ["-i", uuid]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


class NvmlSampler:
    """SM clock + clock-event (throttle) reasons read through NVML every ~2 ms by a thread while
    the timed region runs (the timed region of the default run is ~20 ms: nvidia-smi's fastest
    loop, 50 ms, gives it one sample).  NVML calls release the GIL; timing is by CUDA events."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, device_index: int):
        import pynvml
        import torch
        self.nv = pynvml
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(device_index).uuid)
        try:
            self.h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
        except Exception:
            self.h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
        self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)  # fail here, not in the thread
        self.lines = []  # (sm MHz, reasons bitmask); cleared at the start of the timed region
        self.run = True
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        nv = self.nv
        while self.run:
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                except Exception:
                    rs = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
                self.lines.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        self.run = False
        self.t.join(timeout=2)
        sm = [a for a, _ in self.lines]
        reasons = sorted({name for _, rs in self.lines for bit, name in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.mx,
                "reasons": reasons, "samples": len(sm), "source": "nvml, 2 ms period"}


def clock_sampler(device_index: int):
    try:
        return NvmlSampler(device_index)
    except Exception:
        return ClockSampler(None)


# ----------------------------------------------------------------------------- workloads

def workload(cfg_name, world, rank, scaling, window):
    """-> dict(kind, host arrays for this rank, params, pixels per rank, description)."""
    import numpy as np

    from paper_1210_3165_b200 import workloads as wl
    cfg = wl.CONFIGS[cfg_name]
    win = window or cfg.windows[0]
    if cfg_name in ("c4", "c5", "c1"):
        img = {"c4": wl.c4_image, "c5": wl.c5_image, "c1": wl.c1_image}[cfg_name]()
        H, Wd = img.shape
        r = win // 2
        if scaling == "weak":
            # page = `world` copies of the image stacked vertically; rank i owns copy i
            rows = H * world
            y0, y1 = H * rank, H * (rank + 1)
            top = img[H - r:] if rank > 0 else img[:0]
            bot = img[:r] if rank < world - 1 else img[:0]
            band = img
        else:
            rows = H
            y0, y1 = H * rank // world, H * (rank + 1) // world
            top, band, bot = img[max(y0 - r, 0):y0], img[y0:y1], img[y1:min(y1 + r, H)]
        host_halo = np.ascontiguousarray(np.concatenate([top, band, bot]))
        return dict(kind="rowband", band=np.ascontiguousarray(band), halo=host_halo,
                    a=y0 - len(top), rows=rows, y0=y0, y1=y1, cols=Wd, win=win,
                    method=cfg.method, k=cfg.k, r=cfg.r, px_rank=(y1 - y0) * Wd,
                    desc=(f"{cfg_name}: {H}x{Wd} gray page(s), {cfg.method} W={win} k={cfg.k} "
                          f"R={cfg.r}; {'weak' if scaling == 'weak' else 'strong'} row-band "
                          f"split over {world} GPU(s), {r}-row halos"),
                    shape=[rows, Wd])
    if cfg_name == "c3":
        n_total = 64 * (world if scaling == "weak" else 1)
        per = [i for i in range(n_total) if (i * world) // n_total == rank]
        imgs = np.stack([wl.c3_image(i % 64) for i in per])
        return dict(kind="batch", stack=imgs, win=win, method=cfg.method, k=cfg.k, r=cfg.r,
                    px_rank=imgs.size, shape=[n_total, 2048, 2048],
                    desc=f"c3: {n_total} x 2048x2048 gray, niblack W={win} k={cfg.k}, by image")
    if cfg_name == "c2":
        rgb = wl.c2_rgb()
        return dict(kind="rgb", rgb=rgb, win=win, method=cfg.method, k=cfg.k, r=cfg.r,
                    px_rank=rgb.shape[0] * rgb.shape[1], shape=list(rgb.shape),
                    desc=f"c2: 3508x2480 RGB page, fused to_gray + sauvola W={win}")
    raise ValueError(cfg_name)


def halo_bytes(w, world) -> int:
    """Bytes of halo rows all ranks read from their neighbours per step (NVLink)."""
    if world <= 1:
        return 0
    from paper_1210_3165_b200 import distributed as D
    r = w["win"] // 2
    rows = w["rows"]
    total = 0
    for q in range(world):
        y0, y1 = D.band_bounds(rows, world, q)
        a, z = D.halo_bounds(rows, y0, y1, r)
        total += (y0 - a + z - y1) * w["cols"]
    return int(total)


# ----------------------------------------------------------------------------- our arm

def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1210_3165_b200 import distributed as D
    from paper_1210_3165_b200 import engine
    import paper_1210_3165_b200 as dt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only plumbing: DTB_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 and
    # DTB_BENCH_BACKEND=gloo avoids NCCL's one-rank-per-GPU rule, so the N>1 code path (p2p
    # halo mapping, max-over-ranks timing) can be exercised on a one-GPU box.  Numbers from
    # such a run are not measurements.
    backend = os.environ.get("DTB_BENCH_BACKEND", "nccl")
    if os.environ.get("DTB_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    w = workload(a.config, world, rank, a.scaling, a.window)
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20))
    stream = torch.cuda.current_stream()

    # ---- device-resident buffers, rotated so the per-step footprint defeats L2
    if w["kind"] == "rowband":
        band = torch.from_numpy(w["band"]).to(dev)
        per_step_bytes = 2 * band.numel()
        nrot = max(1, -(-2 * l2 // per_step_bytes))
        bands = [band] + [band.clone() for _ in range(nrot - 1)]
        outs = [torch.empty_like(band) for _ in range(nrot)]
        r = w["win"] // 2
        ha, hz = D.halo_bounds(w["rows"], w["y0"], w["y1"], r)
        use_p2p = (world > 1 and a.halo == "p2p" and
                   all(D.p2p_possible(w["rows"], world, q, r) for q in range(world)))
        halo_bufs = [torch.empty((hz - ha,) + tuple(band.shape[1:]), dtype=torch.uint8,
                                 device=dev) for _ in range(nrot)] if world > 1 and not use_p2p else None
        # p2p: map the neighbours' bands once (CUDA IPC); each step's kernel then reads the
        # halo rows in place over NVLink -- no exchange step.  Bands are constant after setup.
        peers = None
        if use_p2p:
            try:
                hostg = None
                if a.fresh_bands:  # host-only handshake group for the event hand-offs
                    import torch.distributed as dist
                    hostg = (dist.group.WORLD if dist.get_backend() == "gloo"
                             else dist.new_group(backend="gloo"))
                    band_src = band.clone()
                peers = [D.PeerHalos(bands[j], w["rows"], r, events=a.fresh_bands, host_group=hostg)
                         for j in range(nrot)]
                peers[0].barrier()
            except (RuntimeError, ValueError) as exc:  # e.g. VMM allocations without IPC handles
                if rank == 0:
                    print(f"[bench] p2p halos unavailable ({exc}); using NCCL", file=sys.stderr)
                use_p2p, peers = False, None
        if world > 1 and not use_p2p and halo_bufs is None:
            halo_bufs = [torch.empty((hz - ha,) + tuple(band.shape[1:]), dtype=torch.uint8,
                                     device=dev) for _ in range(nrot)]
        w["halo_transport"] = ("none (1 GPU)" if world == 1 else
                     "read in place from the neighbours' HBM over NVLink (CUDA IPC), fused into "
                     "the kernel's row staging" + ("; bands refilled every step, ranks ordered by "
                     "interprocess CUDA events" if a.fresh_bands else "")
                     if use_p2p else "NCCL send/recv copy per step")
        launches_per_step = 1

        def kernel(i):
            if world > 1:
                buf, a0 = D.exchange_halos(bands[i], w["rows"], r, out=halo_bufs[i])
            else:
                buf, a0 = bands[i], w["y0"]
            return buf, a0

        def step(i, ev=None):
            j = i % nrot
            if use_p2p:
                if ev is not None:
                    ev[0].record(stream)
                if a.fresh_bands:  # new rows every step; ranks ordered on the device (IPC events)
                    bands[j].copy_(band_src, non_blocking=True)
                    peers[j].binarize(w["win"], w["method"], w["k"], w["r"], out=outs[j], sync="events")
                else:
                    peers[j].binarize(w["win"], w["method"], w["k"], w["r"], out=outs[j], sync=False)
                if ev is not None:
                    ev[1].record(stream)
                return
            buf, a0 = kernel(j)
            if ev is not None:
                ev[0].record(stream)
            engine.binarize_band(buf, a0, w["rows"], w["y0"], w["y1"], w["win"], w["method"],
                                 w["k"], w["r"], out=outs[j])
            if ev is not None:
                ev[1].record(stream)
    elif w["kind"] == "batch":
        stack = torch.from_numpy(w["stack"]).to(dev)
        per_step_bytes = 2 * stack.numel()
        nrot = max(1, -(-2 * l2 // per_step_bytes))
        stacks = [stack] + [stack.clone() for _ in range(nrot - 1)]
        outs = [torch.empty_like(stack) for _ in range(nrot)]
        launches_per_step = 1

        def step(i, ev=None):
            j = i % nrot
            if ev is not None:
                ev[0].record(stream)
            engine.binarize_batch(stacks[j], w["win"], w["method"], w["k"], w["r"], out=outs[j])
            if ev is not None:
                ev[1].record(stream)
    else:  # rgb fused
        rgb = torch.from_numpy(w["rgb"]).to(dev)
        per_step_bytes = 4 * rgb.shape[0] * rgb.shape[1]
        nrot = max(1, -(-2 * l2 // per_step_bytes))
        rgbs = [rgb] + [rgb.clone() for _ in range(nrot - 1)]
        launches_per_step = 2

        def step(i, ev=None):
            j = i % nrot
            if ev is not None:
                ev[0].record(stream)
            engine.rgb_binarize(rgbs[j], w["win"], w["method"], w["k"], w["r"])
            if ev is not None:
                ev[1].record(stream)

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    sampler = clock_sampler(local) if rank == 0 else None
    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize()

    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(a.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.lines.clear()  # keep only samples taken during the timed region
    t0.record(stream)
    for i in range(a.steps):
        step(i, kev[i])
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    ms = t0.elapsed_time(t1) / a.steps
    kms = statistics.fmean(s.elapsed_time(e) for s, e in kev)
    from paper_1210_3165_b200 import _lib as _dl
    kernel_name = _dl.lib().dtb_last_kernel().decode() or None  # the timed launches' kernel
    if world > 1:
        t = torch.tensor([ms, kms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
    total_px = w["px_rank"] * world if a.scaling == "weak" or w["kind"] != "rowband" else (
        w["shape"][0] * w["shape"][1])
    if w["kind"] == "batch" and a.scaling == "strong":
        total_px = int(np.prod(w["shape"]))
    value = total_px / (ms / 1e3) / 1e6

    # ---- roofline of the dominant kernel (per-launch algorithmic bytes / avg duration)
    alg_bytes = per_step_bytes
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / (kms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(prof):
        try:
            pt = json.load(open(prof))
            # only a capture of this very build, config and split counts
            if (pt.get("config") == a.config and pt.get("window") == w["win"] and
                    pt.get("build") == build_id() and pt.get("n_gpus", 1) == world and
                    pt.get("kernel") == kernel_name):
                traffic = pt.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, w, world, rank, local, dev, barrier)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(w, a.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True,
            "scaling": a.scaling if w["kind"] != "rgb" else "weak",
            "vs_baseline": None, "dtype": DTYPE if kernel_name == "bb_kernel" else DTYPE_PIXEL,
            "data": "synthetic (seeded, paper_1210_3165_b200/workloads.py)",
            "config": {"workload": w["desc"], "image": w["shape"], "window": w["win"],
                       "method": w["method"], "k": w["k"], "r": w["r"],
                       "parallelism": f"{'rowband' if w['kind'] == 'rowband' else 'image'}{world}",
                       **({"halo": w["halo_transport"],
                           "halo_bytes_per_step": halo_bytes(w, world)} if "halo_transport" in w else {}),
                       "l2": (f"{nrot} rotating input/output buffer sets, "
                              f"{nrot * per_step_bytes / 2**20:.0f} MiB per rank >= 2x L2 "
                              f"({l2 / 2**20:.0f} MiB)")},
            "kernel_ms": round(kms, 5), "kernel": kernel_name, "build": build_id(),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "alg_bytes_per_launch": alg_bytes},
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": launches_per_step * a.steps,
            "gpu": torch.cuda.get_device_name(dev),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_band_emulation(a):
    """One GPU: time one middle band of an N-way row-band split of the page through the
    segmented-input entry (dtb_binarize_segments), the halo rows in separate buffers exactly
    as the p2p path maps them from the neighbours, against the whole page in the same
    process.  Reports ms per band, the linear target (whole page / N) and the efficiency."""
    import numpy as np
    import torch

    from paper_1210_3165_b200 import _lib, engine, workloads as wl
    from paper_1210_3165_b200 import distributed as D
    nb = a.emulate_bands
    cfg = wl.CONFIGS[a.config]
    if a.config not in ("c4", "c5", "c1"):
        raise SystemExit("--emulate-bands: row-band configs only (c4, c5, c1)")
    win = a.window or cfg.windows[0]
    r = win // 2
    img = {"c4": wl.c4_image, "c5": wl.c5_image, "c1": wl.c1_image}[a.config]()
    H, Wd = img.shape
    b = nb // 2  # a middle band: both halos come from neighbours
    y0, y1 = D.band_bounds(H, nb, b)
    ha, hz = D.halo_bounds(H, y0, y1, r)
    dev = torch.device("cuda", 0)
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20))
    step_bytes = (hz - ha) * Wd + (y1 - y0) * Wd
    nrot = max(1, -(-2 * l2 // step_bytes))
    sets = []
    for _ in range(nrot):
        top = torch.from_numpy(np.ascontiguousarray(img[ha:y0])).to(dev)
        mid = torch.from_numpy(np.ascontiguousarray(img[y0:y1])).to(dev)
        bot = torch.from_numpy(np.ascontiguousarray(img[y1:hz])).to(dev)
        out = torch.empty((y1 - y0, Wd), dtype=torch.uint8, device=dev)
        segs = [(t.data_ptr(), t.stride(0), t.shape[0], Wd) for t in (top, mid, bot)]
        sets.append((segs, out, (top, mid, bot)))
    page = torch.from_numpy(img).to(dev)
    pout = torch.empty_like(page)
    flush = torch.empty(2 * l2, dtype=torch.uint8, device=dev)

    def timed(fn, reps):
        ts = []
        for i in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(i)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def band(i):
        segs, out, _ = sets[i % nrot]
        engine.binarize_segments(segs, ha, H, y0, y1, win, cfg.method, cfg.k, cfg.r, out=out)

    def whole(i):
        engine.binarize(page, win, cfg.method, cfg.k, cfg.r, want_tmap=False, out=pout)

    for i in range(a.warmup):
        band(i)
        whole(i)
    torch.cuda.synchronize()
    t_band = timed(band, max(5, a.steps))
    kb = _lib.lib().dtb_last_kernel().decode()
    t_page = timed(whole, max(5, a.steps))
    kp = _lib.lib().dtb_last_kernel().decode()
    ok = np.array_equal(sets[0][1].cpu().numpy(), pout.cpu().numpy()[y0:y1])
    print(json.dumps({
        "mode": "band_emulation", "metric": METRIC, "config": a.config, "window": win,
        "bands": nb, "band": b, "band_rows": [y0, y1], "halo_rows": [ha, y0, y1, hz],
        "ms_per_band": round(t_band, 5), "band_kernel": kb,
        "ms_whole_page": round(t_page, 5), "page_kernel": kp,
        "linear_target_ms": round(t_page / nb, 5),
        "efficiency": round(t_page / nb / t_band, 4),
        "emulated_value": round(H * Wd / (t_band / 1e3) / 1e6, 1), "unit": UNIT,
        "halo_bytes_per_band": int((y0 - ha + hz - y1) * Wd),
        "band_equals_page_rows": bool(ok),
        "l2": f"flushed ({2 * l2 >> 20} MiB memset) before every rep"}), flush=True)


def run_e2e(a, w, world, rank, local, dev, barrier):
    """Public API, pinned host in/out, H2D + kernel + D2H inside the timed region."""
    import torch

    import paper_1210_3165_b200 as dt
    from paper_1210_3165_b200 import engine

    stream = torch.cuda.current_stream()
    if w["kind"] == "rowband":
        host_in = torch.from_numpy(w["halo"]).pin_memory()
        host_out = torch.empty((w["y1"] - w["y0"], w["cols"]), dtype=torch.uint8).pin_memory()
        if world == 1 and w["halo"].shape[0] == w["rows"]:
            params = dt.BinarizationParams(method=w["method"], engine="integral", window=w["win"],
                                           r=w["r"], **({"k_sauvola": w["k"]} if w["method"] == "sauvola" else {"k_niblack": w["k"]}))

            def call():
                dt.binarize(host_in, params, return_tmap=False, out=host_out)
        else:
            def call():
                buf = host_in.to(dev, non_blocking=True)
                out = engine.binarize_band(buf, w["a"], w["rows"], w["y0"], w["y1"], w["win"],
                                           w["method"], w["k"], w["r"])
                host_out.copy_(out, non_blocking=True)
                stream.synchronize()
        h2d, d2h = host_in.numel(), host_out.numel()
    elif w["kind"] == "batch":
        host_in = torch.from_numpy(w["stack"]).pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()

        def call():
            s = host_in.to(dev, non_blocking=True)
            out = engine.binarize_batch(s, w["win"], w["method"], w["k"], w["r"])
            host_out.copy_(out, non_blocking=True)
            stream.synchronize()
        h2d, d2h = host_in.numel(), host_out.numel()
    else:
        host_in = torch.from_numpy(w["rgb"]).pin_memory()
        host_out = torch.empty(w["rgb"].shape[:2], dtype=torch.uint8).pin_memory()

        def call():
            s = host_in.to(dev, non_blocking=True)
            out = engine.rgb_binarize(s, w["win"], w["method"], w["k"], w["r"])
            host_out.copy_(out, non_blocking=True)
            stream.synchronize()
        h2d, d2h = host_in.numel(), host_out.numel()
    for _ in range(max(1, a.warmup)):
        call()
    steps = max(3, a.steps // 2)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(steps):
        call()
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = t0.elapsed_time(t1) / steps
    from paper_1210_3165_b200 import _lib as _dl
    e2e_kernel = _dl.lib().dtb_last_kernel().decode() or None
    if world > 1:
        import torch.distributed as dist
        on_dev = os.environ.get("DTB_BENCH_BACKEND", "nccl") == "nccl"
        t = torch.tensor([ms], dtype=torch.float64, device=dev if on_dev else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    px = w["px_rank"] * world
    return {"value": round(px / (ms / 1e3) / 1e6, 1), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
            "ms_per_step": round(ms, 4), "steps": steps, "kernel": e2e_kernel,
            "path": "paper_1210_3165_b200.binarize / engine C-ABI calls, pinned host buffers "
                    "(H2D, compute and D2H overlapped in row chunks; each chunk is a band launch)"}


# ----------------------------------------------------------------------------- CPU arm

def cpu_sample(w):
    """Bounded CPU sample of the workload: <= 2048 rows of the band (plus halo rows)."""
    import numpy as np
    if w["kind"] == "rowband":
        img = w["halo"]
        top = w["y0"] - w["a"]
        n = min(2048, w["y1"] - w["y0"])
        r = w["win"] // 2
        lo, hi = max(top - r, 0), min(top + n + r, img.shape[0])
        sub = np.ascontiguousarray(img[lo:hi])
        return sub, n, (top - lo), f"rows [{w['y0']},{w['y0'] + n}) of the band + {r}-row halos"
    if w["kind"] == "batch":
        return w["stack"][0], w["stack"][0].shape[0], 0, "1 of the 2048x2048 images"
    from oracle import to_gray
    g = to_gray(w["rgb"])
    return g, g.shape[0], 0, "the full page (gray binarize only)"


def cpu_baseline(w, seconds, reps=None):
    """The C restatement of the reference's integral engine on all host threads over a bounded
    sample of the workload, plus the same on one thread and the numpy restatement of the
    reference's own numpy code (oracle/numpy_ref.py, single-threaded as numpy is) on a
    512-row slice -- BASELINE.md section 3."""
    import oracle
    threads = len(os.sched_getaffinity(0))
    sub, n, off, desc = cpu_sample(w)
    px = n * sub.shape[1]
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t = time.perf_counter()
        oracle.binarize(sub, w["win"], w["method"], w["k"], w["r"], tmap=False, threads=threads)
        times.append(time.perf_counter() - t)
        if (reps and len(times) >= reps) or (not reps and time.perf_counter() > t_end):
            break
    med = statistics.median(times)
    one = single_thread_rates(sub, w, min(n, 512))
    total = w["px_rank"]
    return {"value": round(px / med / 1e6, 2), "unit": UNIT, "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "sample_fraction": round(px / total, 6),
            "single_thread": one,
            "sample": f"{desc}: {px} px ({px / total:.4f} of the rank's pixels; the value is that "
                      f"sample's rate), {len(times)} reps, median {med * 1e3:.1f} ms; C restatement "
                      "of the reference integral engine (oracle/oracle.c)"}


def single_thread_rates(sub, w, rows):
    """Mpixel/s on ONE host thread over the first `rows` output rows of the sample: the C port
    and the numpy restatement of the reference's integral engine."""
    import numpy as np

    import oracle
    from oracle import numpy_ref
    r = w["win"] // 2
    sl = np.ascontiguousarray(sub[:min(sub.shape[0], rows + 2 * r)])
    px = sl.shape[0] * sl.shape[1]
    t = time.perf_counter()
    oracle.binarize(sl, w["win"], w["method"], w["k"], w["r"], tmap=False, threads=1)
    c1 = time.perf_counter() - t
    t = time.perf_counter()
    numpy_ref.binarize(sl, w["win"], w["method"], w["k"], w["r"])
    n1 = time.perf_counter() - t
    return {"c_port_mpix_s": round(px / c1 / 1e6, 2),
            "numpy_restatement_mpix_s": round(px / n1 / 1e6, 3),
            "sample_px": int(px)}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    w = workload(a.config, 1, 0, a.scaling, a.window)
    threads = len(os.sched_getaffinity(0))
    sub, n, off, desc = cpu_sample(w)
    px = n * sub.shape[1]
    for _ in range(a.warmup):
        oracle.binarize(sub, w["win"], w["method"], w["k"], w["r"], tmap=False, threads=threads)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        oracle.binarize(sub, w["win"], w["method"], w["k"], w["r"], tmap=False, threads=threads)
    dt = (time.perf_counter() - t0) / a.steps
    v = round(px / dt / 1e6, 2)
    total = w["px_rank"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
            "dtype": "u8 in/out; int64 sums; fp64 epilogue (reference op order)",
            "data": "synthetic (seeded, paper_1210_3165_b200/workloads.py)",
            # the GPU arm's workload and parameters; each step times a bounded sample of it
            "config": {"workload": w["desc"], "image": w["shape"], "window": w["win"],
                       "method": w["method"], "k": w["k"], "r": w["r"],
                       "parallelism": f"cpu{threads}", "sample_fraction": round(px / total, 6)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(), "sample_fraction": round(px / total, 6),
                             "sample": f"{desc}: {px} px per step ({px / total:.4f} of the "
                                       "workload; value = that sample's rate)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(a) -> int:
    """--gpus N > 1 without torchrun: run this script under torch.distributed.run, N ranks."""
    import socket
    if os.environ.get("DTB_BENCH_SAME_DEVICE") != "1":
        import torch
        have = torch.cuda.device_count()
        if have < a.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {a.gpus}: only {have} GPU(s) visible"}))
            return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(a.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        sys.exit(self_launch(a))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != a.gpus and not (a.impl == "reference" and world == 1):
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        run_reference(a)
    elif a.emulate_bands:
        run_band_emulation(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
