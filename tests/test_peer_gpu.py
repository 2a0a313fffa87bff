"""Fused in-place halo reads (SURVEY.md §8 e): dtb_binarize_segments over separate buffers,
and PeerHalos across two processes sharing bands through CUDA IPC.  Both must equal the
whole-page binarization bit for bit.

The two-process test runs both ranks on the one GPU of this sandbox: each kernel only READS
the other's band after a host barrier, so no kernel waits on another; it exercises the IPC
mapping and segment addressing, not NVLink bandwidth."""

import os
import socket

import numpy as np
import pytest
import torch

from paper_1210_3165_b200 import _lib, distributed as D, engine, workloads

pytestmark = pytest.mark.gpu


def _page(h, w, seed=3):
    return workloads.doc_gray(h, w, seed, max(10, h * w // 4000))


@pytest.mark.parametrize("h,w,win,cuts", [(700, 1031, 127, (300, 520)), (257, 4096, 31, (100, 170)),
                                          (64, 200, 15, (20, 40)), (300, 777, 63, (0, 300)),
                                          (1200, 2048, 127, (600, 1100))])
def test_segments_equal_whole_page(h, w, win, cuts):
    img = torch.from_numpy(_page(h, w)).cuda()
    want, _ = engine.binarize(img, win, "sauvola", 0.34, 128.0, want_tmap=False)
    r = win // 2
    c0, c1 = cuts
    # three separate, differently pitched allocations holding rows [0,c0), [c0,c1), [c1,h)
    segs, keep = [], []
    for lo, hi, pad in ((0, c0, 16), (c0, c1, 48), (c1, h, 0)):
        if hi > lo:
            pitch = (w + 15) // 16 * 16 + pad  # 16-byte aligned rows, different per buffer
            buf = torch.zeros((hi - lo, pitch), dtype=torch.uint8, device="cuda")
            buf[:, :w] = img[lo:hi]
            keep.append(buf)
            segs.append((buf.data_ptr(), buf.stride(0), hi - lo, w))
    # output the middle band's rows only (the rows a rank owns), reading its halos in place
    y0, y1 = c0, c1 if c1 > c0 else h
    out = engine.binarize_segments(segs, 0, h, y0, y1, win, "sauvola", 0.34, 128.0)
    assert torch.equal(out, want[y0:y1])
    out_all = engine.binarize_segments(segs, 0, h, 0, h, win, "niblack", -0.2, 128.0)
    want_n, _ = engine.binarize(img, win, "niblack", -0.2, 128.0, want_tmap=False)
    assert torch.equal(out_all, want_n)
    del r


def test_segments_reject_unaligned_and_short():
    img = torch.from_numpy(_page(100, 300)).cuda()
    big = torch.zeros((100, 301), dtype=torch.uint8, device="cuda")
    big[:, 1:] = img
    segs = [(big.data_ptr() + 1, big.stride(0), 100, 300)]  # misaligned base
    with pytest.raises(RuntimeError, match="16-byte"):
        engine.binarize_segments(segs, 0, 100, 0, 100, 15, "sauvola", 0.34, 128.0)
    segs = [(img.data_ptr(), img.stride(0), 50, 300)]
    with pytest.raises(ValueError, match="segments hold"):
        engine.binarize_segments(segs, 0, 100, 0, 60, 15, "sauvola", 0.34, 128.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, rows, cols, win, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        page = _page(rows, cols, seed=11)
        y0, y1 = D.band_bounds(rows, world, rank)
        band = torch.from_numpy(np.ascontiguousarray(page[y0:y1])).cuda()
        ph = D.PeerHalos(band, rows, win // 2)
        out = ph.binarize(win, "sauvola", 0.34, 128.0)
        ph.barrier()
        res = out.cpu().numpy()
        # one-shot API path as well
        out2 = D.binarize_rowbands(band, rows, win, "sauvola", 0.34, 128.0, transport="p2p")
        res2 = out2.cpu().numpy()
        ph.close()
        q.put((rank, y0, y1, res, res2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,win", [(2, 1000, 1536, 127), (3, 900, 2048, 63)])
def test_peer_halos_across_processes(world, rows, cols, win):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(i, world, port, rows, cols, win, q))
             for i in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    page = torch.from_numpy(_page(rows, cols, seed=11)).cuda()
    want, _ = engine.binarize(page, win, "sauvola", 0.34, 128.0, want_tmap=False)
    want = want.cpu().numpy()
    import oracle
    want_cpu, _ = oracle.binarize(_page(rows, cols, seed=11), win, "sauvola", 0.34, 128.0, tmap=False)
    assert np.array_equal(want, want_cpu)  # the multi-process bands are pinned to the oracle too
    for rank, y0, y1, res, res2 in got:
        assert np.array_equal(res, want[y0:y1]), rank
        assert np.array_equal(res2, want[y0:y1]), rank


def _rank_events(rank, world, port, rows, cols, win, steps, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        y0, y1 = D.band_bounds(rows, world, rank)
        band = torch.zeros((y1 - y0, cols), dtype=torch.uint8, device="cuda")
        ph = D.PeerHalos(band, rows, win // 2, events=True)
        fresh = [torch.from_numpy(np.ascontiguousarray(_page(rows, cols, seed=20 + s)[y0:y1])).cuda()
                 for s in range(steps)]
        outs = [torch.empty_like(band) for _ in range(steps)]
        torch.cuda.synchronize()
        dist.barrier()
        # every step refills the band on the stream and binarizes it; ranks are ordered by the
        # interprocess events only (no stream synchronisation inside the loop)
        for s in range(steps):
            band.copy_(fresh[s], non_blocking=True)
            ph.binarize(win, "sauvola", 0.34, 128.0, out=outs[s], sync="events")
        torch.cuda.synchronize()
        dist.barrier()
        ph.close()
        q.put((rank, y0, y1, [o.cpu().numpy() for o in outs]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,win", [(2, 600, 1536, 127), (3, 450, 1024, 31)])
def test_peer_halos_device_side_ordering(world, rows, cols, win):
    """Fresh bands every step, ranks ordered by interprocess CUDA events (publish / retire)
    instead of a stream synchronise + barrier: every step of every rank must equal the whole
    page of that step, against the CPU oracle as well as the GPU whole-page result."""
    import oracle
    import torch.multiprocessing as mp
    steps = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_events, args=(i, world, port, rows, cols, win, steps, q))
             for i in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for s in range(steps):
        page = _page(rows, cols, seed=20 + s)
        want, _ = oracle.binarize(page, win, "sauvola", 0.34, 128.0, tmap=False)
        for rank, y0, y1, outs in got:
            assert np.array_equal(outs[s], want[y0:y1]), (s, rank)
