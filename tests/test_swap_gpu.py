"""GPU: the activation swap engine (fy_swapper_*, include/fuyou/fy_adam.h) —
the GPU -> pinned host (-> SSD) copy path of the reference's activation swap
tasks (proj/src/task_graph.cpp:296-321,357-397) as a standalone component.
Bar: every swapped-in buffer equals the swapped-out one byte for byte, for
CPU and SSD placement, sizes off the 4 KiB grid, buffers larger than one
ring slot, many handles in flight, and event ordering with the caller."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pattern(nbytes, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    return torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev, generator=g)


@pytest.mark.parametrize("placement", ["cpu", "ssd"])
def test_swap_round_trip_many_handles(cuda_dev, tmp_path, placement):
    from paper_2403_06504_b200 import optim as F
    sw = F.Swapper(slot_bytes=1 << 20, slots=3, file_dir=str(tmp_path))
    pl = F.Swapper.CPU if placement == "cpu" else F.Swapper.SSD
    sizes = [4096, 12345, (1 << 20) + 17, 5 * (1 << 20) + 4093, 3 << 20]
    src = [_pattern(n, 100 + i, cuda_dev) for i, n in enumerate(sizes)]
    dst = [torch.zeros_like(t) for t in src]
    # the swapper's streams do not follow torch's: without `ready` events the
    # caller makes its producers (and the zero-fill of dst) complete first
    torch.cuda.synchronize()
    handles = [sw.swap_out(t, pl) for t in src]
    for h, t in zip(reversed(handles), reversed(dst)):  # backward order, like the schedule
        sw.swap_in(h, t)
    sw.sync()
    for a, b in zip(src, dst):
        assert torch.equal(a, b)
    st = sw.stats()
    if pl == F.Swapper.SSD:
        assert st["file_bytes"] >= sum(sizes) and st["io_engine"] in ("io_uring", "pread/pwrite")
    else:
        assert st["host_bytes"] >= sum(sizes)
    for h in handles:
        sw.release(h)
    assert sw.stats()["file_bytes"] == 0
    sw.close()


@pytest.mark.parametrize("placement", ["cpu", "ssd"])
def test_swap_event_ordering(cuda_dev, tmp_path, placement):
    """The producer writes the activation late on its own stream; swap_out
    must wait on `ready`. The consumer overwrites the source as soon as
    `src_free` fires and reads the restored buffer after `done`."""
    from paper_2403_06504_b200 import optim as F
    sw = F.Swapper(slot_bytes=1 << 20, slots=2, file_dir=str(tmp_path))
    pl = F.Swapper.CPU if placement == "cpu" else F.Swapper.SSD
    n = 3 * (1 << 20) + 100
    want = _pattern(n, 7, cuda_dev)
    act = torch.zeros(n, dtype=torch.uint8, device=cuda_dev)
    prod = torch.cuda.Stream()
    ready, src_free, done = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
    for e in (src_free, done):
        e.record()  # torch creates CUDA events lazily
    torch.cuda.synchronize()
    with torch.cuda.stream(prod):
        torch.cuda._sleep(30_000_000)
        act.copy_(want)
        ready.record(prod)
    h = sw.swap_out(act, pl, ready=ready, src_free=src_free)
    with torch.cuda.stream(prod):
        prod.wait_event(src_free)
        act.fill_(0)  # the device buffer is reused for something else
    back = torch.zeros(n, dtype=torch.uint8, device=cuda_dev)
    back_ready = torch.cuda.Event()
    back_ready.record()  # the zero-fill of `back` is queued on torch's stream
    sw.swap_in(h, back, ready=back_ready, done=done)
    cons = torch.cuda.Stream()
    cons.wait_event(done)
    with torch.cuda.stream(cons):
        snap = back.clone()
    torch.cuda.synchronize()
    sw.sync()
    assert torch.equal(snap, want)
    sw.release(h)
    sw.close()


def test_swap_rejects_bad_use(cuda_dev, tmp_path):
    from paper_2403_06504_b200 import optim as F
    from paper_2403_06504_b200._lib import FyError
    sw = F.Swapper(file_dir=str(tmp_path))
    t = torch.zeros(16, dtype=torch.uint8, device=cuda_dev)
    with pytest.raises(FyError):
        sw.swap_in(12345, t)
    with pytest.raises(FyError):
        sw.release(999)
    with pytest.raises(FyError):
        sw.swap_out(t, 7)
    sw.close()
    with pytest.raises(FyError):
        F.Swapper(slots=1)


def test_swap_reports_unusable_swap_dir(cuda_dev):
    """Fault injection: an SSD swap into a directory that does not exist is a
    reported error (FY_ERR_DEVICE), and CPU placement keeps working."""
    from paper_2403_06504_b200 import optim as F
    from paper_2403_06504_b200._lib import FyError
    sw = F.Swapper(file_dir="/nonexistent/fy_swap_dir")
    t = torch.arange(4096, dtype=torch.int32, device=cuda_dev).view(torch.uint8)
    torch.cuda.synchronize()
    with pytest.raises(FyError):
        sw.swap_out(t, F.Swapper.SSD)
    h = sw.swap_out(t, F.Swapper.CPU)
    back = torch.zeros_like(t)
    torch.cuda.synchronize()
    sw.swap_in(h, back)
    sw.sync()
    assert torch.equal(back, t)
    sw.close()


def test_swap_ssd_striped_over_directories(cuda_dev, tmp_path):
    """SSD placement with file_dir = "d0:d1:d2" (one directory per SSD): the
    swap file is striped RAID-0 over the three in 4 MiB units — every
    directory holds data, and every buffer comes back byte for byte."""
    import os
    from paper_2403_06504_b200 import optim as F
    from paper_2403_06504_b200._lib import FyError
    dirs = [tmp_path / f"ssd{i}" for i in range(3)]
    for d in dirs:
        d.mkdir()
    sw = F.Swapper(slot_bytes=8 << 20, slots=3, file_dir=":".join(str(d) for d in dirs))
    sizes = [4096, (8 << 20) + 4093, 21 << 20, 12345]
    src = [_pattern(n, 300 + i, cuda_dev) for i, n in enumerate(sizes)]
    dst = [torch.zeros_like(t) for t in src]
    torch.cuda.synchronize()
    handles = [sw.swap_out(t, F.Swapper.SSD) for t in src]
    sw.sync()
    for d in dirs:
        files = list(d.iterdir())
        assert len(files) == 1 and os.path.getsize(files[0]) > 0, d
    for h, t in zip(handles, dst):
        sw.swap_in(h, t)
    sw.sync()
    for a, b in zip(src, dst):
        assert torch.equal(a, b)
    for h in handles:
        sw.release(h)
    sw.close()
    for bad in (":", f"{dirs[0]}:{dirs[0]}"):
        with pytest.raises(FyError):
            F.Swapper(slot_bytes=1 << 20, slots=2, file_dir=bad)
