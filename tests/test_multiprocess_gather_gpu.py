"""GPU, two processes on one B200 (the N>1 fused path without a second GPU):
each process owns one rank's full-param buffer; the buffers are exchanged as
CUDA IPC handles (torch.multiprocessing), so every rank holds a device
pointer into the OTHER process's memory — what torch symmetric memory hands
bench.py on a multi-GPU node, with the NVLink hop replaced by the same
device. Each rank updates its fy_shard_range slice with
fy_adamw_chunk_gather, storing the bf16 result into both processes'
buffers; after a barrier both full buffers must equal the single-rank
oracle result bit for bit."""
import os
import queue
import socket
import time

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu

N = 3 * 2048 * 17 + 40  # whole tiles + a ragged tail per slice


def _inputs():
    rng = np.random.default_rng(20240817 + 5)
    master = rng.normal(0, 0.02, N).astype(np.float32)
    m = rng.normal(0, 1e-3, N).astype(np.float32)
    v = (rng.normal(0, 1e-3, N) ** 2).astype(np.float32)
    g = torch.from_numpy(rng.normal(0, 1e-3, N).astype(np.float32)).to(torch.bfloat16)
    return master, m, v, g


def _worker(rank, world, port, qs, results):
    import sys
    sys.path.insert(0, os.getcwd())
    import torch.distributed as dist
    from paper_2403_06504_b200 import optim as F
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda:0")
    full = torch.zeros(N, dtype=torch.bfloat16, device=dev)
    torch.cuda.synchronize()
    # exchange the buffers as CUDA IPC handles
    for r in range(world):
        if r != rank:
            qs[r].put((rank, full))
    peers = {rank: full}
    for _ in range(world - 1):
        src, t = qs[rank].get(timeout=120)
        peers[src] = t
    dist.barrier()
    master, m, v, g = _inputs()
    off, cnt = F.shard_range(N, world, rank, 8)
    sl = slice(off, off + cnt)
    dm = torch.from_numpy(master[sl].copy()).to(dev)
    dmm = torch.from_numpy(m[sl].copy()).to(dev)
    dvv = torch.from_numpy(v[sl].copy()).to(dev)
    dg = g[sl].clone().to(dev)
    local = torch.zeros(cnt, dtype=torch.bfloat16, device=dev)
    F.adamw_chunk_gather(dm, dmm, dvv, dg, F.Hparams(), local,
                         [peers[r].data_ptr() + 2 * off for r in range(world)])
    torch.cuda.synchronize()
    dist.barrier()  # every rank's peer stores have landed everywhere
    results.put((rank, full.cpu().view(torch.int16).numpy().view(np.uint16).copy()))
    dist.barrier()  # keep the IPC-shared buffers alive until all ranks copied
    dist.destroy_process_group()


def test_two_process_fused_gather_over_ipc(cuda_dev):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    ctx = mp.get_context("spawn")
    qs = [ctx.Queue() for _ in range(world)]
    results = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, qs, results)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    deadline = time.time() + 300
    while len(got) < world:
        try:
            r, arr = results.get(timeout=2)
            got[r] = arr
        except queue.Empty:
            assert all(p.exitcode in (None, 0) for p in procs), "a rank died"
            assert time.time() < deadline, "timeout"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    master, m, v, g = _inputs()
    op = np.zeros(N, np.uint16)
    O.adamw_step(master, m, v, g.view(torch.int16).numpy().view(np.uint16).copy(), O.BF16, O.scalars(),
                 param_out=op)
    for r in range(world):
        assert np.array_equal(got[r], op), f"rank {r}'s full buffer differs"
