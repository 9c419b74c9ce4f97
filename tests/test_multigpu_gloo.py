"""CPU, world_size 2 (gloo over 127.0.0.1): the N>1 data path of bench.py /
SURVEY.md §8e — every chunk split into 8-aligned slices by fy_shard_range,
each rank updates its slice (the oracle stands in for the kernel on CPU),
the updated bf16 slices are all-gathered (padded to equal size, as
all_gather_into_tensor requires) and the grad sum of squares all-reduced.
The assembled result must equal the single-rank step bit-for-bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

SIZES = [4099, 12 * 64 * 64, 8, 1000003]


def _inputs(n, k):
    rng = np.random.default_rng(20240817 + k)
    st = [rng.normal(0, 0.02, n).astype(np.float32), rng.normal(0, 1e-3, n).astype(np.float32),
          (rng.normal(0, 1e-3, n) ** 2).astype(np.float32)]
    g = torch.from_numpy(rng.normal(0, 1e-3, n).astype(np.float32)).to(torch.bfloat16)
    return st, g.view(torch.int16).numpy().view(np.uint16).copy()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_06504_b200 import optim as F
    sc = O.scalars()
    out = []
    sq_local = 0.0
    for k, n in enumerate(SIZES):
        (m0, m1, m2), g = _inputs(n, k)
        off, cnt = F.shard_range(n, world, rank, 8)
        pad = (-(-n // world) + 7) // 8 * 8
        master, mo, v = m0[off:off + cnt].copy(), m1[off:off + cnt].copy(), m2[off:off + cnt].copy()
        p = np.zeros(cnt, np.uint16)
        s, _ = O.adamw_step(master, mo, v, np.ascontiguousarray(g[off:off + cnt]), O.BF16, sc, param_out=p)
        sq_local += s
        # gloo has no 16-bit all-gather: carry the bf16 bit patterns in int32
        buf = torch.zeros(pad, dtype=torch.int32)
        buf[:cnt] = torch.from_numpy(p.astype(np.int32))
        full = torch.zeros(world * pad, dtype=torch.int32)
        dist.all_gather_into_tensor(full, buf)
        # reassemble: rank r's slice starts at shard_range(n, world, r).offset
        params = np.zeros(n, np.uint16)
        for r in range(world):
            o, c = F.shard_range(n, world, r, 8)
            params[o:o + c] = full[r * pad:r * pad + c].numpy().astype(np.uint16)
        out.append(params)
    t = torch.tensor([sq_local], dtype=torch.float64)
    dist.all_reduce(t)
    if rank == 0:
        q.put(([p.tolist() for p in out], float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_step_equals_single_rank():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    import queue
    import time
    deadline = time.time() + 240
    while True:
        try:
            params, sq = q.get(timeout=2)
            break
        except queue.Empty:
            assert all(p.exitcode in (None, 0) for p in procs), "a rank died"
            assert time.time() < deadline, "timeout"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = O.scalars()
    sq_ref = 0.0
    for k, n in enumerate(SIZES):
        (m0, m1, m2), g = _inputs(n, k)
        p = np.zeros(n, np.uint16)
        s, _ = O.adamw_step(m0, m1, m2, g, O.BF16, sc, param_out=p)
        sq_ref += s
        assert np.array_equal(np.array(params[k], dtype=np.uint16), p), f"chunk {k}"
    assert abs(sq - sq_ref) <= 1e-12 * sq_ref
