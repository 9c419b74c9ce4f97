"""GPU: the sharded optimizer step through the library entry point
(fy_shard_*) against the CPU oracle.

Every chunk is split into `world` slices (fy_shard_range, 8-aligned); each
rank updates its slice and the updated bf16 params are all-gathered into
every rank's arena. Results must equal the single-GPU oracle step of the
WHOLE chunk bit for bit: every rank's states slice, every rank's full
params, and the global grad norm (the per-rank sums are added in a
different order than the oracle's element order: rel 2e-7, the fused
kernel's measured precision bar, test_adamw_gpu.test_grad_norm_precision).

One GPU is available, so world > 1 runs as W shards on the same device —
in one process (fy_shard_connect_ptrs, each shard's step on its own
stream) and in two processes (CUDA IPC handles, fy_shard_connect) — with
the PEER gather (fused epilogue peer stores / copy-engine pushes + device
barriers). NCCL runs on a one-rank communicator (the same calls as at
world > 1; NCCL refuses two ranks on one GPU)."""
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

SIZES = [1 << 20, 3 * 2048 * 17 + 40, 4099, 777777, 8]


class _CAI:
    """A raw device pointer as a torch tensor (no copy)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = dict(shape=(n,), typestr=typestr, data=(ptr, False), version=3)


def dev_u16(ptr, n):
    return torch.as_tensor(_CAI(ptr, n, "<u2"), device="cuda")


def _inputs(sizes, seed=0):
    out = []
    for k, n in enumerate(sizes):
        rng = np.random.default_rng(20240817 + 100 * seed + k)
        master = rng.normal(0, 0.02, n).astype(np.float32)
        m = rng.normal(0, 1e-3, n).astype(np.float32)
        v = (rng.normal(0, 1e-3, n) ** 2).astype(np.float32)
        g = [torch.from_numpy(rng.normal(0, 1e-3, n).astype(np.float32)).to(torch.bfloat16)
             .view(torch.int16).numpy().view(np.uint16).copy() for _ in range(2)]
        out.append(dict(master=master, m=m, v=v, g=g))
    return out


def _oracle(inp, steps):
    """Whole-chunk oracle trajectory with DeepSpeed's step counter (one
    increment per chunk); returns per chunk (master, m, v, params) and the
    per-step grad sums of squares."""
    st = [dict(master=c["master"].copy(), m=c["m"].copy(), v=c["v"].copy(),
               p=np.zeros(c["master"].size, np.uint16)) for c in inp]
    k = O.StepCounter()
    sqs = []
    for i, step in enumerate(steps):
        sq = 0.0
        for c, s in zip(inp, st):
            sc = O.scalars_bt(*k.next(step))
            q, _ = O.adamw_step(s["master"], s["m"], s["v"], c["g"][i], O.BF16, sc, param_out=s["p"])
            sq += q
        sqs.append(sq)
    return st, sqs


def _shard_buffers(F, shard, inp, dev, tier):
    """This rank's slice of every chunk: states [master|m|v] (device or
    pinned host) and grads per step (device)."""
    bufs = []
    for c, x in enumerate(inp):
        sl = shard.slice(c)
        a, b = sl["offset"], sl["offset"] + sl["count"]
        st = np.concatenate([x["master"][a:b], x["m"][a:b], x["v"][a:b]])
        t = torch.from_numpy(st)
        t = t.to(dev) if tier == "device" else t.pin_memory()
        grads = [torch.from_numpy(g[a:b].view(np.int16).copy()).view(torch.bfloat16).to(dev) for g in x["g"]]
        bufs.append(dict(states=t, grads=grads, off=a, cnt=b - a))
    return bufs


def _io(bufs, i):
    return [dict(states=b["states"].data_ptr() if b["cnt"] else None,
                 grad=b["grads"][i].data_ptr() if b["cnt"] else None) for b in bufs]


def _check(F, shards, bufs_per_rank, ref, inp):
    for r, (sh, bufs) in enumerate(zip(shards, bufs_per_rank)):
        for c, (b, x) in enumerate(zip(bufs, ref)):
            n = inp[c]["master"].size
            got = dev_u16(sh.slice(c)["params"], n).cpu().numpy()
            assert np.array_equal(got, x["p"]), f"rank {r} chunk {c}: full params differ"
            a, cnt = b["off"], b["cnt"]
            st = b["states"].cpu().numpy()
            for j, key in enumerate(("master", "m", "v")):
                assert np.array_equal(st[j * cnt:(j + 1) * cnt].view(np.uint32),
                                      x[key][a:a + cnt].view(np.uint32)), f"rank {r} chunk {c} {key}"


@pytest.mark.parametrize("tier", ["device", "host"])
@pytest.mark.parametrize("nccl", [False, True])
def test_shard_world1_matches_oracle(cuda_dev, tier, nccl):
    from paper_2403_06504_b200 import optim as F
    inp = _inputs(SIZES)
    kw = dict(gather="nccl", nccl_id=F.nccl_unique_id()) if nccl else {}
    sh = F.Shard(SIZES, tier=tier, piece_elems=300000 if tier == "host" else 0, **kw)
    bufs = _shard_buffers(F, sh, inp, cuda_dev, tier)
    steps = (10, 11)
    ref, sqs = _oracle(inp, steps)
    for i, step in enumerate(steps):
        sh.step(_io(bufs, i), F.Hparams(step=step), want_grad_norm=True)
        sq, bad = sh.wait()
        assert bad == 0
        assert abs(sq - sqs[i]) <= 2e-7 * sqs[i]
    torch.cuda.synchronize()
    _check(F, [sh], [bufs], ref, inp)
    st = sh.stats()
    assert st["world"] == 1 and st["step_ms"] > 0
    if tier == "host":
        n = sum(SIZES)
        assert st["h2d_bytes"] == 12 * n and st["d2h_bytes"] == 12 * n
    sh.close()


@pytest.mark.parametrize("world,tier", [(2, "device"), (3, "device"), (4, "device"),
                                        (2, "host"), (3, "host")])
def test_shard_single_process_peer(cuda_dev, world, tier):
    """W shards in one process on one GPU, arenas exchanged as pointers,
    fused peer-store gather (device tier) / copy-engine pushes (host tier),
    device barriers; each shard's step on its own stream."""
    single_process_peer(torch.device("cuda:0"), world, tier)


def test_shard_single_process_peer_world8(cuda_dev):
    """World 8 in one process on one GPU: 8 shards x (caller, update, comm)
    streams exceed the default 8 hardware queues (CUDA_DEVICE_MAX_CONNECTIONS),
    and streams that share a queue serialise — a spinning device barrier
    would then block the peer it waits for. One process per GPU (the
    deployment) never shares queues; a process driving many shards on one
    device raises the connection count, as this subprocess does."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32",
               PYTHONPATH=f"{root}:{root / 'tests'}:" + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c",
                        "import torch, test_shard_gpu as t; t.single_process_peer(torch.device('cuda:0'), 8, 'device');"
                        "print('OK')"], env=env, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-3000:]


def _raw_streams(n):
    """Caller streams made with the runtime directly: torch.cuda.Stream()
    would initialise torch's pools (32 streams per priority) and, past
    CUDA_DEVICE_MAX_CONNECTIONS hardware queues, streams share a queue — a
    spinning device barrier then blocks the very peer it waits for."""
    from cuda.bindings import runtime as rt
    out = []
    for _ in range(n):
        err, h = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
        assert err == rt.cudaError_t.cudaSuccess, err
        out.append(torch.cuda.ExternalStream(int(h)))
    return out


def single_process_peer(cuda_dev, world, tier):
    from paper_2403_06504_b200 import optim as F
    inp = _inputs(SIZES, seed=world)
    shards = [F.Shard(SIZES, world=world, rank=r, gather="peer", tier=tier,
                      piece_elems=100000 if tier == "host" else 0) for r in range(world)]
    arenas = [s.arena() for s in shards]
    for s in shards:
        s.connect_ptrs(arenas)
    bufs = [_shard_buffers(F, s, inp, cuda_dev, tier) for s in shards]
    streams = _raw_streams(len(shards))
    steps = (10, 11)
    ref, sqs = _oracle(inp, steps)
    for i, step in enumerate(steps):
        for s, b, st in zip(shards, bufs, streams):
            s.step(_io(b, i), F.Hparams(step=step), want_grad_norm=True, stream=st)
        got = [s.wait() for s in shards]
        for sq, bad in got:
            assert bad == 0
            assert abs(sq - sqs[i]) <= 2e-7 * sqs[i]
        # every rank sums the per-rank partials in rank order: identical
        assert len({g[0] for g in got}) == 1
    torch.cuda.synchronize()
    _check(F, shards, bufs, ref, inp)
    st = shards[0].stats()
    assert st["gather"] == 2 and st["gather_bytes"] > 0
    for s in shards:
        s.close()


def test_shard_validation(cuda_dev):
    from paper_2403_06504_b200 import optim as F
    from paper_2403_06504_b200._lib import FyError
    with pytest.raises(FyError, match="gather"):
        F.Shard([1024], world=2, rank=0)
    with pytest.raises(FyError, match="nccl_id"):
        F.Shard([1024], world=2, rank=0, gather="nccl")
    with pytest.raises(FyError, match="rank"):
        F.Shard([1024], world=2, rank=2, gather="peer")
    sh = F.Shard([1024, 4096], world=2, rank=1, gather="peer")
    with pytest.raises(FyError, match="connect"):
        sh.step([dict(states=1, grad=1)] * 2, F.Hparams())
    sh.close()


def _worker(rank, world, port, tier, results):
    import sys
    sys.path.insert(0, os.getcwd())
    import torch.distributed as dist
    from paper_2403_06504_b200 import optim as F
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    sh = F.Shard(SIZES, world=world, rank=rank, gather="peer", tier=tier,
                 piece_elems=200000 if tier == "host" else 0)
    handles = [None] * world
    dist.all_gather_object(handles, sh.ipc_handle())
    sh.connect(handles)
    inp = _inputs(SIZES, seed=7)
    bufs = _shard_buffers(F, sh, inp, dev, tier)
    sqs = []
    for i, step in enumerate((10, 11)):
        sh.step(_io(bufs, i), F.Hparams(step=step), want_grad_norm=True)
        sqs.append(sh.wait()[0])
    torch.cuda.synchronize()
    params = [dev_u16(sh.slice(c)["params"], n).cpu().numpy().copy() for c, n in enumerate(SIZES)]
    states = [(b["off"], b["cnt"], b["states"].cpu().numpy().copy()) for b in bufs]
    results.put((rank, params, states, sqs))
    dist.barrier()  # keep the arenas mapped until every rank has read its own
    sh.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("tier", ["device", "host"])
def test_shard_two_processes_ipc(cuda_dev, tier):
    """Two processes (ranks) on one GPU through fy_shard_ipc_handle /
    fy_shard_connect — the product path a multi-GPU node runs per GPU."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tier, results)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    deadline = time.time() + 400
    while len(got) < world:
        try:
            r, *rest = results.get(timeout=2)
            got[r] = rest
        except queue.Empty:
            assert all(p.exitcode in (None, 0) for p in procs), "a rank died"
            assert time.time() < deadline, "timeout"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    inp = _inputs(SIZES, seed=7)
    ref, sqs = _oracle(inp, (10, 11))
    for r in range(world):
        params, states, rsq = got[r]
        for c, x in enumerate(ref):
            assert np.array_equal(params[c], x["p"]), f"rank {r} chunk {c} params"
            a, cnt, st = states[c]
            for j, key in enumerate(("master", "m", "v")):
                assert np.array_equal(st[j * cnt:(j + 1) * cnt].view(np.uint32), x[key][a:a + cnt].view(np.uint32))
        for q, qr in zip(rsq, sqs):
            assert abs(q - qr) <= 2e-7 * qr
    assert got[0][2] == got[1][2]  # the same global norm on both ranks


@pytest.mark.parametrize("world", [1, 2, 3])
def test_shard_in_place_gradients_in_the_arena(cuda_dev, world):
    """The reference's in-place convention on the product path (what the
    bench's headline and INTEGRATION.md §4 do): each rank lands its slice's
    gradients in its own slot of the chunk's arena region (own_params) and
    the update overwrites them with the params — then the gather fills the
    other slots. Two consecutive steps (the second step's grads written into
    the slot again), bit-exact vs the oracle in every rank's arena."""
    from paper_2403_06504_b200 import optim as F
    inp = _inputs(SIZES, seed=40 + world)
    shards = [F.Shard(SIZES, world=world, rank=r, gather="peer" if world > 1 else None, tier="device")
              for r in range(world)]
    if world > 1:
        arenas = [s.arena() for s in shards]
        for s in shards:
            s.connect_ptrs(arenas)
    bufs = [_shard_buffers(F, s, inp, cuda_dev, "device") for s in shards]
    streams = _raw_streams(world)
    steps = (10, 11)
    ref, sqs = _oracle(inp, steps)
    for i, step in enumerate(steps):
        ios = []
        for s, b in zip(shards, bufs):
            io = []
            for c, bb in enumerate(b):
                slot = s.own_params(c)
                if bb["cnt"]:
                    slot.copy_(bb["grads"][i])  # the gradients land in the arena slot
                io.append(dict(states=bb["states"].data_ptr() if bb["cnt"] else None,
                               grad=slot.data_ptr() if bb["cnt"] else None))
            ios.append(io)
        torch.cuda.synchronize()
        for s, io, st in zip(shards, ios, streams):
            s.step(io, F.Hparams(step=step), want_grad_norm=True, stream=st)
        for s in shards:
            sq, bad = s.wait()
            assert bad == 0 and abs(sq - sqs[i]) <= 2e-7 * sqs[i]
    torch.cuda.synchronize()
    _check(F, shards, bufs, ref, inp)
    for s in shards:
        s.close()


@pytest.mark.parametrize("world", [1, 2])
def test_shard_host_gradients_device_states(cuda_dev, world):
    """grads_on_host: HBM-resident states, the slice's gradients in pinned
    HOST memory (H2D through the shard's chunk pipeline) and the updated
    params D2H into the SAME host buffer (the e2e contract: host grads in,
    host params out), plus the all-gather into every rank's arena. Two
    steps, bit-exact vs the oracle: arena params, device states and the
    host buffer (the rank's own slice of the params)."""
    from paper_2403_06504_b200 import optim as F
    inp = _inputs(SIZES, seed=60 + world)
    shards = [F.Shard(SIZES, world=world, rank=r, gather="peer" if world > 1 else None, tier="device",
                      grads_on_host=True, params_to_host=True) for r in range(world)]
    if world > 1:
        arenas = [s.arena() for s in shards]
        for s in shards:
            s.connect_ptrs(arenas)
    bufs = [_shard_buffers(F, s, inp, cuda_dev, "device") for s in shards]
    host = [[torch.empty(max(b["cnt"], 1), dtype=torch.bfloat16).pin_memory() for b in bb] for bb in bufs]
    streams = _raw_streams(world)
    steps = (10, 11)
    ref, sqs = _oracle(inp, steps)
    for i, step in enumerate(steps):
        ios = []
        for bb, hh in zip(bufs, host):
            io = []
            for b, h in zip(bb, hh):
                if b["cnt"]:
                    h[:b["cnt"]].copy_(b["grads"][i].cpu())   # this step's grads, host side
                io.append(dict(states=b["states"].data_ptr() if b["cnt"] else None,
                               grad=h.data_ptr() if b["cnt"] else None,
                               h_param=h.data_ptr() if b["cnt"] else None))
            ios.append(io)
        for s, io, st in zip(shards, ios, streams):
            s.step(io, F.Hparams(step=step), want_grad_norm=True, stream=st)
        for s in shards:
            sq, bad = s.wait()
            assert bad == 0 and abs(sq - sqs[i]) <= 2e-7 * sqs[i]
        st = shards[0].stats()
        n_own = sum(b["cnt"] for b in bufs[0])
        assert st["h2d_bytes"] == 2 * n_own and st["d2h_bytes"] == 2 * n_own
    torch.cuda.synchronize()
    _check(F, shards, bufs, ref, inp)
    for r, (bb, hh) in enumerate(zip(bufs, host)):
        for c, (b, h) in enumerate(zip(bb, hh)):
            if b["cnt"]:
                own = ref[c]["p"][b["off"]:b["off"] + b["cnt"]]
                assert np.array_equal(h[:b["cnt"]].view(torch.int16).numpy().view(np.uint16), own), (r, c)
    for s in shards:
        s.close()


def test_shard_fp16_loss_scaled(cuda_dev):
    """DeepSpeed's fp16 mode through the sharded step: fp16 gradients at a
    loss scale of 2^16 (grad_scale 2^-16), fp16 params gathered into every
    rank's arena; W = 2 in one process, two steps, bit-exact vs the oracle
    (same unscale arithmetic) in states and params."""
    from paper_2403_06504_b200 import optim as F
    sizes = [4099, 3 * 2048 * 17 + 40, 8]
    world, scale = 2, 2.0 ** -16
    rng = np.random.default_rng(20240901)
    inp = []
    for n in sizes:
        g = [torch.from_numpy((rng.normal(0, 1e-3, n) / scale).astype(np.float32)).to(torch.float16)
             .view(torch.int16).numpy().view(np.uint16).copy() for _ in range(2)]
        inp.append(dict(master=rng.normal(0, 0.02, n).astype(np.float32),
                        m=rng.normal(0, 1e-3, n).astype(np.float32),
                        v=(rng.normal(0, 1e-3, n) ** 2).astype(np.float32), g=g))
    # oracle: whole chunks, DeepSpeed counter, fp16 grads / params
    ref = [dict(master=c["master"].copy(), m=c["m"].copy(), v=c["v"].copy(), p=np.zeros(c["master"].size, np.uint16))
           for c in inp]
    k = O.StepCounter()
    steps = (10, 11)
    for i, step in enumerate(steps):
        for c, r in zip(inp, ref):
            O.adamw_step(r["master"], r["m"], r["v"], c["g"][i], O.FP16, O.scalars_bt(*k.next(step)),
                         grad_scale=scale, param_out=r["p"], param_dtype=O.FP16)
    shards = [F.Shard(sizes, world=world, rank=r, gather="peer", tier="device", grad_dtype=torch.float16,
                      param_dtype=torch.float16) for r in range(world)]
    arenas = [s.arena() for s in shards]
    for s in shards:
        s.connect_ptrs(arenas)
    bufs = []
    for s in shards:
        b = []
        for c, x in enumerate(inp):
            sl = s.slice(c)
            a, e = sl["offset"], sl["offset"] + sl["count"]
            st = torch.from_numpy(np.concatenate([x["master"][a:e], x["m"][a:e], x["v"][a:e]])).to(cuda_dev)
            gr = [torch.from_numpy(g[a:e].view(np.int16).copy()).view(torch.float16).to(cuda_dev) for g in x["g"]]
            b.append(dict(states=st, grads=gr, off=a, cnt=e - a))
        bufs.append(b)
    streams = _raw_streams(world)
    for i, step in enumerate(steps):
        for s, b, st in zip(shards, bufs, streams):
            s.step(_io(b, i), F.Hparams(step=step, grad_scale=scale), stream=st)
        for s in shards:
            s.wait()
    torch.cuda.synchronize()
    _check(F, shards, bufs, ref, inp)
    for s in shards:
        s.close()
