"""GPU parity + ordering of the streamed (out-of-core) optimizer step
(fy_pipeline_*): host-resident [master|m|v] per chunk, H2D -> fused Adam ->
D2H, against the CPU oracle; and the executed timeline against the
reference's optimizer-block dependencies (task_graph.cpp:453-503): read gate
depth 2, update after its read, write-back after its update, slot reuse
after the previous write-back."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _bits_equal(x, y):
    return bool(np.array_equal(x.view(np.uint32), y.view(np.uint32)))


def _make_chunks(sizes, seed, dev, grads_on_host):
    chunks, ref = [], []
    for k, n in enumerate(sizes):
        rng = np.random.default_rng(20240817 + seed + k)
        st = np.empty(3 * n, np.float32)
        st[:n] = rng.normal(0, 0.02, n)
        st[n:2 * n] = rng.normal(0, 1e-3, n)
        st[2 * n:] = rng.normal(0, 1e-3, n) ** 2
        g = torch.from_numpy(rng.normal(0, 1e-3, n).astype(np.float32)).to(torch.bfloat16)
        h_states = torch.from_numpy(st.copy()).pin_memory()
        h_param = torch.zeros(n, dtype=torch.bfloat16).pin_memory()
        grad = g.pin_memory() if grads_on_host else g.to(dev)
        chunks.append(dict(n=n, h_states_t=h_states, grad_t=grad, h_param_t=h_param))
        ref.append(dict(states=st, grad=g.view(torch.int16).numpy().view(np.uint16).copy()))
    return chunks, ref


def _desc(chunks):
    return [dict(n=c["n"], h_states=c["h_states_t"].data_ptr(), grad=c["grad_t"].data_ptr(),
                 h_param=c["h_param_t"].data_ptr()) for c in chunks]


@pytest.mark.parametrize("grads_on_host,slots", [(False, 3), (True, 2), (False, 4)])
def test_pipeline_matches_oracle(cuda_dev, grads_on_host, slots):
    from paper_2403_06504_b200 import optim as F
    sizes = [1 << 20, (1 << 20) + 3, 4099, 777777, 1 << 19, 8]
    chunks, ref = _make_chunks(sizes, 1, cuda_dev, grads_on_host)
    pipe = F.ChunkPipeline(max(sizes), slots=slots, grads_on_host=grads_on_host)
    sq_total = 0.0
    counter = O.StepCounter()  # the pipeline keeps DeepSpeed's step counter
    for step in (10, 11):
        hp = F.Hparams(step=step)
        pipe.step(_desc(chunks), hp, want_grad_norm=True)
        sq, bad = pipe.wait()
        assert bad == 0
        sq_ref = 0.0
        for r in ref:
            sc = O.scalars_bt(*counter.next(step))
            n = r["grad"].size
            st = r["states"]
            r["param"] = np.zeros(n, np.uint16)
            mst, mm, vv = st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy()
            s, _ = O.adamw_step(mst, mm, vv, r["grad"], O.BF16, sc, param_out=r["param"])
            sq_ref += s
            r["states"] = np.concatenate([mst, mm, vv])
        assert abs(sq - sq_ref) <= 2e-7 * sq_ref
        for c, r in zip(chunks, ref):
            assert _bits_equal(c["h_states_t"].numpy(), r["states"])
            assert np.array_equal(c["h_param_t"].view(torch.int16).numpy().view(np.uint16),
                                  r["param"])
        tim, total = pipe.timings(len(sizes))
        assert total > 0
        for i, t in enumerate(tim):
            assert t["upd"][0] >= t["h2d"][1], "update before its state read"
            assert t["d2h"][0] >= t["upd"][1], "write-back before its update"
            if i >= 2:
                assert t["h2d"][0] >= tim[i - 2]["upd"][1], "read gate (depth 2) violated"
            if i >= slots:
                assert t["h2d"][0] >= tim[i - slots]["d2h"][1], "slot reused before write-back"
    pipe.close()


def test_pipeline_rejects_bad_args(cuda_dev):
    from paper_2403_06504_b200 import optim as F
    from paper_2403_06504_b200._lib import FyError
    pipe = F.ChunkPipeline(1024, slots=2)
    with pytest.raises(FyError):
        pipe.step([dict(n=4096, h_states=1, grad=1, h_param=1)], F.Hparams())
    with pytest.raises(FyError):
        pipe.wait()
    pipe.close()
    with pytest.raises(FyError):
        F.ChunkPipeline(1024, slots=1)


def test_pipeline_waits_for_grad_ready_events(cuda_dev):
    """Each chunk's update must wait on its producer's event (the backward
    that writes the grads): the grads are written late on a
    side stream (after a ~50 ms spin); reading them early would use zeros."""
    from paper_2403_06504_b200 import optim as F
    sizes = [1 << 20, (1 << 20) + 5, 65536]
    chunks, ref = _make_chunks(sizes, 7, cuda_dev, grads_on_host=False)
    late = [c["grad_t"].clone() for c in chunks]
    for c in chunks:
        c["grad_t"].zero_()
    side = torch.cuda.Stream()
    evs = []
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        for c, g in zip(chunks, late):
            torch.cuda._sleep(50_000_000)
            c["grad_t"].copy_(g)
            e = torch.cuda.Event()
            e.record(side)
            evs.append(e)
    desc = _desc(chunks)
    for d, e in zip(desc, evs):
        d["grad_ready"] = e.cuda_event
    pipe = F.ChunkPipeline(max(sizes), slots=2)
    pipe.step(desc, F.Hparams(step=10))
    pipe.wait()
    sc = O.scalars(step=10)
    for c, r in zip(chunks, ref):
        n = r["grad"].size
        st = r["states"]
        mst, mm, vv = st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy()
        O.adamw_step(mst, mm, vv, r["grad"], O.BF16, sc)
        assert _bits_equal(c["h_states_t"].numpy(), np.concatenate([mst, mm, vv]))
    pipe.close()


def test_pipeline_resident_states_host_grads_device_param_copy(cuda_dev):
    """The e2e configuration of bench.py (and its N>1 form): states in HBM,
    bf16 grads read from pinned host memory, params written back over the
    grads in host memory AND kept on the device (chunk.d_param, the rank's
    slice of the full-param buffer that the all-gather then fills)."""
    from paper_2403_06504_b200 import optim as F
    sizes = [1 << 20, 4099, (1 << 18) + 8]
    chunks, ref = _make_chunks(sizes, 11, cuda_dev, grads_on_host=True)
    d_states = [c["h_states_t"].to(cuda_dev) for c in chunks]
    d_params = [torch.zeros(c["n"], dtype=torch.bfloat16, device=cuda_dev) for c in chunks]
    pipe = F.ChunkPipeline(max(sizes), slots=3, grads_on_host=True, params_to_host=True,
                           keep_params_on_device=True, states_on_device=True)
    desc = [dict(n=c["n"], h_states=s.data_ptr(), grad=c["grad_t"].data_ptr(),
                 h_param=c["grad_t"].data_ptr(), d_param=p.data_ptr())
            for c, s, p in zip(chunks, d_states, d_params)]
    pipe.step(desc, F.Hparams(step=10))
    pipe.wait()
    sc = O.scalars(step=10)
    for c, s, p, r in zip(chunks, d_states, d_params, ref):
        n = r["grad"].size
        st = r["states"]
        mst, mm, vv = st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy()
        op = np.zeros(n, np.uint16)
        O.adamw_step(mst, mm, vv, r["grad"], O.BF16, sc, param_out=op)
        assert _bits_equal(s.cpu().numpy(), np.concatenate([mst, mm, vv]))
        assert np.array_equal(p.cpu().view(torch.int16).numpy().view(np.uint16), op)
        assert np.array_equal(c["grad_t"].view(torch.int16).numpy().view(np.uint16), op)
    pipe.close()


def test_numa_local_pinned_host_memory(cuda_dev):
    """fy_host_alloc places the host tier on the GPU's NUMA node (PCI sysfs)
    and page-locks it: the pages report that node (move_pages) when the
    platform has one, and copies to / from it are page-locked DMA (the
    pipeline's bit-exact results above run on these buffers)."""
    import ctypes as C
    from paper_2403_06504_b200._lib import LIB, check
    node = C.c_int()
    check(LIB.fy_device_numa_node(0, C.byref(node)))
    p = C.c_void_p()
    n = 64 << 20
    check(LIB.fy_host_alloc(n, C.byref(p)))
    try:
        got = C.c_int()
        check(LIB.fy_host_numa_node(p, C.byref(got)))
        if node.value >= 0:
            assert got.value == node.value
        host = torch.frombuffer((C.c_uint8 * n).from_address(p.value), dtype=torch.uint8)
        host[:] = 7
        d = host.to(cuda_dev, non_blocking=True)
        torch.cuda.synchronize()
        assert int(d.sum().item()) == 7 * n
    finally:
        check(LIB.fy_host_free(p))
    q = C.c_void_p()
    check(LIB.fy_host_alloc_on(1 << 20, -2, C.byref(q)))  # no placement policy
    check(LIB.fy_host_free(q))


@pytest.mark.parametrize("states_on_device", [False, True])
def test_pipeline_strided_pieces_equal_whole_chunk(cuda_dev, states_on_device):
    """fy_chunk.states_stride: one chunk's SoA [master | m | v] (stride n)
    streamed as P pieces (each piece's master/m/v rows at stride n: one copy
    per row for host states, strided kernel pointers for device states)
    equals the oracle on the whole chunk. This is how the bench's e2e path
    splits a 13B block into pipeline units without re-laying out HBM."""
    from paper_2403_06504_b200 import optim as F
    n, pieces = (1 << 20) + 24, 4
    bounds = [0, 262144, 524296, 786440, n]  # 8-aligned, ragged last piece
    chunks, ref = _make_chunks([n], 21, cuda_dev, grads_on_host=True)
    c = chunks[0]
    states = c["h_states_t"].to(cuda_dev) if states_on_device else c["h_states_t"]
    pipe = F.ChunkPipeline(max(b - a for a, b in zip(bounds, bounds[1:])), slots=3,
                           grads_on_host=True, params_to_host=True, states_on_device=states_on_device)
    desc = [dict(n=b - a, h_states=states.data_ptr() + 4 * a, grad=c["grad_t"].data_ptr() + 2 * a,
                 h_param=c["h_param_t"].data_ptr() + 2 * a, states_stride=n)
            for a, b in zip(bounds, bounds[1:])]
    assert len(desc) == pieces
    pipe.step(desc, F.Hparams(step=10), want_grad_norm=True)
    sq, bad = pipe.wait()
    st = ref[0]["states"]
    mst, mm, vv = st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy()
    op = np.zeros(n, np.uint16)
    sq_ref, _ = O.adamw_step(mst, mm, vv, ref[0]["grad"], O.BF16, O.scalars(step=10), param_out=op)
    got = states.cpu().numpy() if states_on_device else states.numpy()
    assert _bits_equal(got, np.concatenate([mst, mm, vv]))
    assert np.array_equal(c["h_param_t"].view(torch.int16).numpy().view(np.uint16), op)
    assert abs(sq - sq_ref) <= 2e-7 * sq_ref and bad == 0
    with pytest.raises(Exception):
        pipe.step([dict(desc[0], states_stride=5)], F.Hparams(step=11))
    pipe.close()


def test_pipeline_update_done_events(cuda_dev):
    """fy_chunk.update_done is recorded right after the chunk's update: a
    side stream that waits on it and snapshots the chunk's device params
    (what an overlapped all-gather would send) sees the updated values."""
    from paper_2403_06504_b200 import optim as F
    sizes = [1 << 21, (1 << 20) + 8, 1 << 21]
    chunks, ref = _make_chunks(sizes, 31, cuda_dev, grads_on_host=False)
    d_params = [torch.zeros(n, dtype=torch.bfloat16, device=cuda_dev) for n in sizes]
    snaps = [torch.zeros(n, dtype=torch.bfloat16, device=cuda_dev) for n in sizes]
    evs = [torch.cuda.Event() for _ in sizes]
    for e in evs:
        e.record()  # torch creates the CUDA event lazily, on first record
    desc = _desc(chunks)
    for d, p, e in zip(desc, d_params, evs):
        d["d_param"] = p.data_ptr()
        d["update_done"] = e.cuda_event
    pipe = F.ChunkPipeline(max(sizes), slots=2, params_to_host=True, keep_params_on_device=True)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    pipe.step(desc, F.Hparams(step=10))
    for p, s, e in zip(d_params, snaps, evs):
        side.wait_event(e)
        with torch.cuda.stream(side):
            s.copy_(p)
    pipe.wait()
    torch.cuda.synchronize()
    sc = O.scalars(step=10)
    for s, r in zip(snaps, ref):
        n = r["grad"].size
        st = r["states"]
        op = np.zeros(n, np.uint16)
        O.adamw_step(st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy(), r["grad"], O.BF16, sc, param_out=op)
        assert np.array_equal(s.cpu().view(torch.int16).numpy().view(np.uint16), op)
    pipe.close()


@pytest.mark.parametrize("overflow", [False, True])
def test_pipeline_device_side_clip_and_skip(cuda_dev, overflow):
    """Streamed step with enqueue-only clipping / overflow skip
    (fy_pipeline_set_controls + fy_clip_coef): clipped updates are bit-exact
    vs the oracle with the combined scale; a skipped step writes the
    unchanged states back and bf16(master) as params."""
    from paper_2403_06504_b200 import optim as F
    sizes = [1 << 20, 4099, (1 << 19) + 8]
    chunks, ref = _make_chunks(sizes, 41, cuda_dev, grads_on_host=False)
    if overflow:
        chunks[1]["grad_t"][7] = float("inf")
        ref[1]["grad"][7] = 0x7F80
    ws = torch.zeros(F.workspace_floats(), device=cuda_dev)
    sq = torch.zeros(1, dtype=torch.float64, device=cuda_dev)
    bad = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    coef = torch.zeros(1, dtype=torch.float32, device=cuda_dev)
    skip = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    for k, c in enumerate(chunks):
        F.grad_stats(c["grad_t"], 1.0, sq, ws, nonfinite=bad, accumulate=k > 0)
    F.clip_coef(sq, bad, 1e-3, coef, skip)
    pipe = F.ChunkPipeline(max(sizes), slots=2)
    pipe.set_controls(coef, skip)
    pipe.step(_desc(chunks), F.Hparams(step=10))
    pipe.wait()
    torch.cuda.synchronize()
    assert int(skip.item()) == int(overflow)
    c_val = float(coef.item())
    for c, r in zip(chunks, ref):
        n = r["grad"].size
        st = r["states"]
        mst, mm, vv = st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy()
        if overflow:
            want_p = torch.from_numpy(mst).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        else:
            want_p = np.zeros(n, np.uint16)
            O.adamw_step(mst, mm, vv, r["grad"], O.BF16, O.scalars(step=10),
                         grad_scale=float(np.float32(1.0) * np.float32(c_val)), param_out=want_p)
        assert _bits_equal(c["h_states_t"].numpy(), np.concatenate([mst, mm, vv]))
        assert np.array_equal(c["h_param_t"].view(torch.int16).numpy().view(np.uint16), want_p)
    pipe.close()


def test_pipeline_mixed_resident_and_streamed_chunks(cuda_dev):
    """FY_CHUNK_STATES_ON_DEVICE: chunks whose states stay in HBM (spare HBM
    holding part of an out-of-core model's states) mixed with streamed ones
    in one step; all bit-exact vs the oracle, resident states updated in
    place on the device, every chunk's params written to host."""
    from paper_2403_06504_b200 import optim as F
    from paper_2403_06504_b200._lib import FY_CHUNK_STATES_ON_DEVICE
    sizes = [1 << 20, (1 << 20) + 8, 4099, 1 << 19]
    chunks, ref = _make_chunks(sizes, 51, cuda_dev, grads_on_host=False)
    resident = {0, 2}
    dev_states = {k: chunks[k]["h_states_t"].to(cuda_dev) for k in resident}
    desc = _desc(chunks)
    for k in resident:
        desc[k]["h_states"] = dev_states[k].data_ptr()
        desc[k]["flags"] = FY_CHUNK_STATES_ON_DEVICE
    pipe = F.ChunkPipeline(max(sizes), slots=2)
    counter = O.StepCounter()
    for step in (10, 11):
        pipe.step(desc, F.Hparams(step=step))
        pipe.wait()
        for k, (c, r) in enumerate(zip(chunks, ref)):
            sc = O.scalars_bt(*counter.next(step))
            n = r["grad"].size
            st = r["states"]
            mst, mm, vv = st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy()
            op = np.zeros(n, np.uint16)
            O.adamw_step(mst, mm, vv, r["grad"], O.BF16, sc, param_out=op)
            r["states"] = np.concatenate([mst, mm, vv])
            got = dev_states[k].cpu().numpy() if k in resident else c["h_states_t"].numpy()
            assert _bits_equal(got, r["states"]), f"chunk {k} step {step}"
            assert np.array_equal(c["h_param_t"].view(torch.int16).numpy().view(np.uint16), op)
    pipe.close()


def _traj():
    from pathlib import Path
    g = np.load(Path(__file__).resolve().parent / "golden" / "adamw_trajectory_golden.npz")
    return g, [int(x) for x in g["sizes"]], int(g["steps"])


def test_pipeline_deepspeed_trajectory_bit_exact(cuda_dev):
    """Six consecutive steps from fresh states over four chunks through the
    pipeline, which keeps DeepSpeed's step counter (chunk 0 of every step on
    the running product of beta^t, the others on pow): bit-exact vs the
    oracle run with the same counter, step by step."""
    from paper_2403_06504_b200 import optim as F
    g, sizes, steps = _traj()
    host, ref = [], []
    for c, n in enumerate(sizes):
        st = np.concatenate([g[f"c{c}_master0"], np.zeros(2 * n, np.float32)])
        host.append(dict(n=n, h_states_t=torch.from_numpy(st.copy()).pin_memory(),
                         h_param_t=torch.zeros(n, dtype=torch.bfloat16).pin_memory()))
        ref.append([st[:n].copy(), st[n:2 * n].copy(), st[2 * n:].copy()])
    pipe = F.ChunkPipeline(max(sizes), slots=2)
    k = O.StepCounter()
    for s in range(steps):
        grads = [torch.from_numpy(np.ascontiguousarray(g[f"c{c}_grads"][s]).view(np.int16)).view(torch.bfloat16)
                 .to(cuda_dev) for c in range(len(sizes))]
        desc = [dict(n=h["n"], h_states=h["h_states_t"].data_ptr(), grad=gr.data_ptr(),
                     h_param=h["h_param_t"].data_ptr()) for h, gr in zip(host, grads)]
        pipe.step(desc, F.Hparams(step=s + 1))
        pipe.wait()
        for c, (h, r) in enumerate(zip(host, ref)):
            op = np.zeros(h["n"], np.uint16)
            O.adamw_step(*r, np.ascontiguousarray(g[f"c{c}_grads"][s]), O.BF16, O.scalars_bt(*k.next(s + 1)),
                         param_out=op)
            assert _bits_equal(h["h_states_t"].numpy(), np.concatenate(r)), f"step {s + 1} chunk {c}"
            assert np.array_equal(h["h_param_t"].view(torch.int16).numpy().view(np.uint16), op)
    pipe.close()


def test_chunks_with_counter_hparams_vs_torch_and_oracle(cuda_dev):
    """fy_adamw_chunks with per-chunk hyper-parameters from fy_adam_counter
    (chunk 0 differs from the rest: separate launches inside one call), fed
    from torch's previous state every step: bit-exact vs the oracle and
    within the north star's tolerance of torch.optim.AdamW (per-element
    relative 1e-6 where well conditioned, summand bound everywhere;
    tests/test_oracle_golden.trajectory_check)."""
    from paper_2403_06504_b200 import optim as F
    from test_oracle_golden import oracle_trajectory, trajectory_check
    g, sizes, steps = _traj()
    counter = F.StepCounter()
    by_step = {}
    for s, c, old, st, gold, gb in oracle_trajectory():
        by_step.setdefault(s, []).append((c, old, st, gold, gb))
    for s in range(steps):
        entries = by_step[s]
        dev = []
        for c, old, st, gold, gb in entries:
            t = [torch.from_numpy(x.copy()).to(cuda_dev) for x in old]
            gr = torch.from_numpy(gb.view(np.int16).copy()).view(torch.bfloat16).to(cuda_dev)
            dev.append((t, gr, counter.next(F.Hparams(step=s + 1))))
        # one call; runs of equal hp share a launch
        from paper_2403_06504_b200._lib import LIB, AdamwArgs, check
        import ctypes as C
        arr = (AdamwArgs * len(dev))()
        for i, (t, gr, hp) in enumerate(dev):
            a = arr[i]
            a.master, a.exp_avg, a.exp_avg_sq = (x.data_ptr() for x in t)
            a.grad, a.grad_dtype, a.n, a.hp = gr.data_ptr(), 0, t[0].numel(), hp.c()
        check(LIB.fy_adamw_chunks(arr, len(dev), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        for (c, old, st, gold, gb), (t, gr, hp) in zip(entries, dev):
            got = [x.cpu().numpy() for x in t]
            for x, y in zip(got, st):
                assert _bits_equal(x, y), f"step {s + 1} chunk {c} vs oracle"
            trajectory_check(s, c, old, got, gold, gb)
