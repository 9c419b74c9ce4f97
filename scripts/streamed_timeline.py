#!/usr/bin/env python
"""Copy-engine timeline of the streamed (out-of-core) step as a Chrome trace.

65B-shaped chunks (805,306,368 params) with master/m/v in NUMA-local pinned
host memory (fy_host_alloc), each streamed as 4 pipeline pieces through
fy_pipeline_*; one step alone, then one step while a synthetic backward
(bf16 GEMMs of the 65B block on another stream) produces each block's
gradients and gates its pieces (fy_chunk.grad_ready). Per-piece H2D / update
/ D2H intervals come from the pipeline's CUDA events (fy_pipeline_timings).

Writes gpurun_out/streamed_timeline.json (chrome://tracing / Perfetto) and
prints per-lane busy fractions.
usage: python scripts/streamed_timeline.py [chunks]
"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

H = 8192
N = 12 * H * H
K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P = 4
n = N // P
dev = torch.device("cuda")

ptrs, hs, hp_ = [], [], []
for _ in range(K * P):
    st, pp = C.c_void_p(), C.c_void_p()
    check(LIB.fy_host_alloc(12 * n, C.byref(st)))
    check(LIB.fy_host_alloc(2 * n, C.byref(pp)))
    ptrs += [st, pp]
    hs.append(st.value)
    hp_.append(pp.value)
gen = torch.Generator(device=dev)
grads = []
for k in range(K):
    gen.manual_seed(20240817 + 1000 + k)
    grads.append((torch.randn(N, device=dev, generator=gen) * 1e-3).to(torch.bfloat16))
    for q in range(P):
        tmp = torch.empty(3 * n, device=dev)
        tmp[:n].normal_(0, 0.02, generator=gen)
        tmp[n:2 * n].normal_(0, 1e-3, generator=gen)
        tmp[2 * n:].normal_(0, 1e-3, generator=gen).square_()
        torch.from_numpy(np.ctypeslib.as_array((C.c_float * (3 * n)).from_address(hs[k * P + q]))).copy_(tmp)
torch.cuda.synchronize()

pipe = F.ChunkPipeline(n, slots=4, grads_on_host=False, params_to_host=True)
chunks = [dict(n=n, h_states=hs[k * P + q], grad=grads[k].data_ptr() + 2 * n * q, h_param=hp_[k * P + q])
          for k in range(K) for q in range(P)]
hp = F.Hparams()
pipe.step(chunks, hp)
pipe.wait()

# synthetic backward of the 65B block (b=16, s=1024): recompute + dgrad + wgrad
t = 16 * 1024
dims = [(H, 3 * H), (H, H), (H, 4 * H), (4 * H, H)]
X = [torch.randn(t, i, device=dev, dtype=torch.bfloat16) for i, _ in dims]
Y = [torch.randn(t, o, device=dev, dtype=torch.bfloat16) for _, o in dims]
W = [torch.randn(i, o, device=dev, dtype=torch.bfloat16) * 0.01 for i, o in dims]
G = [torch.empty(i, o, device=dev, dtype=torch.bfloat16) for i, o in dims]
bwd = torch.cuda.Stream(dev)

events = []
for mode in ("alone", "with_backward"):
    if mode == "with_backward":
        base = torch.cuda.Event(enable_timing=True)
        bevs = []
        torch.cuda.synchronize()
        with torch.cuda.stream(bwd):
            base.record(bwd)
            for k in range(K):
                s_ev = torch.cuda.Event(enable_timing=True)
                s_ev.record(bwd)
                for j in range(4):
                    torch.matmul(X[j], W[j], out=Y[j])
                for j in reversed(range(4)):
                    torch.matmul(Y[j], W[j].t(), out=X[j])
                    torch.matmul(X[j].t(), Y[j], out=G[j])
                e_ev = torch.cuda.Event(enable_timing=True)
                e_ev.record(bwd)
                bevs.append((s_ev, e_ev))
        for k in range(K):
            for q in range(P):
                chunks[k * P + q]["grad_ready"] = bevs[k][1].cuda_event
    pipe.step(chunks, hp)
    pipe.wait()
    torch.cuda.synchronize()
    tim, step_ns = pipe.timings(K * P)
    pid = 1 if mode == "alone" else 2
    events.append({"name": "process_name", "ph": "M", "pid": pid, "tid": 0,
                   "args": {"name": f"streamed step ({mode})"}})
    for tid, lane in enumerate(("H2D copy engine", "optimizer (fused AdamW)", "D2H copy engine",
                                "backward (bf16 GEMMs)")):
        events.append({"name": "thread_name", "ph": "M", "pid": pid, "tid": tid, "args": {"name": lane}})
    for i, tm in enumerate(tim):
        k, q = divmod(i, P)
        for tid, key, nbytes in ((0, "h2d", 12 * n), (1, "upd", 0), (2, "d2h", 14 * n)):
            a, b = tm[key]
            events.append({"name": f"{key} chunk{k}.{q}", "ph": "X", "pid": pid, "tid": tid,
                           "ts": a / 1e3, "dur": max(b - a, 1) / 1e3,
                           "args": {"bytes": nbytes, "GBps": nbytes / max(b - a, 1) if nbytes else None}})
    busy = {key: sum(tm[key][1] - tm[key][0] for tm in tim) / step_ns for key in ("h2d", "upd", "d2h")}
    line = {"mode": mode, "step_ms": step_ns / 1e6, "busy_frac": busy,
            "params_per_s": K * N / (step_ns * 1e-9), "d2h_GBps": 14 * N * K / step_ns}
    if mode == "with_backward":
        # backward lane: relative to `base`, recorded just before the step was
        # enqueued (the pipeline's own step-start event is internal), so the
        # two clocks agree to within the enqueue time (~tens of us)
        for k, (s_ev, e_ev) in enumerate(bevs):
            events.append({"name": f"backward block{k}", "ph": "X", "pid": pid, "tid": 3,
                           "ts": base.elapsed_time(s_ev) * 1e3, "dur": s_ev.elapsed_time(e_ev) * 1e3})
        line["backward_ms"] = base.elapsed_time(bevs[-1][1])
    print(json.dumps(line), flush=True)

out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
(out / "streamed_timeline.json").write_text(json.dumps({"traceEvents": events}))
pipe.close()
for p in ptrs:
    check(LIB.fy_host_free(p))
