#!/usr/bin/env python
"""Where do the ~0.4 ms between the shard step and the list launch go?
40 13B chunks, interleaved rounds: (a) fy_shard_step (per-chunk events for
update_ms + chunk-done events), (b) fy_adamw_chunk per chunk (update + norm
reduction, no events), (c) fy_adamw_chunks (one call). JSON lines."""
import collections
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402

L, N = 40, 12 * 5120 * 5120
dev = torch.device("cuda")
sh = F.Shard([N] * L, tier="device")
states = []
grads = []
for k in range(L):
    st = torch.empty(3 * N, device=dev)
    st[:N].normal_(0, 0.02)
    st[N:2 * N].normal_(0, 1e-3)
    st[2 * N:].normal_(0, 1e-3).square_()
    states.append(st)
    g = sh.own_params(k)
    g.copy_((torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16))
    grads.append(g)
io = [dict(states=s.data_ptr(), grad=g.data_ptr()) for s, g in zip(states, grads)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
stream = torch.cuda.current_stream()


def a():
    sh.step(io, hp, want_grad_norm=True, stream=stream)
    sh.wait()


def b():
    for k in range(L):
        st = states[k]
        F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], grads[k], hp, param_out=grads[k], grad_sq_sum=sq,
                      workspace=ws, accumulate_sq=k > 0)


multi = [(s[:N], s[N:2 * N], s[2 * N:], g, g) for s, g in zip(states, grads)]


def c():
    F.adamw_chunks(multi, hp, grad_sq_sum=sq, workspace=ws)


arms = {"shard_step": a, "per_chunk": b, "list": c}
res = collections.defaultdict(list)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(6):
    for name in (list(arms) if r % 2 == 0 else list(arms)[::-1]):
        fn = arms[name]
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 3)
for name, xs in res.items():
    print(json.dumps({"arm": name, "median_ms": round(statistics.median(xs), 3), "all": [round(x, 3) for x in xs]}))
sh.close()
