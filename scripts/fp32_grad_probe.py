#!/usr/bin/env python
"""fp32 gradients: TMA path (18 B/element stages) vs LSU path, 20 chunks of
the 13B block (30 B/param of traffic: 4 grad r + 12 state r + 12 state w + 2
param w), alternating, ~2 s each."""
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

N, K = 12 * 5120 * 5120, 20
dev = torch.device("cuda")
st = [torch.rand(3 * N, device=dev) * 1e-3 for _ in range(K)]
g = [torch.randn(N, device=dev) * 1e-3 for _ in range(K)]
p = [torch.empty(N, dtype=torch.bfloat16, device=dev) for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()


def step():
    for k in range(K):
        F.adamw_chunk(st[k][:N], st[k][N:2 * N], st[k][2 * N:], g[k], hp, param_out=p[k], grad_sq_sum=sq,
                      workspace=ws, accumulate_sq=k > 0)


for name, tune in (("tma", (1, 3, 0)), ("lsu", (0, 2, 2)), ("tma_2", (1, 3, 0)), ("lsu_2", (0, 2, 2))):
    check(LIB.fy_adamw_tune(*tune))
    step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.time()
    a.record()
    while time.time() - t0 < 2.0:
        step()
        reps += 1
        torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(json.dumps({"path": name, "ms_per_step": ms, "gbs_at_30B": 30 * N * K / (ms * 1e-3) / 1e9}), flush=True)
check(LIB.fy_adamw_tune(1, 0, 0))
