#!/usr/bin/env python
"""The product's automatic shape under an SM budget (fy_adamw_sm_budget,
no explicit tune): bandwidth of K 13B blocks at 32..148 CTAs. JSON lines."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
N = 12 * 5120 * 5120
dev = torch.device("cuda")
blocks = [(torch.rand(3 * N, device=dev) * 1e-3, (torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16))
          for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
BUDGETS = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [32, 48, 64, 96, 128, 0]
for budget in BUDGETS:
    check(LIB.fy_adamw_sm_budget(budget))
    best = 1e30
    for _ in range(3):
        for st, g in blocks:
            F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], g, hp, param_out=g, grad_sq_sum=sq, workspace=ws)
        torch.cuda.synchronize()
        a.record()
        for st, g in blocks:
            F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], g, hp, param_out=g, grad_sq_sum=sq, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(json.dumps({"ctas": budget or 148, "shape": "auto", "gbs": round(28 * N * K / (best * 1e-3) / 1e9)}),
          flush=True)
check(LIB.fy_adamw_sm_budget(0))
