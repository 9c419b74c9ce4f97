#!/usr/bin/env python
"""Sweep-build probe (build/sweep/liboffsim_sweep.so): the SM-budgeted
fused step with separate load / store DMA warps (SPLIT) beside 16 consumer
warps vs the product's single DMA thread, at 32 / 64 / 96 / 148 CTAs and
3 / 4 / 6 stages; K 13B blocks per timing, interleaved rounds. JSON lines."""
import collections
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import check, load_sweep_lib  # noqa: E402

SW = load_sweep_lib()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
N = 12 * 5120 * 5120
dev = torch.device("cuda")
blocks = [(torch.rand(3 * N, device=dev) * 1e-3, (torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16))
          for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()


def step():
    for st, g in blocks:
        F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], g, hp, param_out=g, grad_sq_sum=sq, workspace=ws,
                      accumulate_sq=True, lib=SW)


variants = [("single", 4, 0), ("single", 6, 0), ("split", 3, 1), ("split", 4, 1), ("split", 6, 1)]
res = collections.defaultdict(list)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(3):
    for budget in (32, 64, 96, 148):
        for name, stages, split in (variants if r % 2 == 0 else variants[::-1]):
            check(SW.fy_adamw_sm_budget(budget))
            check(SW.fy_adamw_tune(1, stages, 16))
            check(SW.fy_adamw_tune_bulk(2048, split, 0))
            step()
            torch.cuda.synchronize()
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            res[(budget, name, stages)].append(28 * N * K / (a.elapsed_time(b) * 1e-3) / 1e9)
check(SW.fy_adamw_sm_budget(0))
check(SW.fy_adamw_tune(1, 0, 0))
check(SW.fy_adamw_tune_bulk(2048, 0, 0))
for (budget, name, stages), xs in sorted(res.items()):
    print(json.dumps({"ctas": budget, "dma": name, "stages": stages, "warps": 16,
                      "median_gbs": round(statistics.median(xs)), "all": [round(x) for x in xs]}))
