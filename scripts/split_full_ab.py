#!/usr/bin/env python
"""Sweep-build A/B on the WHOLE GPU: the product default (single DMA
thread, 3 stages, 16 consumer warps) vs separate load / store DMA warps
with 4 or 6 stages; K 13B blocks, interleaved rounds with alternating
order. JSON lines + medians."""
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
K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ROUNDS = int(sys.argv[2]) if len(sys.argv) > 2 else 8
N = 12 * 5120 * 5120
dev = torch.device("cuda")
blocks = [(torch.rand(3 * N, device=dev) * 1e-3, (torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16))
          for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
variants = {"default": (0, 0, 0), "split4": (4, 16, 1), "split6": (6, 16, 1)}
res = collections.defaultdict(list)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
names = list(variants)
for r in range(ROUNDS):
    for name in (names if r % 2 == 0 else names[::-1]):
        stages, warps, split = variants[name]
        check(SW.fy_adamw_tune(1, stages, warps))
        check(SW.fy_adamw_tune_bulk(2048, split, 0))
        for _ in range(2):
            torch.cuda.synchronize()
            a.record()
            for st, g in blocks:
                F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], g, hp, param_out=g, grad_sq_sum=sq, workspace=ws,
                              accumulate_sq=True, lib=SW)
            b.record()
            torch.cuda.synchronize()
        res[name].append(28 * N * K / (a.elapsed_time(b) * 1e-3) / 1e9)
check(SW.fy_adamw_tune(1, 0, 0))
check(SW.fy_adamw_tune_bulk(2048, 0, 0))
for name, xs in res.items():
    print(json.dumps({"variant": name, "median_gbs": round(statistics.median(xs)), "all": [round(x) for x in xs]}))
