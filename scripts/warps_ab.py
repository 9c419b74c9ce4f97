#!/usr/bin/env python
"""A/B: TMA consumer warps (product default vs 8 vs 16) for the C1 list
launch (12 x 7.08M params, one fy_adamw_chunks call, 20 back-to-back steps)
and for fp32 gradients (8 13B blocks, 30 B/param), interleaved rounds with
alternating order. JSON lines + medians."""
import collections
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

dev = torch.device("cuda")
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
L, n = 12, 12 * 768 * 768
st = [torch.rand(3 * n, device=dev) * 1e-3 for _ in range(L)]
g = [(torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16) for _ in range(L)]
c1 = [(s[:n], s[n:2 * n], s[2 * n:], gg, gg) for s, gg in zip(st, g)]
N, K = 12 * 5120 * 5120, 8
big = [(torch.rand(3 * N, device=dev) * 1e-3, torch.randn(N, device=dev) * 1e-3,
        torch.empty(N, dtype=torch.bfloat16, device=dev)) for _ in range(K)]


def c1_step():
    for _ in range(20):
        F.adamw_chunks(c1, hp, grad_sq_sum=sq, workspace=ws)


def fp32_step():
    for s, gg, p in big:
        F.adamw_chunk(s[:N], s[N:2 * N], s[2 * N:], gg, hp, param_out=p, grad_sq_sum=sq, workspace=ws)


arms = {"c1_list": (c1_step, 28 * L * n * 20), "fp32_grads_13b": (fp32_step, 30 * N * K)}
variants = [0, 8, 16]
res = collections.defaultdict(list)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(8):
    for arm, (fn, nbytes) in arms.items():
        for w in (variants if r % 2 == 0 else variants[::-1]):
            check(LIB.fy_adamw_tune(1, 0, w))
            fn()
            torch.cuda.synchronize()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            res[(arm, w)].append(nbytes / (ms * 1e-3) / 1e9)
check(LIB.fy_adamw_tune(1, 0, 0))
for (arm, w), xs in res.items():
    print(json.dumps({"arm": arm, "warps": w or "default", "median_gbs": statistics.median(xs),
                      "all": [round(x) for x in xs]}))
