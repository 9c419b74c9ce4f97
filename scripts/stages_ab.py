#!/usr/bin/env python
"""A/B of the fused step's TMA pipeline shape on the WHOLE GPU (148 CTAs):
(stages, consumer warps) variants interleaved round-robin over several
rounds, each timing K back-to-back 13B-block launches (CUDA events), so
power-cap / clock drift hits every variant alike. JSON lines + a summary."""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ROUNDS = int(sys.argv[2]) if len(sys.argv) > 2 else 6
N = 12 * 5120 * 5120
dev = torch.device("cuda")
states = []
for k in range(K):
    st = torch.empty(3 * N, device=dev)
    st[:N].normal_(0, 0.02)
    st[N:2 * N].normal_(0, 1e-3)
    st[2 * N:].normal_(0, 1e-3).square_()
    states.append((st, (torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16)))
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
variants = [(0, 0), (3, 8), (4, 8), (6, 8), (3, 16), (4, 16)]  # (0, 0) = product default
if len(sys.argv) > 3:  # e.g. "3:8,3:16"
    variants = [tuple(int(x) for x in v.split(":")) for v in sys.argv[3].split(",")]
res = {v: [] for v in variants}


def step():
    for st, g in states:
        F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], g, hp, param_out=g, grad_sq_sum=sq, workspace=ws,
                      accumulate_sq=True)


a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(ROUNDS):
    for v in (variants if r % 2 == 0 else variants[::-1]):  # alternate the order
        check(LIB.fy_adamw_tune(1, v[0], v[1]))
        step()
        torch.cuda.synchronize()
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        res[v].append(ms)
        print(json.dumps({"round": r, "stages": v[0], "warps": v[1], "ms": ms,
                          "gbs": 28 * N * K / (ms * 1e-3) / 1e9}), flush=True)
check(LIB.fy_adamw_tune(1, 0, 0))
for v, xs in res.items():
    med = statistics.median(xs)
    print(json.dumps({"summary": True, "stages": v[0], "warps": v[1], "median_ms": med,
                      "median_gbs": 28 * N * K / (med * 1e-3) / 1e9, "min_ms": min(xs)}))
