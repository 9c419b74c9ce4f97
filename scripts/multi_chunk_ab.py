#!/usr/bin/env python
"""A/B, interleaved: the 13B step (40 chunks x 314.6M params, HBM-resident)
as 40 per-chunk launches vs one fy_adamw_chunks launch, and the C1 step (12 x
7.08M) likewise. Prints ms per step for each arm over alternating reps."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402

dev = torch.device("cuda")
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()


def run(L, h, reps):
    n = 12 * h * h
    st = [torch.rand(3 * n, device=dev) * 1e-3 for _ in range(L)]
    g = [(torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16) for _ in range(L)]
    chunks = [(s[:n], s[n:2 * n], s[2 * n:], gg, gg) for s, gg in zip(st, g)]

    def per_chunk():
        for k, c in enumerate(chunks):
            F.adamw_chunk(*c[:4], hp, param_out=c[4], grad_sq_sum=sq, accumulate_sq=k > 0, workspace=ws)

    def multi():
        F.adamw_chunks(chunks, hp, grad_sq_sum=sq, workspace=ws)

    def multi_one_each():  # the multi-chunk kernel, one chunk per launch (codegen vs schedule)
        for k, c in enumerate(chunks):
            F.adamw_chunks([c], hp, grad_sq_sum=sq, accumulate_sq=k > 0, workspace=ws)

    res = {"per_chunk": [], "multi": [], "multi_one_each": []}
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    arms = (("per_chunk", per_chunk), ("multi", multi), ("multi_one_each", multi_one_each))
    for _, fn in arms:
        fn()
    for _ in range(reps):
        for name, fn in arms:
            torch.cuda.synchronize()
            a.record()
            for _ in range(3):
                fn()
            b.record()
            torch.cuda.synchronize()
            res[name].append(a.elapsed_time(b) / 3)
    del st, g, chunks
    torch.cuda.empty_cache()
    return {k: sorted(v) for k, v in res.items()}


print(json.dumps({"c1": run(12, 768, 10)}))
print(json.dumps({"c2_13b": run(40, 5120, 5)}))
