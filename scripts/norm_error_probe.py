#!/usr/bin/env python
"""Diagnostic: relative error of the fused kernel's grad sum of squares
(per-tile fp32 sums flushed to double, per-CTA partials, ordered double
reduction) against an exact-order float64 sum (numpy, sum of (double)g^2 —
the oracle's definition), over sizes from a tail-only chunk to a 13B block,
both paths, bf16 and fp16-scaled grads. JSON lines."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

dev = torch.device("cuda")
ws = torch.zeros(F.workspace_floats(), device=dev)
for path, label in ((1, "tma"), (0, "lsu")):
    check(LIB.fy_adamw_tune(path, 0, 0))
    for n in (1000, 7077888, 12 * 5120 * 5120):
        for dt, scale in ((torch.bfloat16, 1.0), (torch.float16, 2.0 ** -16)):
            g32 = torch.randn(n, device=dev, generator=torch.Generator(device=dev).manual_seed(n)) * 1e-3
            g = (g32 / scale).to(dt)
            st = torch.zeros(3 * n, device=dev)
            sq = torch.zeros(1, dtype=torch.float64, device=dev)
            F.adamw_chunk(st[:n], st[n:2 * n], st[2 * n:], g, F.Hparams(grad_scale=scale), grad_sq_sum=sq,
                          workspace=ws)
            torch.cuda.synchronize()
            gs = (g.float() * scale).double()          # the kernel squares fp32(g * scale)
            ref = float((gs * gs).sum())               # float64 sum (pairwise on the GPU)
            exact = float(np.sum(np.square(gs.cpu().numpy()), dtype=np.float64))
            print(json.dumps({"path": label, "n": n, "dtype": str(dt), "rel_err_vs_f64": abs(sq.item() - exact) / exact,
                              "torch_f64_vs_numpy_f64": abs(ref - exact) / exact}), flush=True)
check(LIB.fy_adamw_tune(1, 0, 0))
