"""fy_grad_stats rate on one 13B-shaped chunk of bf16 grads (314.6M params,
2 B/param read), CUDA events, best of 20."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2403_06504_b200 import optim as F  # noqa: E402

n = 12 * 5120 * 5120
dev = torch.device("cuda")
g = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
bad = torch.zeros(1, dtype=torch.int32, device=dev)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
F.grad_stats(g, 1.0, sq, ws, bad)
best = 1e30
for _ in range(20):
    torch.cuda.synchronize()
    a.record()
    F.grad_stats(g, 1.0, sq, ws, bad)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(json.dumps({"params": n, "ms": round(best, 4), "gbs_read": round(2 * n / best / 1e6, 1)}))
