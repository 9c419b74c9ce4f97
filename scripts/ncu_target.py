"""Small ncu target (diagnostic): a few fused-Adam launches on 13B-block
chunks (314,572,800 params, 8.8 GB of traffic each) with the default kernel
configuration, so multi-pass ncu captures can use --replay-mode application
(each pass re-runs this short script instead of replaying the kernel in
place, which perturbs the TMA kernel's timing and counters)."""
import sys
from pathlib import Path

import torch

# optional argv[1]: SM budget (fy_adamw_sm_budget CTAs) for the budgeted regime
BUDGET = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

if BUDGET:
    check(LIB.fy_adamw_sm_budget(BUDGET))

N = 12 * 5120 * 5120
dev = torch.device("cuda")
chunks = []
for k in range(2):
    st = torch.empty(3 * N, device=dev)
    st[:N].normal_(0, 0.02)
    st[N:2 * N].normal_(0, 1e-3)
    st[2 * N:].normal_(0, 1e-3).square_()
    chunks.append((st, (torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16)))
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
bad = torch.zeros(1, dtype=torch.int32, device=dev)
hp = F.Hparams()
for i in range(6):
    st, g = chunks[i % 2]
    F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], g, hp, param_out=g, grad_sq_sum=sq,
                  workspace=ws, nonfinite=bad)
torch.cuda.synchronize()
print("ok", sq.item())
