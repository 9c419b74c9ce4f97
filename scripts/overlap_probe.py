#!/usr/bin/env python
"""SM budget of the fused optimizer and its overlap with a backward pass
(SURVEY.md §7 "overlap contention": on B200 the optimizer shares SMs and HBM
with backward, where Fuyou's CPU optimizer used idle cores).

1. bandwidth of the fused step vs its SM budget (fy_adamw_sm_budget):
   K chunks of the 13B block, budgets 16..148 CTAs (one per SM);
2. a synthetic backward of K 13B-shaped blocks (b=8, s=1024: recompute
   forward + dgrad + wgrad bf16 GEMMs, 72*t*h^2 FLOP per block) on one
   stream, and each block's optimizer update launched on a high-priority
   stream as soon as that block's backward is done, for several budgets:
   step time vs backward alone and optimizer alone.
Prints JSON lines."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
h, t = 5120, 8 * 1024
N = 12 * h * h
dev = torch.device("cuda")
states = [torch.rand(3 * N, device=dev) * 1e-3 for _ in range(K)]
grads = [(torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16) for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
opt_s = torch.cuda.Stream(priority=-1)
bwd_s = torch.cuda.Stream(priority=0)


def opt_block(k, stream):
    st = states[k]
    F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], grads[k], hp, param_out=grads[k], grad_sq_sum=sq,
                  workspace=ws, accumulate_sq=True, stream=stream)


dims = [(h, 3 * h), (h, h), (h, 4 * h), (4 * h, h)]
X = [torch.randn(t, i, device=dev, dtype=torch.bfloat16) * 0.1 for i, _ in dims]
Y = [torch.randn(t, o, device=dev, dtype=torch.bfloat16) * 0.1 for _, o in dims]
W = [torch.randn(i, o, device=dev, dtype=torch.bfloat16) * 0.01 for i, o in dims]
G = [torch.empty(i, o, device=dev, dtype=torch.bfloat16) for i, o in dims]
Ys = [torch.empty_like(y) for y in Y]   # outputs never feed back into inputs:
Xs = [torch.empty_like(x) for x in X]   # constant operands, constant power


def bwd_block():
    for j in range(4):
        torch.matmul(X[j], W[j], out=Ys[j])          # recompute forward
    for j in reversed(range(4)):
        torch.matmul(Y[j], W[j].t(), out=Xs[j])      # dgrad
        torch.matmul(X[j].t(), Y[j], out=G[j])       # wgrad


def timed(fn, reps=3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


# 1. bandwidth vs SM budget
for budget in (16, 32, 48, 64, 96, 128, 0):
    check(LIB.fy_adamw_sm_budget(budget))
    ms = timed(lambda: [opt_block(k, torch.cuda.current_stream()) for k in range(K)])
    print(json.dumps({"probe": "budget", "ctas": budget or 148, "ms": ms,
                      "gbs": 28 * N * K / (ms * 1e-3) / 1e9}), flush=True)
check(LIB.fy_adamw_sm_budget(0))

# 2. overlap with a backward
t_bwd = timed(lambda: [bwd_block() for _ in range(K)])
flops = 72 * t * h * h * K
print(json.dumps({"probe": "backward_alone", "ms": t_bwd, "tflops": flops / (t_bwd * 1e-3) / 1e12}), flush=True)
t_opt = timed(lambda: [opt_block(k, torch.cuda.current_stream()) for k in range(K)])


def both():
    cur = torch.cuda.current_stream()
    bwd_s.wait_stream(cur)
    opt_s.wait_stream(cur)
    for k in range(K):
        with torch.cuda.stream(bwd_s):
            bwd_block()
            e = torch.cuda.Event()
            e.record(bwd_s)
        opt_s.wait_event(e)
        opt_block(k, opt_s)
    cur.wait_stream(bwd_s)
    cur.wait_stream(opt_s)


for budget in (0, 96, 64, 32):
    check(LIB.fy_adamw_sm_budget(budget))
    t_both = timed(both)
    serial = t_bwd + t_opt
    print(json.dumps({"probe": "overlap", "opt_ctas": budget or 148, "ms_both": t_both, "ms_backward_alone": t_bwd,
                      "ms_optimizer_alone": t_opt, "ms_serial": serial,
                      "hidden_fraction_of_optimizer": (serial - t_both) / t_opt}), flush=True)
check(LIB.fy_adamw_sm_budget(0))
