"""Generate tests/golden/adamw_torch_golden.npz (committed fixture).

Pins the CPU AdamW restatement (oracle/adamw_oracle.c) against an independent
implementation of the same published algorithm, torch.optim.AdamW / Adam
(torch 2.11.0, CPU, foreach=False, fused=False). The reference itself has no
Adam arithmetic to pin against ("parity unpinned").

Inputs follow SURVEY.md §8d: master ~ N(0, 0.02^2), m ~ N(0, 1e-3^2),
v = N(0, 1e-3)^2, grads bf16(N(0, 1e-3^2)) (fp16 case: fp16(g * 2^16) with
grad_scale 2^-16), steps 10..12, lr 1e-4, betas (0.9, 0.95), eps 1e-8,
wd 0.1, seed 20240817 + case index. n = 4099 exercises the 8-wide vector tail.

Run:  python tests/golden/make_adamw_golden.py
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import torch

OUT = Path(__file__).resolve().parent / "adamw_torch_golden.npz"
N = 4099
STEPS = 3
FIRST_STEP = 10


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def fp16_bits(t: torch.Tensor) -> np.ndarray:
    return t.to(torch.float16).view(torch.int16).numpy().view(np.uint16)


def make_case(idx: int, grad_kind: str, adamw: bool, wd: float):
    rng = np.random.default_rng(20240817 + idx)
    master = rng.normal(0, 0.02, N).astype(np.float32)
    m = rng.normal(0, 1e-3, N).astype(np.float32)
    v = (rng.normal(0, 1e-3, N) ** 2).astype(np.float32)
    grads_f = [rng.normal(0, 1e-3, N).astype(np.float32) for _ in range(STEPS)]
    # special values in the first few elements: zero grad, zero state, tiny
    # (denormal-range) grads, large grads
    for g in grads_f:
        g[0] = 0.0
        g[1] = 1e-30
        g[2] = -3e-39
        g[3] = 5.0
    m[4] = 0.0
    v[4] = 0.0
    grad_scale = 1.0
    if grad_kind == "bf16":
        grads_bits = [bf16_bits(torch.from_numpy(g)) for g in grads_f]
        grads_true = [torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).float() for b in grads_bits]
    else:
        grad_scale = 2.0 ** -16
        grads_bits = [fp16_bits(torch.from_numpy(g) * 2.0 ** 16) for g in grads_f]
        grads_true = [torch.from_numpy(b.view(np.int16)).view(torch.float16).float() * grad_scale
                      for b in grads_bits]

    p = torch.nn.Parameter(torch.from_numpy(master.copy()))
    cls = torch.optim.AdamW if adamw else torch.optim.Adam
    opt = cls([p], lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=wd, foreach=False,
              fused=False)
    opt.state[p] = {"step": torch.tensor(float(FIRST_STEP - 1)),
                    "exp_avg": torch.from_numpy(m.copy()),
                    "exp_avg_sq": torch.from_numpy(v.copy())}
    outs = []
    for s in range(STEPS):
        p.grad = grads_true[s].clone()
        opt.step()
        st = opt.state[p]
        outs.append((p.detach().numpy().copy(), st["exp_avg"].numpy().copy(),
                     st["exp_avg_sq"].numpy().copy()))
    tag = f"case{idx}"
    d = {
        f"{tag}_master0": master, f"{tag}_m0": m, f"{tag}_v0": v,
        f"{tag}_grads": np.stack(grads_bits),
        f"{tag}_meta": np.array([0 if grad_kind == "bf16" else 1, int(adamw), wd, grad_scale,
                                 FIRST_STEP], dtype=np.float64),
    }
    for s, (pp, mm, vv) in enumerate(outs):
        d[f"{tag}_master{s + 1}"] = pp
        d[f"{tag}_m{s + 1}"] = mm
        d[f"{tag}_v{s + 1}"] = vv
    return d


def main():
    cases = [("bf16", True, 0.1), ("fp16", True, 0.1), ("bf16", False, 0.01), ("bf16", True, 0.0)]
    out = {"ncases": np.array(len(cases)), "n": np.array(N), "steps": np.array(STEPS),
           "torch_version": np.array(torch.__version__)}
    for i, (gk, aw, wd) in enumerate(cases):
        out.update(make_case(i, gk, aw, wd))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
