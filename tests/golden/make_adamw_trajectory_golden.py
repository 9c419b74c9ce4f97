"""Generate tests/golden/adamw_trajectory_golden.npz (committed fixture): a
consecutive-step AdamW trajectory over several chunks, for the step-counter
semantics of DeepSpeed's CPU Adam (the first chunk of every step on the
running product of beta^t, the others on pow; see
make_step_counter_golden.py).

Independent implementation: torch.optim.AdamW 2.11 (CPU, foreach=False,
fused=False), one parameter tensor per chunk in one optimizer, fresh states
(m = v = 0) at step 1, STEPS consecutive steps; betas (0.9, 0.95), lr 1e-4,
eps 1e-8, wd 0.1 (GPT-3 settings); bf16 gradients
~ N(0, 1e-3^2) per step; master ~ N(0, 0.02^2); seed 20240817 + chunk.
torch evaluates bias corrections in double (1 - beta**step), so it differs
from DeepSpeed's float path by ulps: the tests compare against it with a
tolerance, and bit-exactly against the oracle.
Run:  python tests/golden/make_adamw_trajectory_golden.py
"""
from pathlib import Path

import numpy as np
import torch

OUT = Path(__file__).resolve().parent / "adamw_trajectory_golden.npz"
SIZES = [4099, 2048, 777, 8]
STEPS = 6


def main():
    ps, grads = [], []
    for c, n in enumerate(SIZES):
        rng = np.random.default_rng(20240817 + c)
        ps.append(torch.nn.Parameter(torch.from_numpy(rng.normal(0, 0.02, n).astype(np.float32))))
        grads.append([torch.from_numpy(rng.normal(0, 1e-3, n).astype(np.float32)).to(torch.bfloat16)
                      for _ in range(STEPS)])
    out = {"sizes": np.array(SIZES), "steps": np.array(STEPS), "torch_version": np.array(torch.__version__)}
    for c in range(len(SIZES)):
        out[f"c{c}_master0"] = ps[c].detach().numpy().copy()
        out[f"c{c}_grads"] = np.stack([g.view(torch.int16).numpy().view(np.uint16) for g in grads[c]])
    opt = torch.optim.AdamW(ps, lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1, foreach=False,
                            fused=False)
    for s in range(STEPS):
        for c, p in enumerate(ps):
            p.grad = grads[c][s].float()
        opt.step()
        for c, p in enumerate(ps):
            st = opt.state[p]
            out[f"c{c}_master{s + 1}"] = p.detach().numpy().copy()
            out[f"c{c}_m{s + 1}"] = st["exp_avg"].numpy().copy()
            out[f"c{c}_v{s + 1}"] = st["exp_avg_sq"].numpy().copy()
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
