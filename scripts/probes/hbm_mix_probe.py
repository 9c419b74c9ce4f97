"""Probe (r02ax): HBM bandwidth by traffic mix on this B200 — read-only
(sum), write-only (fill), copy (1:1) — to see how much the 50/50 read/write
mix of the Adam step (14 B read + 14 B write per param) costs against
one-directional streams. 8 GiB buffers, best of 10, CUDA events."""
import json
import torch

dev = torch.device("cuda")
n = 1 << 31  # 2 Gi fp32 = 8 GiB
a = torch.empty(n, dtype=torch.float32, device=dev).normal_()
b = torch.empty(n, dtype=torch.float32, device=dev)
out = torch.empty(1, dtype=torch.float32, device=dev)


def best(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) * 1e-3)
    return nbytes / min(t) / 1e9, nbytes / sorted(t)[len(t) // 2] / 1e9


res = {}
res["read_only_sum"] = best(lambda: torch.sum(a, dim=0, out=out[0]), 4 * n)
res["write_only_fill"] = best(lambda: b.fill_(1.0), 4 * n)
res["write_only_zero"] = best(lambda: b.zero_(), 4 * n)
res["copy_1to1"] = best(lambda: b.copy_(a), 8 * n)
res["add_2r1w"] = best(lambda: torch.add(a[: n // 2], a[n // 2:], out=b[: n // 2]), 12 * (n // 2))
print(json.dumps({k: {"best_gbs": v[0], "median_gbs": v[1]} for k, v in res.items()}, indent=1))
