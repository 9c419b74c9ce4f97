"""GPU tuning sweep of the fused Adam kernel (diagnostic, not the bench).

Times fy_adamw_chunk over K chunks of the 13B block size (314,572,800
params; 8.8 GB of traffic per launch >> L2) for each (unroll, ctas_per_sm)
and prints achieved GB/s at 28 B/param against MEASURED_PEAKS.json.
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import check, load_sweep_lib  # noqa: E402

LIB = load_sweep_lib()  # the sweep build (make sweep): product + experimental TMA variants

N = 12 * 5120 * 5120
K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
dev = torch.device("cuda")
states = [torch.rand(3 * N, device=dev) * 1e-3 for _ in range(K)]
grads = [(torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16) for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
bad = torch.zeros(1, dtype=torch.int32, device=dev)
hp = F.Hparams()
results = []
# (path, unroll/stages, ctas_per_sm/consumer warps, tile, split)
configs = ([(0, 2, 2, 2048, 0)] + [(1, st, 0, 2048, 0) for st in (2, 3, 4)]
           + [(1, st, 4, 2048, 0) for st in (2, 3)]
           + [(1, 3, 0, 1024, 0), (1, 2, 0, 4096, 0), (1, 3, 0, 4096, 0)]
           + [(1, st, 0, 2048, 1) for st in (2, 3, 4)] + [(1, 4, 0, 1024, 1), (1, 3, 0, 4096, 1)])
configs = [c + (0,) for c in configs]
if len(sys.argv) > 2 and sys.argv[2] == "probes":  # hints / speed of light vs the default
    configs = [(1, 3, 0, 2048, 0, p) for p in (0, 1, 2, 3)]
if len(sys.argv) > 2 and sys.argv[2] == "default-only":
    configs = [(1, 3, 0, 2048, 0, 0)]
for path, unroll, cps, tile, split, probe in configs * 2:  # two passes: run-to-run noise is part of the answer
        check(LIB.fy_adamw_tune(path, unroll, cps))
        check(LIB.fy_adamw_tune_bulk(tile, split, probe))
        def launch(k):
            st = states[k]
            F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], grads[k], hp, param_out=grads[k],
                          grad_sq_sum=sq, workspace=ws, nonfinite=bad, lib=LIB)
        for k in range(K):
            launch(k)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 3
        ev[0].record()
        for r in range(reps):
            for k in range(K):
                launch(k)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / (reps * K)
        gbs = 28 * N / (ms * 1e-3) / 1e9
        results.append(dict(path=path, unroll=unroll, ctas_per_sm=cps, tile=tile, split=split, probe=probe, ms=ms,
                            gbs=gbs, frac=gbs / peak))
        print(f"path={path} unroll={unroll} ctas_per_sm={cps} tile={tile} split={split} probe={probe}: {ms:.3f} ms/launch  "
              f"{gbs:.0f} GB/s  {gbs / peak:.3f} of peak", flush=True)
check(LIB.fy_adamw_tune(1, 0, 0))
check(LIB.fy_adamw_tune_bulk(2048, 0, 0))
best = max(results, key=lambda r: r["gbs"])
print("BEST", json.dumps(best))
out = ROOT / "gpurun_out" / "kernel_sweep.json"
out.parent.mkdir(exist_ok=True)
out.write_text(json.dumps(results, indent=1))
