#!/usr/bin/env python
"""Round-2 probe: can the HBM-resident update hide under a backward?
(Fuyou's overlap premise.)

1. stages x consumer warps x SM budget: bandwidth of the fused step over K
   13B blocks with the TMA pipeline at 3/4/6 stages (28 KB per stage in
   flight per SM), 8 or 16 consumer warps, and at most B CTAs (one per SM)
   — is one SM's share bounded by its bytes in flight (Little's law) or by
   its consumers' arithmetic?
2. overlap: a synthetic backward (bf16 GEMMs of K 13B blocks, b=8 s=1024)
   on one stream and each block's update on a high-priority stream as soon
   as its backward is done, for SM budgets B with the GEMMs given the other
   148 - B SMs (cuBLAS SM carveout = B) or all SMs (no carveout).
Prints JSON lines."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
PHASES = sys.argv[2].split(",") if len(sys.argv) > 2 else ["stages", "overlap"]
h, t = 5120, 8 * 1024
N = 12 * h * h
dev = torch.device("cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
states = [torch.rand(3 * N, device=dev) * 1e-3 for _ in range(K)]
grads = [(torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16) for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
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
Ys = [torch.empty_like(y) for y in Y]
Xs = [torch.empty_like(x) for x in X]


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


try:
    import pynvml
    pynvml.nvmlInit()
    _NV = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # noqa: BLE001
    _NV = None


def powered(fn, seconds=2.0):
    """Run fn back to back for ~seconds; NVML board power (median, W) and
    SM clock sampled every 10 ms, energy per call = mean power x time per
    call (J). The energy bookkeeping behind the power-cap reading."""
    import threading
    import time
    ms = timed(fn, reps=2)
    reps = max(3, int(seconds * 1e3 / ms))
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetPowerUsage(_NV) / 1e3,
                            pynvml.nvmlDeviceGetClockInfo(_NV, pynvml.NVML_CLOCK_SM)))
            time.sleep(0.01)
    th = threading.Thread(target=sample) if _NV is not None else None
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if th:
        th.start()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    if th:
        stop.set()
        th.join()
    per = a.elapsed_time(b) / reps
    steady = samples[len(samples) // 3:] if samples else []
    pw = sorted(x[0] for x in steady)
    mhz = sorted(x[1] for x in steady)
    p_med = pw[len(pw) // 2] if pw else None
    return {"ms": per, "power_w": p_med, "sm_mhz": mhz[len(mhz) // 2] if mhz else None,
            "energy_j": p_med * per * 1e-3 if p_med else None}


def emit(d):
    print(json.dumps(d), flush=True)


if "stages" in PHASES:
    for budget in (32, 48, 64, 96, 128, 0):
        for warps in (8, 16):
            for stages in (3, 4, 6):
                check(LIB.fy_adamw_sm_budget(budget))
                check(LIB.fy_adamw_tune(1, stages, warps))
                ms = timed(lambda: [opt_block(k, torch.cuda.current_stream()) for k in range(K)])
                emit({"probe": "stages_x_budget", "ctas": budget or sms, "warps": warps, "stages": stages,
                      "ms": ms, "gbs": 28 * N * K / (ms * 1e-3) / 1e9})
    check(LIB.fy_adamw_tune(1, 0, 0))
    check(LIB.fy_adamw_sm_budget(0))

if "overlap" in PHASES:
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

    t_opt_full = timed(lambda: [opt_block(k, torch.cuda.current_stream()) for k in range(K)])
    t_bwd_full = timed(lambda: [bwd_block() for _ in range(K)])
    emit({"probe": "alone", "ms_optimizer_all_sms": t_opt_full, "ms_backward_all_sms": t_bwd_full,
          "tflops": 72 * t * h * h * K / (t_bwd_full * 1e-3) / 1e12})
    for budget in (0, 96, 64, 48, 32):
        for carve in ((False, True) if budget else (False,)):
            check(LIB.fy_adamw_sm_budget(budget))
            torch._C._set_sm_carveout_experimental(budget if carve else 0)
            t_bwd = timed(lambda: [bwd_block() for _ in range(K)])
            t_opt = timed(lambda: [opt_block(k, torch.cuda.current_stream()) for k in range(K)])
            t_both = timed(both)
            emit({"probe": "overlap", "opt_ctas": budget or sms, "gemm_carveout": budget if carve else 0,
                  "ms_both": t_both, "ms_backward_alone": t_bwd, "ms_optimizer_alone": t_opt,
                  "ms_serial_full_gpu": t_bwd_full + t_opt_full,
                  "hidden_fraction_vs_full_gpu_serial": (t_bwd_full + t_opt_full - t_both) / t_opt_full})
    torch._C._set_sm_carveout_experimental(0)
    check(LIB.fy_adamw_sm_budget(0))

if "power" in PHASES:
    # energy bookkeeping under the board power cap: if the backward and the
    # update each run AT the cap alone, running them together cannot take
    # less than (E_backward + E_update - P_idle x t) / P_cap
    idle = None
    if _NV is not None:
        import time
        torch.cuda.synchronize()
        time.sleep(1.0)
        idle = pynvml.nvmlDeviceGetPowerUsage(_NV) / 1e3
        cap = pynvml.nvmlDeviceGetEnforcedPowerLimit(_NV) / 1e3
    else:
        cap = None

    def both_on(opt_stream_fn):
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

    for path, label in ((1, "tma"), (0, "lsu")):
        check(LIB.fy_adamw_tune(path, 0, 0))
        check(LIB.fy_adamw_sm_budget(0))
        b = powered(lambda: [bwd_block() for _ in range(K)])
        o = powered(lambda: [opt_block(k, torch.cuda.current_stream()) for k in range(K)])
        c = powered(lambda: both_on(None))
        emit({"probe": "power", "path": label, "idle_w": idle, "cap_w": cap,
              "backward": b, "optimizer": o, "both": c,
              "serial_ms": b["ms"] + o["ms"],
              "hidden_fraction": (b["ms"] + o["ms"] - c["ms"]) / o["ms"],
              "energy_bound_ms": ((b["energy_j"] + o["energy_j"]) / cap * 1e3
                                  if cap and b["energy_j"] and o["energy_j"] else None)})
    check(LIB.fy_adamw_tune(1, 0, 0))
