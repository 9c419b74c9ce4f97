#!/usr/bin/env python
"""Power / clock vs kernel variant in the sustained regime: each variant runs
the whole 13B set back to back for ~3 s while NVML samples power and SM
clock every 20 ms. Variants: the product TMA kernel, the no-arithmetic probe
(same traffic), the LSU kernel. Prints one JSON line per variant."""
import json
import statistics
import sys
import threading
import time
from pathlib import Path

import pynvml
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import check, load_sweep_lib  # noqa: E402

LIB = load_sweep_lib()  # the sweep build (make sweep): product + experimental TMA variants

N = 12 * 5120 * 5120
K = 40
dev = torch.device("cuda")
states = [torch.rand(3 * N, device=dev) * 1e-3 for _ in range(K)]
grads = [(torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16) for _ in range(K)]
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def step():
    for k in range(K):
        st = states[k]
        F.adamw_chunk(st[:N], st[N:2 * N], st[2 * N:], grads[k], hp, param_out=grads[k], grad_sq_sum=sq,
                      workspace=ws, lib=LIB)


VARIANTS = {
    "default": (("tma_default", (1, 3, 0), (2048, 0, 0)), ("tma_no_arithmetic", (1, 3, 0), (2048, 0, 2)),
                ("lsu_unroll2", (0, 2, 2), (2048, 0, 0)), ("tma_default_again", (1, 3, 0), (2048, 0, 0))),
    # DMA thread computing addresses after (product) vs before (probe 4) each stage wait
    "hoist": (("tma_after_wait", (1, 3, 0), (2048, 0, 0)), ("tma_hoisted", (1, 3, 0), (2048, 0, 4)),
              ("tma_after_wait_2", (1, 3, 0), (2048, 0, 0)), ("tma_hoisted_2", (1, 3, 0), (2048, 0, 4))),
    # refill the previous tile's stage (wait_group.read 1) vs the one just stored
    "lag": (("tma_default", (1, 3, 0), (2048, 0, 0)), ("lag_3stages", (1, 3, 0), (2048, 0, 5)),
            ("lag_4stages", (1, 3, 0), (2048, 0, 6)), ("tma_default_2", (1, 3, 0), (2048, 0, 0)),
            ("lag_3stages_2", (1, 3, 0), (2048, 0, 5)), ("lag_4stages_2", (1, 3, 0), (2048, 0, 6))),
    # SM budget (fy_adamw_sm_budget): fewer CTAs (one per SM) draw less
    # power; does the DRAM stay saturated and the clock rise?
    "budget": tuple((f"sms_{b or 148}{'_2' if rep else ''}", (1, 3, 0), (2048, 0, 0), b)
                    for rep in (0, 1) for b in (0, 132, 120, 104)),
}
for name, tune, bulk, *budget in VARIANTS[sys.argv[1] if len(sys.argv) > 1 else "default"]:
    check(LIB.fy_adamw_tune(*tune))
    check(LIB.fy_adamw_tune_bulk(*bulk))
    check(LIB.fy_adamw_sm_budget(budget[0] if budget else 0))
    step()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            time.sleep(0.02)
    th = threading.Thread(target=sampler)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    a.record()
    reps = 0
    t0 = time.time()
    while time.time() - t0 < 3.0:
        step()
        reps += 1
        if reps % 5 == 0:
            torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = a.elapsed_time(b) / reps
    tail = samples[len(samples) // 3:]  # steady part
    print(json.dumps({"variant": name, "ms_per_step": ms, "gbs": 28 * N * K / (ms * 1e-3) / 1e9,
                      "power_w_median": statistics.median(p for p, _ in tail),
                      "sm_mhz_median": statistics.median(c for _, c in tail), "samples": len(tail)}), flush=True)
check(LIB.fy_adamw_tune(1, 0, 0))
check(LIB.fy_adamw_tune_bulk(2048, 0, 0))
