#!/usr/bin/env python
"""Probe: H2D / D2H copy rate vs copy size from cudaHostAlloc memory (torch
pin_memory) and from fy_host_alloc memory (mmap + mbind + cudaHostRegister),
copies back to back from one 1.25 GB buffer, median of 5 passes."""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

TOTAL = 5 * 256 << 20
dev = torch.device("cuda")
d = torch.empty(TOTAL, dtype=torch.uint8, device=dev)
pin = torch.empty(TOTAL, dtype=torch.uint8, pin_memory=True)
p = C.c_void_p()
check(LIB.fy_host_alloc(TOTAL, C.byref(p)))
reg = torch.frombuffer((C.c_uint8 * TOTAL).from_address(p.value), dtype=torch.uint8)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, h in (("cudaHostAlloc", pin), ("fy_host_alloc", reg)):
    for mb in (16, 64, 160, 640):
        size = mb << 20
        for direction in ("h2d", "d2h"):
            rates = []
            for _ in range(5):
                torch.cuda.synchronize()
                a.record()
                for off in range(0, TOTAL - size + 1, size):
                    if direction == "h2d":
                        d[off:off + size].copy_(h[off:off + size], non_blocking=True)
                    else:
                        h[off:off + size].copy_(d[off:off + size], non_blocking=True)
                b.record()
                torch.cuda.synchronize()
                n = (TOTAL // size) * size
                rates.append(n / (a.elapsed_time(b) * 1e-3) / 1e9)
            print(json.dumps({"alloc": name, "copy_mb": mb, "dir": direction,
                              "gbs_median": statistics.median(rates)}), flush=True)
check(LIB.fy_host_free(p))
