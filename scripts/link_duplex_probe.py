#!/usr/bin/env python
"""Probe: does the host link deliver more duplex bandwidth with more copy
streams per direction (several copy engines) or other copy sizes?
Prints one JSON line per configuration: per-direction GB/s with H2D and
D2H running concurrently, k streams each, each stream copying `size` chunks
back to back (1 GiB total per direction), pinned memory from fy_host_alloc."""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

dev = torch.device("cuda")
TOTAL = 1 << 30


def host(nbytes):
    p = C.c_void_p()
    check(LIB.fy_host_alloc(nbytes, C.byref(p)))
    return p, torch.frombuffer((C.c_uint8 * nbytes).from_address(p.value), dtype=torch.uint8)


hp_up, h_up = host(TOTAL)
hp_dn, h_dn = host(TOTAL)
d_up = torch.empty(TOTAL, dtype=torch.uint8, device=dev)
d_dn = torch.empty(TOTAL, dtype=torch.uint8, device=dev)


def run(k, size, directions=("up", "down")):
    ups = [torch.cuda.Stream() for _ in range(k)]
    dns = [torch.cuda.Stream() for _ in range(k)]
    best = {}
    for _ in range(3):
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        ends = {}
        for name, streams, dst, src in (("up", ups, d_up, h_up), ("down", dns, h_dn, d_dn)):
            if name not in directions:
                continue
            evs = []
            for i, s in enumerate(streams):
                s.wait_event(start)
                with torch.cuda.stream(s):
                    for off in range(i * size, TOTAL, k * size):
                        n = min(size, TOTAL - off)
                        dst[off:off + n].copy_(src[off:off + n], non_blocking=True)
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(s)
                    evs.append(e)
            ends[name] = evs
        torch.cuda.synchronize()
        for name, evs in ends.items():
            t = max(start.elapsed_time(e) for e in evs) * 1e-3
            best[name] = max(best.get(name, 0.0), TOTAL / t / 1e9)
    return best


for k in (1, 2, 4):
    for size in (16 << 20, 64 << 20, 256 << 20):
        print(json.dumps({"streams_per_dir": k, "copy_mb": size >> 20, "duplex_gbs": run(k, size)}), flush=True)
print(json.dumps({"simplex_h2d": run(1, 256 << 20, ("up",)), "simplex_d2h": run(1, 256 << 20, ("down",))}))
check(LIB.fy_host_free(hp_up))
check(LIB.fy_host_free(hp_dn))
