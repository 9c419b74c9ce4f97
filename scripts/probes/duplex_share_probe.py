"""Probe (r02aq): can the host link give D2H more than its ~50 GB/s duplex
share when H2D is throttled? D2H copies 64 MiB pieces back to back (2 GiB);
H2D copies 64 MiB pieces separated by a spin kernel (torch.cuda._sleep) that
idles the H2D engine for a fraction `idle` of the time. Prints per-direction
GB/s over the D2H window and their sum, one JSON line per idle fraction."""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

dev = torch.device("cuda")
PIECE = 64 << 20
NP = 32


def host(nbytes):
    p = C.c_void_p()
    check(LIB.fy_host_alloc(nbytes, C.byref(p)))
    return torch.frombuffer((C.c_uint8 * nbytes).from_address(p.value), dtype=torch.uint8)


h_up, h_dn = host(PIECE * 4), host(PIECE * 4)
d_up = torch.empty(PIECE * 4, dtype=torch.uint8, device=dev)
d_dn = torch.empty(PIECE * 4, dtype=torch.uint8, device=dev)
up, dn = torch.cuda.Stream(), torch.cuda.Stream()

# cycles per ms of torch.cuda._sleep
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
torch.cuda._sleep(10_000_000)
b.record()
torch.cuda.synchronize()
cyc_per_ms = 10_000_000 / a.elapsed_time(b)


def copy_ms(direction):
    s = up if direction == "up" else dn
    with torch.cuda.stream(s):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(8):
            if direction == "up":
                d_up[(i % 4) * PIECE:(i % 4 + 1) * PIECE].copy_(h_up[(i % 4) * PIECE:(i % 4 + 1) * PIECE], non_blocking=True)
            else:
                h_dn[(i % 4) * PIECE:(i % 4 + 1) * PIECE].copy_(d_dn[(i % 4) * PIECE:(i % 4 + 1) * PIECE], non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 8


simplex = {"h2d_gbs": PIECE / copy_ms("up") / 1e6, "d2h_gbs": PIECE / copy_ms("down") / 1e6}
print(json.dumps({"simplex": simplex, "cyc_per_ms": cyc_per_ms}), flush=True)
piece_ms = PIECE / 50e9 * 1e3

for idle in [0.0, 0.05, 0.1, 0.15, 0.2, 0.25, 0.3, 0.4]:
    best = None
    for rep in range(3):
        torch.cuda.synchronize()
        go = torch.cuda.Event(enable_timing=True)
        go.record()
        up.wait_event(go)
        dn.wait_event(go)
        d_end = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(dn):
            for i in range(NP):
                j = i % 4
                h_dn[j * PIECE:(j + 1) * PIECE].copy_(d_dn[j * PIECE:(j + 1) * PIECE], non_blocking=True)
            d_end.record(dn)
        up_ends = []
        sleep_cyc = int(idle / (1 - idle) * piece_ms * cyc_per_ms) if idle > 0 else 0
        with torch.cuda.stream(up):
            for i in range(int(NP * 1.5)):
                j = i % 4
                d_up[j * PIECE:(j + 1) * PIECE].copy_(h_up[j * PIECE:(j + 1) * PIECE], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True)
                e.record(up)
                up_ends.append(e)
                if sleep_cyc:
                    torch.cuda._sleep(sleep_cyc)
        torch.cuda.synchronize()
        t_d = go.elapsed_time(d_end)
        n_up = sum(1 for e in up_ends if go.elapsed_time(e) <= t_d)
        r = {"idle": idle, "d2h_gbs": NP * PIECE / t_d / 1e6, "h2d_gbs": n_up * PIECE / t_d / 1e6}
        r["sum_gbs"] = r["d2h_gbs"] + r["h2d_gbs"]
        if best is None or r["d2h_gbs"] > best["d2h_gbs"]:
            best = r
    print(json.dumps(best), flush=True)
