#!/usr/bin/env python
"""Probe: can the fused kernel drive the host link itself (zero-copy)?

The streamed step and the e2e path move optimizer data over PCIe with the
copy engines (cudaMemcpyAsync into HBM staging, then the kernel). Pinned host
memory is mapped into the GPU's address space (UVA), so the fused kernel can
instead load/store host memory directly — LSU loads or cp.async.bulk — and
skip the staging round trip through HBM. This script measures, on one B200:

  copy engines : H2D, D2H and concurrent H2D+D2H of 1 GiB (pinned)
  e2e-zc       : one 13B chunk (314.6M params), states in HBM, bf16 grads
                 read from and bf16 params written to pinned host memory by
                 the kernel (2 B/param each way over the link)
  streamed-zc  : master/m/v in pinned host memory read and written by the
                 kernel (12 B/param each way), grads in HBM, bf16 params
                 written to pinned host (14 B/param D2H in total)

for the LSU path (fy_adamw_tune path 0) and the TMA bulk path (path 1), and
checks every zero-copy result bit-exactly against the same step run on HBM.
Output: one JSON object per line on stdout.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402
from paper_2403_06504_b200 import optim as F  # noqa: E402

dev = torch.device("cuda:0")
GiB = 1 << 30


def timed(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) * 1e-3)
    return best


def copy_engines():
    h = torch.empty(GiB, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(GiB, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(GiB, dtype=torch.uint8, device=dev)
    d2 = torch.empty(GiB, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timed(lambda: h.copy_(d, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    t_both = timed(both)
    return {"probe": "copy_engines", "h2d_gbs": GiB / t_h2d / 1e9, "d2h_gbs": GiB / t_d2h / 1e9,
            "duplex_each_gbs": GiB / t_both / 1e9}


def states(n, where, seed):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    p = torch.empty(n, device=dev).normal_(0, 0.02, generator=g)
    m = torch.empty(n, device=dev).normal_(0, 1e-3, generator=g)
    v = torch.empty(n, device=dev).normal_(0, 1e-3, generator=g).square_()
    gr = (torch.randn(n, device=dev, generator=g) * 1e-3).to(torch.bfloat16)
    if where == "host":
        p, m, v = (x.cpu().pin_memory() for x in (p, m, v))
    return p, m, v, gr


def run_case(name, n, states_on_host, grads_on_host, params_on_host, path, stages_or_unroll, reps=4):
    check(LIB.fy_adamw_tune(path, stages_or_unroll, 0))
    hp = F.Hparams()
    p, m, v, gr = states(n, "host" if states_on_host else "dev", 7)
    # reference: the same step entirely in HBM
    rp, rm, rv = (x.to(dev).clone() for x in (p, m, v))
    rout = torch.empty(n, dtype=torch.bfloat16, device=dev)
    check(LIB.fy_adamw_tune(1, 0, 0))
    F.adamw_chunk(rp, rm, rv, gr, hp, param_out=rout, stream=torch.cuda.current_stream(dev))
    torch.cuda.synchronize()
    check(LIB.fy_adamw_tune(path, stages_or_unroll, 0))
    g_in = gr.cpu().pin_memory() if grads_on_host else gr
    out = torch.empty(n, dtype=torch.bfloat16, pin_memory=True) if params_on_host else \
        torch.empty(n, dtype=torch.bfloat16, device=dev)
    # one checked step on copies of the initial states
    cp, cm, cv = (x.clone() if not states_on_host else x.clone().pin_memory() for x in (p, m, v))
    F.adamw_chunk(cp, cm, cv, g_in, hp, param_out=out, stream=torch.cuda.current_stream(dev))
    torch.cuda.synchronize()
    exact = all(torch.equal(a.to(dev).view(torch.int32), b.view(torch.int32))
                for a, b in ((cp, rp), (cm, rm), (cv, rv)))
    exact = exact and torch.equal(out.to(dev).view(torch.int16), rout.view(torch.int16))
    del cp, cm, cv, rp, rm, rv, rout
    t = timed(lambda: F.adamw_chunk(p, m, v, g_in, hp, param_out=out,
                                      stream=torch.cuda.current_stream(dev)), reps)
    h2d = n * ((12 if states_on_host else 0) + (2 if grads_on_host else 0))
    d2h = n * ((12 if states_on_host else 0) + (2 if params_on_host else 0))
    res = {"probe": name, "path": "tma" if path == 1 else "lsu", "knob": stages_or_unroll, "n": n,
           "s": t, "params_per_s": n / t, "link_h2d_gbs": h2d / t / 1e9, "link_d2h_gbs": d2h / t / 1e9,
           "bit_exact_vs_hbm": bool(exact)}
    check(LIB.fy_adamw_tune(1, 0, 0))
    return res


def main(argv):
    """argv: cases like `ce`, `e2e:0:4` (probe:path:knob), `str:1:3`; each
    case is best run in its own process (a fault must not poison the rest)."""
    n13 = 12 * 5120 * 5120
    n_s = 100 * 1000 * 1024  # 1.2 GB per fp32 state array
    for case in argv or ["ce"]:
        if case == "ce":
            print(json.dumps(copy_engines()), flush=True)
            continue
        kind, path, knob = case.split(":")
        try:
            if kind == "e2e":
                r = run_case("e2e_zc", n13, False, True, True, int(path), int(knob))
            else:
                r = run_case("streamed_zc", n_s, True, False, True, int(path), int(knob), reps=3)
            print(json.dumps(r), flush=True)
        except Exception as e:  # probe: report and continue
            print(json.dumps({"probe": case, "error": str(e)}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
