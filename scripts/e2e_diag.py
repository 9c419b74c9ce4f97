#!/usr/bin/env python
"""A/B of the e2e pipeline shape (bench.py e2e: 13B set, HBM states, host
bf16 grads in / params out): pieces per block x staging slots, interleaved
rounds, per-direction link rates from the pipeline's own events."""
import ctypes as C
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402
from paper_2403_06504_b200._lib import LIB, check  # noqa: E402

L, N = 40, 12 * 5120 * 5120
dev = torch.device("cuda")
states = [torch.rand(3 * N, device=dev) * 1e-3 for _ in range(L)]
hbuf = []
for k in range(L):
    p = C.c_void_p()
    check(LIB.fy_host_alloc(2 * N, C.byref(p)))
    hbuf.append(p)
    np.ctypeslib.as_array((C.c_uint16 * N).from_address(p.value))[:] = 0x3A83
hp = F.Hparams()
configs = [(1, 3), (1, 4), (2, 3), (4, 3), (4, 4)]
pipes = {}
for P, S in configs:
    bounds = [min(N, (N * q // P + 7) // 8 * 8) for q in range(P)] + [N]
    spans = [(a, b) for a, b in zip(bounds, bounds[1:]) if b > a]
    pipe = F.ChunkPipeline(max(b - a for a, b in spans), slots=S, grads_on_host=True, params_to_host=True,
                           states_on_device=True)
    chunks = [dict(n=b - a, h_states=states[k].data_ptr() + 4 * a, states_stride=N, grad=hbuf[k].value + 2 * a,
                   h_param=hbuf[k].value + 2 * a) for k in range(L) for a, b in spans]
    pipes[(P, S)] = (pipe, chunks)
res = {c: [] for c in configs}
for rnd in range(4):
    for c in configs:
        pipe, chunks = pipes[c]
        pipe.step(chunks, hp)
        pipe.wait()
        t0 = time.perf_counter()
        for _ in range(2):
            pipe.step(chunks, hp)
            pipe.wait()
        el = (time.perf_counter() - t0) / 2
        if rnd > 0:
            res[c].append(2 * N * L / el / 1e9)
for c in configs:
    print(json.dumps({"pieces": c[0], "slots": c[1], "each_way_gbs_median": statistics.median(res[c]),
                      "all": [round(x, 2) for x in res[c]]}))
