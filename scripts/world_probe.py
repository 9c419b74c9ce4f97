#!/usr/bin/env python
"""Diagnostic: W shards in ONE process on one GPU (fused peer-store gather,
device barriers) for several W and CUDA_DEVICE_MAX_CONNECTIONS values, each
in its own subprocess with a short barrier timeout. Prints one JSON line per
run: pass / fail, wall time, error tail."""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

root = Path(__file__).resolve().parents[1]
runs = [(w, c) for w in (2, 4, 8) for c in (8, 32)]
if len(sys.argv) > 1:
    runs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]]  # world:connections
for world, conns in runs:
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS=str(conns), FY_BARRIER_TIMEOUT_S=os.environ.get("FY_BARRIER_TIMEOUT_S", "60"),
               PYTHONPATH=f"{root}:{root / 'tests'}:" + os.environ.get("PYTHONPATH", ""))
    t0 = time.time()
    r = subprocess.run([sys.executable, "-c",
                        f"import torch, test_shard_gpu as t; t.single_process_peer(torch.device('cuda:0'), {world}, 'device');"
                        "print('OK')"], env=env, capture_output=True, text=True, timeout=300, cwd=root)
    print(json.dumps({"world": world, "connections": conns, "ok": r.returncode == 0 and "OK" in r.stdout,
                      "wall_s": round(time.time() - t0, 1), "err": r.stderr[-400:]}), flush=True)
