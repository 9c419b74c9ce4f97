#!/usr/bin/env python
"""Diagnostic: executed vs DES-predicted makespan of small iterations in
both launch modes (CUDA graph vs per-task stream issue), a few repetitions
each. JSON lines."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import exec_api as X  # noqa: E402

cases = {
    "c1_b8_resident": (X.scenario(batch=8), {"tier": "host", "compute_rate": 1.4e15, "resident_groups": "all"}),
    "c1_b8": (X.scenario(batch=8), {"tier": "host", "compute_rate": 1.4e15}),
}
for tag, (sc, opts) in cases.items():
    for mode in ("graph", "stream"):
        for rep in range(3):
            st, s, _, err = X.execute(sc, {**opts, "launch": mode})
            print(json.dumps({"case": tag, "launch": s.get("launch"), "rep": rep,
                              "executed_ms": s["executed"]["makespan_s"] * 1e3,
                              "predicted_ms": s["predicted"]["makespan_s"] * 1e3,
                              "executed_over_predicted": s["executed_over_predicted"],
                              "busy_ms": {k: round(v * 1e3, 3) for k, v in s["executed"]["busy_s"].items()}}),
                  flush=True)
