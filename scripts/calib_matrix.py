#!/usr/bin/env python
"""Calibration matrix (diagnostic): executed vs DES-predicted vs analytic
makespan over more iterations than the GPU test holds (C1 b=8..128, 13B
slices of 4 / 8 blocks at b=8 / 32, a 65B slice with resident states, the
file tier). JSON lines."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import exec_api as X  # noqa: E402

sys.path.insert(0, str(ROOT / "scripts"))
from exec_cases import CASES as cases  # noqa: E402

for tag, (sc, opts) in cases.items():
    st, s, _, err = X.execute(sc, opts)
    if st != 0 and not s:
        print(json.dumps({"case": tag, "status": st, "error": err[:300]}), flush=True)
        continue
    ex = s["executed"]["makespan_s"]
    print(json.dumps({"case": tag, "status": st, "launch": s.get("launch"), "executed_s": ex,
                      "predicted_s": s["predicted"]["makespan_s"],
                      "des_err": abs(s["predicted"]["makespan_s"] - ex) / ex,
                      "analytic_s": s["analytic"]["t_iter_s"],
                      "analytic_err": abs(s["analytic"]["t_iter_s"] - ex) / ex,
                      "all_invariants_pass": s["all_invariants_pass"],
                      "tasks": s["task_count"]}), flush=True)
