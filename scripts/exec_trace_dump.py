#!/usr/bin/env python
"""Dump executed traces (offsim_execute) + summaries for offline analysis of
executed vs planned makespan. Writes gpurun_out/exec_<tag>_{summary,trace}.json."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "scripts"))
import exec_api as X  # noqa: E402

out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
from exec_cases import CASES as cases  # noqa: E402
# args: [tag ...] [--opts JSON] (extra ExecOptions merged into every case)
args = sys.argv[1:]
extra = {}
if "--opts" in args:
    i = args.index("--opts")
    extra = json.loads(args[i + 1])
    del args[i:i + 2]
suffix = ""
if "--suffix" in args:
    i = args.index("--suffix")
    suffix = args[i + 1]
    del args[i:i + 2]
for tag in (args or list(cases)):
    sc, opts = cases[tag]
    opts = {**opts, **extra}
    st, summ, trace, err = X.execute(sc, opts, want_trace=True)
    (out / f"exec_{tag}{suffix}_summary.json").write_text(json.dumps(summ, indent=1))
    (out / f"exec_{tag}{suffix}_trace.json").write_text(trace or "")
    (out / f"exec_{tag}{suffix}_scenario.json").write_text(sc)
    print(tag, st, err, summ["executed"]["makespan_s"], summ["planned"]["makespan_s"])
