#!/usr/bin/env python
"""Calibration: measure this box's engine rates through the
executor's own calibration (offsim_execute measured_rates) on two workloads
— a 4-block slice of the 13B shape with real bf16 GEMMs (large copies) and
GPT-2-small C1 (small copies) — and persist them as a named hardware preset,
`b200-measured`, next to the reference's modeled presets
(proj/src/presets.cpp:33-50): an inline-override object of the a100-12ssd
preset that any scenario can name as its "hardware" (the reference's own
scenario schema, no new keys).

  bw_gpu        host link per direction: the executed graph's own copies
                replayed one direction at a time (H2D, the binding lane of
                every measured iteration); per workload
  cpu_opt_tput  the fused Adam kernel (params/s, HBM-resident states)
  gpu_tput      bf16 cuBLAS FLOP/s of the model's own layer GEMMs replayed
                back to back (compute_effective_flops)
  bw_s2c/bw_c2s the file tier (O_DIRECT io_uring) when measured, else the
                preset's SSD array is kept
  gpu_mem/cpu_mem this box

usage: calibrate_b200.py [out.json]  (default paper_2403_06504_b200/presets/b200_measured.json)"""
import datetime
import json
import socket
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import exec_api as X  # noqa: E402

out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "paper_2403_06504_b200" / "presets" / "b200_measured.json"
runs = {
    "13b_4blk": (X.scenario(layers=4, heads=40, hidden=5120, batch=8, name="13b4"),
                 {"tier": "host", "compute_mode": "gemm"}),
    "c1_b8": (X.scenario(batch=8), {"tier": "host", "compute_mode": "gemm"}),
    "13b_file": (X.scenario(layers=2, heads=40, hidden=5120, batch=8, name="13b2"),
                 {"tier": "file", "file_dir": "/tmp/offsim_calibrate", "compute_mode": "gemm"}),
}
rates = {}
for tag, (sc, opts) in runs.items():
    st, summ, _, err = X.execute(sc, opts)
    if st != 0:
        print(f"{tag}: status {st} {err}", file=sys.stderr)
        continue
    rates[tag] = summ["measured_rates"]
big, small = rates["13b_4blk"], rates.get("c1_b8", {})
f = rates.get("13b_file", {})
hw = {"preset": "a100-12ssd", "name": "b200-measured",
      "bw_gpu": big["h2d_simplex_effective_bps"],
      "cpu_opt_tput": big["optimizer_params_per_s"],
      "gpu_tput": big.get("compute_effective_flops") or big["compute_flops"],
      "gpu_mem": 180000000000}
if f.get("file_read_effective_bps"):
    hw.update(n_ssd=1, bw_s2c=f["file_read_effective_bps"], bw_c2s=f["file_write_effective_bps"])
doc = {"hardware": hw,
       "per_workload_bw_gpu": {"13b_shape_large_copies": big["h2d_simplex_effective_bps"],
                               "c1_small_copies": small.get("h2d_simplex_effective_bps")},
       "provenance": {"when": datetime.datetime.now(datetime.timezone.utc).isoformat(timespec="seconds"),
                      "host": socket.gethostname(), "script": "scripts/calibrate_b200.py",
                      "measured_rates": rates}}
out.parent.mkdir(parents=True, exist_ok=True)
out.write_text(json.dumps(doc, indent=1) + "\n")
print(json.dumps(doc["hardware"]))
