"""Probe (r02bb): the C1 b=8 file-tier iteration executed N times in a row in
one process (bench's case: hardware with cpu_mem 1 GB would force SSD
checkpoints; here the bench's own options) — executed vs DES-predicted per
run and the file lane's busy time, to separate disk noise from the model."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import exec_api as X  # noqa: E402

sc = X.scenario(batch=8)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    for warm in (True, False):
        st, s, _, err = X.execute(sc, {"tier": "file", "file_dir": "/tmp/offsim_rep", "compute_rate": 1.4e15,
                                       "warm_files": warm})
        ex = s["executed"]["makespan_s"]
        pr = s["predicted"]["makespan_s"]
        r = s["measured_rates"]
        print(json.dumps({"run": i, "warm": warm, "status": st, "executed_s": ex, "predicted_s": pr,
                          "ratio": ex / pr, "warmup_s": s.get("file_warmup_s"),
                          "read_eff_gbs": r["file_read_effective_bps"] / 1e9,
                          "write_eff_gbs": r["file_write_effective_bps"] / 1e9,
                          "read_loaded_gbs": r.get("file_read_loaded_bps", 0) / 1e9,
                          "write_loaded_gbs": r.get("file_write_loaded_bps", 0) / 1e9,
                          "ssd_link_overlap": r.get("ssd_link_overlap"),
                          "legs": {k: round(v["gbs"], 2) for k, v in s["legs"].items() if "ssd" in k}}),
              flush=True)
