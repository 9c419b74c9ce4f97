"""Probe (r02aq): the C5 swap sweep's file READ leg (b=8, forced SSD
placement) runs at 0.55-0.69 of the run's own replayed read rate, while a
standalone IoEngine write-then-reverse-read of the same 40 x 84 MB pattern
reads at 4.5-5.2 GB/s (r02aq_file_rw.txt). Executes the swap-only iteration
with its trace and prints, per file-lane task, start / duration / GB/s and
what else was running, under a few option variants."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import exec_api as X  # noqa: E402

sc = json.dumps({"schema_version": 1, "model": {"preset": "gpt3-13b", "batch_size": 8, "seq_len": 2048},
                 "hardware": "a100-12ssd", "variant": "overlapped"})
variants = {
    "default": {},
    "no_verify": {"verify_swaps": False},
    "no_fixed": {"fixed_buffers": False},
    "stream_launch": {"launch": "stream"},
}
only = sys.argv[1:] or list(variants)
for name in only:
    opts = {"tier": "file", "swap_only": True, "max_blocks": 40, "placement": "ssd",
            "file_dir": "/tmp/offsim_swap"}
    opts.update(variants[name])
    st, summ, tr, err = X.execute(sc, opts, want_trace=True)
    t = json.loads(tr)["traceEvents"]
    lanes = {e["tid"]: e["args"]["name"] for e in t if e.get("ph") == "M" and "args" in e}
    evs = sorted([(lanes.get(e["tid"], str(e["tid"])), e["name"], e["ts"], e["dur"]) for e in t
                  if e.get("ph") == "X"], key=lambda x: x[2])
    if name == only[0]:
        print(json.dumps({"lanes": sorted(set(lanes.values()))}), flush=True)
    fl = [e for e in evs if "ssd" in e[0].lower()]
    rd = [e for e in fl if "s2c" in e[1]]
    wr = [e for e in fl if "c2s" in e[1]]
    legs = summ.get("legs", {})
    rates = summ.get("measured_rates", {})
    print(json.dumps({"variant": name, "status": st, "err": err,
                      "makespan_s": summ["executed"]["makespan_s"],
                      "read_leg": legs.get("link_ssd/s2c/activations"),
                      "write_leg": legs.get("link_ssd/c2s/activations"),
                      "file_read_bps": rates.get("file_read_bps"),
                      "file_read_effective_bps": rates.get("file_read_effective_bps"),
                      "n_read_events": len(rd), "n_write_events": len(wr)}), flush=True)
    if name == only[0]:
        for e in wr[:3] + wr[-2:] + rd[:8] + rd[-3:]:
            other = [o[0] + ":" + o[1] for o in evs if o is not e and o[2] < e[2] + e[3] and o[2] + o[3] > e[2]]
            print("  ", e[0], e[1], "ts_ms %.2f dur_ms %.2f" % (e[2] / 1e3, e[3] / 1e3), "overlaps", other[:6])
