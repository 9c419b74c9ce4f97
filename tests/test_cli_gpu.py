"""GPU: the CLI's `execute` subcommand on the B200 (the
reference's trace export proj/src/trace_export.cpp:46-93 and CLI
proj/tools/offsim_main.cpp:112-225): `build/offsim execute ... --trace t.json`
runs a whole C1 iteration on real engines and writes a Chrome trace of the
EXECUTED timeline. Checks: exit status 0; the summary reports every
invariant passing; the trace has one thread (tid) per lane with its name,
events sorted by start time within each lane, one complete ("X") event per
executed task, copy-engine lanes present, and per lane the event durations
summing to the summary's busy_s."""
import json
import subprocess
from collections import defaultdict
from pathlib import Path

import pytest

from exec_api import scenario

pytestmark = pytest.mark.gpu

EXE = Path(__file__).resolve().parents[1] / "build" / "offsim"
LANES = {"GPU compute", "CPU compute", "CPU to GPU", "GPU to CPU", "SSD array"}


@pytest.mark.parametrize("variant", ["overlapped", "pipelined"])
def test_cli_execute_writes_valid_executed_trace(cuda_dev, tmp_path, variant):
    if not EXE.exists():
        pytest.skip("build/offsim not built")
    sc = tmp_path / "c1.json"
    sc.write_text(scenario(variant=variant))
    tr = tmp_path / "t.json"
    out = tmp_path / "summary.json"
    # the pipelined variant stages gradients through the SSD tier: files
    opts = {"tier": "host", "compute_rate": 1.4e15}
    if variant == "pipelined":
        opts = {"tier": "file", "file_dir": str(tmp_path / "tier"), "compute_rate": 1.4e15}
    r = subprocess.run([str(EXE), "execute", "--scenario", str(sc), "--exec",
                        json.dumps(opts), "--trace", str(tr),
                        "--out", str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    s = json.loads(out.read_text())
    assert s["all_invariants_pass"], [e for e in s["invariants"] if not e["pass"]]
    d = json.loads(tr.read_text())
    ev = d["traceEvents"]
    names = {e["tid"]: e["args"]["name"] for e in ev if e.get("ph") == "M" and e["name"] == "thread_name"}
    assert set(names.values()) == LANES and len(names) == len(LANES)  # one tid per lane
    xs = [e for e in ev if e.get("ph") == "X"]
    assert len(xs) == s["task_count"]  # one complete event per executed task
    per_lane = defaultdict(list)
    for e in xs:
        assert e["tid"] in names
        per_lane[names[e["tid"]]].append(e)
    # the copy engines really ran (host <-> device legs of the optimizer)
    assert per_lane["CPU to GPU"] and per_lane["GPU to CPU"]
    busy = s["executed"]["busy_s"]
    key = {"GPU compute": "gpu_compute", "CPU compute": "cpu_compute", "CPU to GPU": "link_c2g",
           "GPU to CPU": "link_g2c", "SSD array": "link_ssd"}
    for lane, evs in per_lane.items():
        ts = [e["ts"] for e in evs]
        assert ts == sorted(ts), f"{lane}: events not sorted by start"
        total_s = sum(e["dur"] for e in evs) * 1e-6
        assert abs(total_s - busy[key[lane]]) <= 1e-6 * max(1.0, len(evs)) + 1e-3 * busy[key[lane]], lane
    # one X event per executed task (task names unique per event)
    assert len({e["name"] for e in xs}) == len(xs)
