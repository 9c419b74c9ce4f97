"""Executed-iteration cases shared by scripts/exec_trace_dump.py and
scripts/calib_matrix.py: (scenario JSON, offsim_execute options)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
import exec_api as X  # noqa: E402

CASES = {
    "c1_b8": (X.scenario(batch=8), {"tier": "host", "compute_rate": 1.4e15}),
    "c1_b128": (X.scenario(batch=128), {"tier": "host", "compute_rate": 1.4e15}),
    "13b_4blk": (X.scenario(layers=4, heads=40, hidden=5120, batch=8, name="13b4"),
                 {"tier": "host", "compute_mode": "gemm"}),
    "c1_b8_resident": (X.scenario(batch=8), {"tier": "host", "compute_rate": 1.4e15,
                                             "resident_groups": "all"}),
    "c1_b32": (X.scenario(batch=32), {"tier": "host", "compute_rate": 1.4e15}),
    "c1_b64": (X.scenario(batch=64), {"tier": "host", "compute_rate": 1.4e15}),
    "13b_8blk": (X.scenario(layers=8, heads=40, hidden=5120, batch=8, name="13b8"),
                 {"tier": "host", "compute_mode": "gemm_dataflow"}),
    "13b_8blk_b32": (X.scenario(layers=8, heads=40, hidden=5120, batch=32, name="13b8"),
                     {"tier": "host", "compute_mode": "gemm_dataflow"}),
    "65b_4blk_resident": (X.scenario(layers=4, heads=64, hidden=8192, batch=8, name="65b4"),
                          {"tier": "host", "compute_mode": "gemm_dataflow", "resident_groups": "all"}),
    "c1_b8_file": (X.scenario(batch=8), {"tier": "file", "file_dir": "/tmp/offsim_dump_file", "compute_rate": 1.4e15}),
    "13b_2blk_file": (X.scenario(layers=2, heads=40, hidden=5120, batch=8, name="13b2"),
                      {"tier": "file", "file_dir": "/tmp/offsim_dump_file", "compute_mode": "gemm"}),
    "13b_4blk_resident": (X.scenario(layers=4, heads=40, hidden=5120, batch=8, name="13b4"),
                          {"tier": "host", "compute_mode": "gemm_dataflow", "resident_groups": "all"}),
}
