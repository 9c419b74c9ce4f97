"""CPU: the CLI (tools/offsim_main.cpp, links the C ABI only) passes the
reference's CLI smoke tests (proj/tests/CMakeLists.txt:29-36) and adds
`execute` (dry run here; the GPU run is covered by test_executor_gpu)."""
import json
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parents[1] / "build" / "offsim"


def run(*args):
    if not EXE.exists():
        pytest.skip("build/offsim not built")
    return subprocess.run([str(EXE), *args], capture_output=True, text=True, timeout=120)


def test_reference_cli_smoke_tests():
    assert run("plan", "--preset", "13b-a100-b32").returncode == 0
    assert run("simulate", "--preset", "13b-a100-b32", "--variant", "serial").returncode == 0
    assert run("validate", "--preset", "13b-a100-b32").returncode == 0
    assert run("presets").returncode == 0
    assert run("plan").returncode != 0                                             # WILL_FAIL
    assert run("plan", "--preset", "175b-4090-b8", "--batch", "96").returncode == 3  # infeasible


def test_execute_dry_run_and_trace(tmp_path):
    r = run("execute", "--preset", "13b-a100-b8", "--exec", '{"dry_run": true}')
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    assert d["dry_run"] and d["all_invariants_pass"]
    tr = tmp_path / "t.json"
    r = run("simulate", "--preset", "13b-a100-b8", "--trace", str(tr))
    assert r.returncode == 0 and json.loads(tr.read_text())["traceEvents"]
