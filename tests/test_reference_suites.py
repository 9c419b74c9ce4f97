"""CPU: the reference's OWN test suites, unmodified, run against this repo's
implementation (drop-in check of the C++ API and the C ABI):
  build/ref_unit_tests_on_b200   proj/tests/test_{workload,hardware,cost_model,
                                 planner,sim,capacity,scenario}.cpp + main.cpp
                                 on the doctest shim, linked to this core
  build/ref_capi_tests_on_b200   proj/tests/test_capi.cpp linked to
                                 paper_2403_06504_b200/lib/liboffsim.so.0
  build/ref_acceptance_on_b200   proj/tests/acceptance/acceptance_main.cpp
They are compiled by `make reftests` where /root/reference exists; the shim
is calibrated by the same suites passing against the compiled reference
(oracle/_ref/ref_unit_tests, ref_capi_tests)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITES = ["workload", "hardware", "cost_model", "planner", "sim", "capacity", "scenario"]


def _run(exe, *args):
    if not exe.exists():
        pytest.skip(f"{exe.name} not built (needs /root/reference at build time)")
    return subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_on_b200_core(suite):
    r = _run(ROOT / "build" / "ref_unit_tests_on_b200", f"--test-suite={suite}")
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout and "test cases: 0 " not in r.stdout


def test_reference_capi_suite_on_product_library():
    r = _run(ROOT / "build" / "ref_capi_tests_on_b200")
    assert r.returncode == 0, r.stderr[-2000:]
    assert "6 passed" in r.stdout


def test_reference_acceptance_on_b200_core():
    r = _run(ROOT / "build" / "ref_acceptance_on_b200")
    assert r.returncode == 0, r.stdout[-2000:]
    assert "ACCEPTANCE: 9/9 criteria passed" in r.stdout


def test_reference_acceptance_c8_with_this_cli():
    """Acceptance C8's subprocess half (byte-identical reruns of plan /
    simulate+trace / sweep / capacity / validate through the CLI binary,
    acceptance_main.cpp:471-525) — the reference skips it when no CLI is
    built; here it runs against this repo's CLI (tools/offsim_main.cpp, C ABI
    only)."""
    import os
    cli = ROOT / "build" / "offsim"
    if not cli.exists():
        pytest.skip("build/offsim not built")
    exe = ROOT / "build" / "ref_acceptance_on_b200"
    if not exe.exists():
        pytest.skip("ref_acceptance_on_b200 not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900,
                       env={**os.environ, "OFFSIM_CLI": str(cli)})
    assert r.returncode == 0, r.stdout[-2000:]
    assert "ACCEPTANCE: 9/9 criteria passed" in r.stdout
    c8 = [ln for ln in r.stdout.splitlines() if ln.startswith("CRITERION 8 [PASS]")]
    assert c8 and "CLI" in c8[0] and "library level only" not in r.stdout


def test_shim_calibrated_against_reference():
    r = _run(ROOT / "oracle" / "_ref" / "ref_unit_tests")
    assert r.returncode == 0 and "54 passed" in r.stdout
