"""CPU: bit-exact parity of the offsim core restatement (planner, schedule
builder, DES, trace checks, reports, C ABI) with the compiled reference.

Three layers of evidence:
  1. tests/parity/offsim_dump.cpp compiled against THIS repo's headers and
     core (build/offsim_dump) reproduces the committed digests generated from
     the reference build (tests/golden/offsim_parity_digests.txt): every
     SwapPlan field (doubles compared as hex floats), task, dependency,
     memory effect, DES event time, invariant and per-(lane, payload) byte
     total over 729 cases incl. the 220-scenario acceptance matrix;
  2. every C-ABI output of the product library hashes to the reference's
     (tests/golden/offsim_capi_golden.json);
  3. when the reference build is present (oracle/_ref), the same outputs are
     compared live, byte for byte.
"""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT / "tests"))

from offsim_capi import capi_outputs, load_offsim  # noqa: E402

PRODUCT = ROOT / "paper_2403_06504_b200" / "lib" / "liboffsim.so.0"
REF_SO = ROOT / "oracle" / "_ref" / "liboffsim_ref.so"
REF_DUMP = ROOT / "oracle" / "_ref" / "offsim_dump_ref"


def _lines(text):
    return [l.split(" ", 2) for l in text.strip().splitlines()]


@pytest.fixture(scope="module")
def my_dump():
    exe = ROOT / "build" / "offsim_dump"
    assert exe.exists(), "build/offsim_dump missing: run __graft_entry__.build()"
    return subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout


def test_dump_digests_match_reference_golden(my_dump):
    gold = _lines((GOLD / "offsim_parity_digests.txt").read_text())
    mine = _lines(my_dump)
    assert len(mine) == len(gold) == 729
    bad = [(g[0], g[1], m[1]) for g, m in zip(gold, mine) if g[:2] != m[:2]]
    assert not bad, f"{len(bad)} cases differ, first: {bad[:5]}"


def test_dump_covers_acceptance_matrix_and_configs(my_dump):
    names = [l[0] for l in _lines(my_dump)]
    assert sum(n.startswith("matrix/") for n in names) == 660
    assert any(n.startswith("cfg/C5-13b-s2048-b64") for n in names)
    assert any(n.startswith("preset/175b-4090-b8") for n in names)


@pytest.mark.skipif(not REF_DUMP.exists(), reason="reference build absent (GPU box)")
def test_dump_matches_live_reference(my_dump):
    ref = subprocess.run([str(REF_DUMP)], check=True, capture_output=True, text=True).stdout
    assert ref == my_dump


def test_capi_outputs_match_reference_golden():
    mine = capi_outputs(load_offsim(PRODUCT), hashed=True)
    gold = json.loads((GOLD / "offsim_capi_golden.json").read_text())
    assert set(mine) == set(gold)
    bad = sorted(k for k in gold if mine[k] != gold[k])
    assert not bad, f"{len(bad)} C-ABI outputs differ: {bad[:8]}"


def _outputs_in_subprocess(lib_path):
    # one library per process: both export the same C and C++ symbols, and
    # GNU-unique template statics would be shared between them in-process
    code = ("import json,sys; sys.path.insert(0, %r); from offsim_capi import capi_outputs, "
            "load_offsim; print(json.dumps(capi_outputs(load_offsim(%r), hashed=False)))"
            % (str(ROOT / "tests"), str(lib_path)))
    out = subprocess.run([sys.executable, "-c", code], check=True, capture_output=True, text=True)
    return json.loads(out.stdout)


@pytest.mark.skipif(not REF_SO.exists(), reason="reference build absent (GPU box)")
def test_capi_outputs_match_live_reference():
    mine = _outputs_in_subprocess(PRODUCT)
    ref = _outputs_in_subprocess(REF_SO)
    assert set(mine) == set(ref)
    for k in ref:
        assert mine[k] == ref[k], f"{k} differs"


def test_swap_plan_goldens_from_baseline_md():
    """BASELINE.md §2 / SURVEY.md A9: 13B s=2048 sweep on a100 — coefficients
    0/0/1/1, swapped layers 0/0/160/160, d_f 3.36/6.71/134.2/268.4 GB, cpu."""
    lines = {l[0]: l for l in _lines((GOLD / "offsim_parity_digests.txt").read_text())}
    expect = {8: ("3355443200", "n=0"), 16: ("6710886400", "n=0"),
              32: ("134217728000", "n=160"), 64: ("268435456000", "n=160")}
    for b, (d_f, n) in expect.items():
        summary = lines[f"cfg/C5-13b-s2048-b{b}/overlapped"][2]
        fields = summary.split()
        assert fields[2] == d_f and n in summary and fields[6] == "0", summary
