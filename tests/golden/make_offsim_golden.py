"""Generate the committed offsim parity fixtures from the COMPILED REFERENCE.

Requires oracle/_ref (built by `make ref` from /root/reference sources):
  * tests/golden/offsim_parity_digests.txt — output of oracle/_ref/offsim_dump_ref
    (one fnv1a digest of the canonical plan/graph/DES-trace/invariant dump per
    case: scenario presets x variants, BASELINE configs C1-C5, planner modes,
    and the 220-scenario acceptance matrix x 3 variants);
  * tests/golden/offsim_capi_golden.json — sha256 of every C-ABI output
    (offsim_plan / _simulate summary+trace / _validate / _scenario_to_json /
    _preset_names / _sweep / _capacity, and status+last_error of error paths)
    produced by oracle/_ref/liboffsim_ref.so.

Run: python tests/golden/make_offsim_golden.py
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "tests"))

from offsim_capi import capi_outputs, load_offsim  # noqa: E402


def main():
    ref_dump = ROOT / "oracle" / "_ref" / "offsim_dump_ref"
    out = subprocess.run([str(ref_dump)], check=True, capture_output=True, text=True).stdout
    (ROOT / "tests" / "golden" / "offsim_parity_digests.txt").write_text(out)
    lib = load_offsim(ROOT / "oracle" / "_ref" / "liboffsim_ref.so")
    golden = {k: v for k, v in capi_outputs(lib, hashed=True).items()}
    (ROOT / "tests" / "golden" / "offsim_capi_golden.json").write_text(
        json.dumps(golden, indent=1, sort_keys=True) + "\n")
    print(f"{len(out.splitlines())} digests, {len(golden)} C-ABI outputs")


if __name__ == "__main__":
    main()
