"""CPU: the C-ABI headers are plain C (a C caller — cgo, a C runtime, the
INTEGRATION.md §4 snippet — compiles them with -std=c11 -Wall -Werror) and
the snippet links against the product library."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2403_06504_b200" / "lib"


def test_c_abi_headers_compile_and_link_as_c11(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc missing")
    if not (LIB / "liboffsim.so.0").exists():
        pytest.skip("library not built")
    exe = tmp_path / "snippet"
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                        str(ROOT / "tests" / "parity" / "c_abi_shard_snippet.c"), f"-L{LIB}", "-l:liboffsim.so.0",
                        f"-Wl,-rpath,{LIB}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert exe.exists()
