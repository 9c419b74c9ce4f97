"""CPU: the product library loads without a GPU and exports every function
declared in include/**/*.h (the drop-in boundary); pure-host entry points
behave (no CUDA compute is called here)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADERS = sorted((ROOT / "include").rglob("*.h"))
DECL = re.compile(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b((?:offsim|fy)_[a-z0-9_]+)\s*\(", re.M)


def declared():
    names = set()
    for h in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in DECL.finditer(text):
            if "typedef" in text[max(0, m.start() - 40):m.start() + 1].split("\n")[-1]:
                continue
            names.add(m.group(1))
    return sorted(names)


def test_headers_found():
    assert any(h.name == "fy_adam.h" for h in HEADERS)
    assert len(declared()) >= 10


@pytest.mark.parametrize("name", declared())
def test_symbol_exported(name):
    from paper_2403_06504_b200._lib import LIB
    assert hasattr(LIB, name), f"{name} declared in include/ but not exported"


def test_shard_range_partitions():
    from paper_2403_06504_b200 import optim as F
    for n in (1, 7, 8, 4099, 314572800, 7077888):
        for world in (1, 2, 3, 4, 8):
            covered = 0
            prev_end = 0
            for r in range(world):
                off, cnt = F.shard_range(n, world, r, 8)
                assert off == prev_end
                if r < world - 1 and cnt > 0 and off + cnt < n:
                    assert cnt % 8 == 0 and off % 8 == 0
                prev_end = off + cnt
                covered += cnt
            assert covered == n


def test_errors_are_status_codes():
    from paper_2403_06504_b200._lib import LIB, FY_ERR_CONFIG
    off, cnt = C.c_uint64(), C.c_uint64()
    assert LIB.fy_shard_range(10, 0, 0, 8, C.byref(off), C.byref(cnt)) == FY_ERR_CONFIG
    assert b"rank" in LIB.fy_last_error()
    assert LIB.fy_adamw_chunk(None, None) == FY_ERR_CONFIG
    assert LIB.fy_last_error() == b"null argument"
    assert LIB.fy_version().startswith(b"0.")
