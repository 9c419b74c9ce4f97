#!/usr/bin/env python
"""One iteration of an 8-block 13B-shaped slice with optimizer states in
O_DIRECT files streamed through 3-slot pinned rings (bench.ssd_tier_phase),
printed as JSON (the SSD tier at scale; opt-in in the bench)."""
import ctypes as C  # noqa: F401
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2403_06504_b200._lib as LIBM  # noqa: E402


class F:
    LIB = LIBM.LIB


print(json.dumps(bench.ssd_tier_phase(F, blocks=int(sys.argv[1]) if len(sys.argv) > 1 else 8)))
