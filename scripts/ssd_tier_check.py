"""Runs bench.ssd_tier_phase alone: one file-tier (SSD) iteration of a 13B-shaped slice.
usage: python scripts/ssd_tier_check.py [blocks]"""
import json, sys
ARGS = sys.argv[1:]
sys.path.insert(0,'.')
import bench
import paper_2403_06504_b200._lib as LIBM
class F:
    LIB = LIBM.LIB
    check = staticmethod(LIBM.check)
r = bench.ssd_tier_phase(F, blocks=int(ARGS[0]) if ARGS else 4)
print(json.dumps(r, indent=1))
