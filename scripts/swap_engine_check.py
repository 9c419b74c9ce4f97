"""Runs bench.swap_engine_phase alone (the fy_swapper_* activation swap engine)."""
import json, sys
sys.argv = ['bench.py']
sys.path.insert(0, '.')
import torch, bench
import paper_2403_06504_b200._lib as LIBM
import paper_2403_06504_b200.optim as optim
class F:
    LIB = LIBM.LIB
    check = staticmethod(LIBM.check)
F.optim = optim
print(json.dumps(bench.swap_engine_phase(torch, F), indent=1))
