"""A/B of io_uring registered (fixed) buffers on the SSD tier: the file-tier
iteration of a 13B-shaped slice (bench.ssd_tier_phase) with the staging
rings registered (READ/WRITE_FIXED) and not, alternating.
usage: python scripts/fixed_io_ab.py [blocks] [rounds]"""
import json
import sys

sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2403_06504_b200._lib as LIBM  # noqa: E402


class F:
    LIB = LIBM.LIB
    check = staticmethod(LIBM.check)


blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for i in range(rounds):
    for fixed in (True, False):
        r = bench.ssd_tier_phase(F, blocks=blocks, fixed_buffers=fixed)
        hp = r["hw_predicted"]
        print(json.dumps({"fixed": fixed, "round": i, "makespan_s": round(r["makespan_s"], 4),
                          "file_lane_gbs": r["file_lane_gbs"] and round(r["file_lane_gbs"], 3),
                          "cal_read_gbs": round(hp["bw_s2c"] / 1e9, 3), "cal_write_gbs": round(hp["bw_c2s"] / 1e9, 3),
                          "io_requests": r["io_requests"], "ok": r["all_invariants_pass"]}), flush=True)
