"""SSD-tier iteration of a 13B-shaped slice (bench.ssd_tier_phase) at several
io_uring depths per device: where does this box's disk saturate?
usage: python scripts/io_depth_sweep.py [blocks] [depth ...]"""
import json
import sys

sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2403_06504_b200._lib as LIBM  # noqa: E402


class F:
    LIB = LIBM.LIB
    check = staticmethod(LIBM.check)


blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
depths = [int(x) for x in sys.argv[2:]] or [4, 8, 32, 128, 32]
for d in depths:
    r = bench.ssd_tier_phase(F, blocks=blocks, io_depth=d)
    hp = r["hw_predicted"]
    print(json.dumps({"io_depth": d, "makespan_s": round(r["makespan_s"], 4),
                      "file_lane_gbs": r["file_lane_gbs"] and round(r["file_lane_gbs"], 3),
                      "cal_read_gbs": round(hp["bw_s2c"] / 1e9, 3), "cal_write_gbs": round(hp["bw_c2s"] / 1e9, 3),
                      "ok": r["all_invariants_pass"]}), flush=True)
