"""SSD-tier iteration of a 13B-shaped slice with the tier files in one
directory vs striped over N directories (bench.ssd_tier_phase). On a box
with one disk every directory is the same device: this checks the striped
path end to end (all invariants, bit-checked swaps) and that it costs
nothing; on an NVMe array each directory would be one SSD.
usage: python scripts/stripe_ab.py [blocks] [dirs] [rounds]"""
import json
import sys

sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2403_06504_b200._lib as LIBM  # noqa: E402


class F:
    LIB = LIBM.LIB
    check = staticmethod(LIBM.check)


blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ndirs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for i in range(rounds):
    for fd in ("/tmp/offsim_ssd_tier", [f"/tmp/offsim_ssd_tier_{d}" for d in range(ndirs)]):
        r = bench.ssd_tier_phase(F, blocks=blocks, file_dir=fd)
        hp = r["hw_predicted"]
        print(json.dumps({"devices": r["file_devices"], "round": i, "makespan_s": round(r["makespan_s"], 4),
                          "file_lane_gbs": r["file_lane_gbs"] and round(r["file_lane_gbs"], 3),
                          "cal_read_gbs": round(hp["bw_s2c"] / 1e9, 3), "cal_write_gbs": round(hp["bw_c2s"] / 1e9, 3),
                          "executed_over_predicted": round(r["executed_over_predicted"], 3),
                          "ok": r["all_invariants_pass"]}), flush=True)
