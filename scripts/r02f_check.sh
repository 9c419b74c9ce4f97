# round 2, call f: calibration with the compute replay (traces), the
# persisted b200-measured preset, and the world-W probe (connections)
OUT=gpurun_out; mkdir -p $OUT
(timeout 900 python scripts/exec_trace_dump.py c1_b8 c1_b8_resident c1_b128 13b_4blk 13b_4blk_resident > $OUT/r02f_trace_dump.log 2>&1; echo "dump rc=$?" >> $OUT/r02f_trace_dump.log)
(timeout 900 python scripts/calibrate_b200.py $OUT/b200_measured.json > $OUT/r02f_calibrate.log 2>&1; echo "cal rc=$?" >> $OUT/r02f_calibrate.log)
(timeout 1200 python scripts/world_probe.py > $OUT/r02f_world_probe.jsonl 2>&1; echo "probe rc=$?" >> $OUT/r02f_world_probe.jsonl)
