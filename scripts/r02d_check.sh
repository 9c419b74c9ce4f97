# round 2, call d: the two r02c failures, the default bench (OOM fix),
# executed-iteration traces (calibration analysis), the overlap / power
# probe, and a fresh ncu capture of the default fused kernel
OUT=gpurun_out; mkdir -p $OUT
(timeout 900 python -m pytest tests/test_shard_gpu.py tests/test_cli_gpu.py -q -m gpu -p no:cacheprovider --timeout 600 > $OUT/r02d_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02d_pytest_gpu.log)
(timeout 900 python bench.py > $OUT/r02d_bench.json 2> $OUT/r02d_bench.err; echo "bench rc=$?" >> $OUT/r02d_bench.err)
(timeout 900 python scripts/exec_trace_dump.py c1_b8 c1_b8_resident c1_b128 13b_4blk 13b_4blk_resident > $OUT/r02d_trace_dump.log 2>&1; echo "dump rc=$?" >> $OUT/r02d_trace_dump.log)
(timeout 600 python scripts/budget_overlap_probe.py 8 power,overlap > $OUT/r02d_overlap_power.jsonl 2>&1; echo "probe rc=$?" >> $OUT/r02d_overlap_power.jsonl)
(timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:adamw --csv python scripts/ncu_target.py > $OUT/r02d_traffic_single_pass.csv 2>&1; echo "ncu1 rc=$?" >> $OUT/r02d_traffic_single_pass.csv)
(timeout 900 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:adamw_bulk -c 1 -o $OUT/r02d_adamw_full python scripts/ncu_target.py > $OUT/r02d_ncu_full.log 2>&1; echo "ncu2 rc=$?" >> $OUT/r02d_ncu_full.log)
