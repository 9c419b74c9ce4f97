# round 2, call q: ncu of the default (16-consumer-warp) fused kernel
OUT=gpurun_out; mkdir -p $OUT
(timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:adamw --csv python scripts/ncu_target.py > $OUT/r02q_traffic_single_pass.csv 2>&1; echo "ncu1 rc=$?" >> $OUT/r02q_traffic_single_pass.csv)
(timeout 900 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:adamw_bulk -c 1 -o $OUT/r02q_adamw_full python scripts/ncu_target.py > $OUT/r02q_ncu_full.log 2>&1; echo "ncu2 rc=$?" >> $OUT/r02q_ncu_full.log)
(timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r02q_launch_list.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-streamed --no-cpu-baseline --no-swap-sweep --no-configs --no-iteration --shard-blocks 0 > $OUT/r02q_ncu_bench.log 2>&1; echo "ncu3 rc=$?" >> $OUT/r02q_ncu_bench.log)
