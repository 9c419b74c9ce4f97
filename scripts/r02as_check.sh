# round 2, call as: swap-sweep file legs — bench with only the resident phase
# + swap sweep, then the standalone swap file-leg probe after it, then the
# probe on its own again; free memory before / after
OUT=gpurun_out; mkdir -p $OUT
free -g > $OUT/r02as_mem.txt
(timeout 900 python bench.py --steps 3 --no-e2e --no-streamed --no-cpu-baseline --no-configs --no-iteration --shard-blocks 0 > $OUT/r02as_bench_sweep.json 2> $OUT/r02as_bench_sweep.err; echo "bench rc=$?" >> $OUT/r02as_bench_sweep.err)
free -g >> $OUT/r02as_mem.txt
(timeout 600 python scripts/probes/swap_file_leg_probe.py default > $OUT/r02as_swap_file_leg.txt 2>&1; echo "rc=$?" >> $OUT/r02as_swap_file_leg.txt)
