OUT=gpurun_out; mkdir -p $OUT
(timeout 1200 python -m pytest tests/test_shard_gpu.py -q -m gpu -p no:cacheprovider > $OUT/r02an_shard.log 2>&1; echo "rc=$?" >> $OUT/r02an_shard.log)
(timeout 600 python scripts/shard_overhead_probe.py > $OUT/r02an_shard_overhead.jsonl 2>&1)
(timeout 900 python bench.py --no-configs --no-swap-sweep --no-iteration --shard-blocks 0 --no-streamed --no-cpu-baseline > $OUT/r02an_bench.json 2> $OUT/r02an_bench.err; echo "rc=$?" >> $OUT/r02an_bench.err)
