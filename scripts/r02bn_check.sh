# round 2, call bn: warp-uniform divide / sqrt fast paths in the TMA consumer (adam_quad):
# kernel bit-exactness tests, the SM-budget sweep, a default bench line
OUT=gpurun_out; mkdir -p $OUT
(timeout 1500 python -m pytest tests/test_adamw_gpu.py tests/test_fullsize_gpu.py tests/test_pipeline_gpu.py tests/test_shard_gpu.py -q -p no:cacheprovider --timeout 900 > $OUT/r02bn_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/r02bn_pytest.log)
(timeout 600 python scripts/budget_default_probe.py 6 > $OUT/r02bn_budget_default.jsonl 2>&1)
(timeout 900 python bench.py --no-e2e --no-streamed --no-cpu-baseline --no-swap-sweep --no-configs --no-iteration --shard-blocks 0 > $OUT/r02bn_bench.json 2> $OUT/r02bn_bench.err; echo "bench rc=$?" >> $OUT/r02bn_bench.err)
