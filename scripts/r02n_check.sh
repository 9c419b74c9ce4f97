# round 2, call n: 16 consumer warps by default — A/Bs, kernel tests, bench
OUT=gpurun_out; mkdir -p $OUT
(timeout 600 python scripts/stages_ab.py 20 6 0:0,3:8 > $OUT/r02n_stages_ab.jsonl 2>&1)
(timeout 600 python scripts/warps_ab.py > $OUT/r02n_warps_ab.jsonl 2>&1)
(timeout 1800 python -m pytest tests/test_adamw_gpu.py tests/test_shard_gpu.py tests/test_pipeline_gpu.py -q -m gpu -p no:cacheprovider --timeout 900 > $OUT/r02n_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02n_pytest_gpu.log)
(timeout 900 python bench.py > $OUT/r02n_bench.json 2> $OUT/r02n_bench.err; echo "bench rc=$?" >> $OUT/r02n_bench.err)
