# round 2, call bs: split + adam_quad from 16 CTAs — budget tests + kernel tests, budget sweep
OUT=gpurun_out; mkdir -p $OUT
(timeout 1500 python -m pytest tests/test_adamw_gpu.py tests/test_shard_gpu.py tests/test_pipeline_gpu.py -q -p no:cacheprovider --timeout 900 > $OUT/r02bs_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/r02bs_pytest.log)
(timeout 600 python scripts/budget_default_probe.py 6 8,16,32,48,64,96,128,0 > $OUT/r02bs_budget.jsonl 2>&1)
