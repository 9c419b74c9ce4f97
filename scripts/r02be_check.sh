# round 2, call be: file replay under copy-engine load (blended by the planned file/link overlap):
# executor GPU tests, the C1 file-tier repeat probe, the 13B SSD-tier iteration, the default bench
OUT=gpurun_out; mkdir -p $OUT
(timeout 1500 python -m pytest tests/test_executor_gpu.py tests/test_calibration_gpu.py tests/test_cli_gpu.py -q -p no:cacheprovider --timeout 900 > $OUT/r02be_pytest_exec.log 2>&1; echo "pytest rc=$?" >> $OUT/r02be_pytest_exec.log)
(timeout 700 python scripts/probes/file_tier_repeat.py 3 > $OUT/r02be_file_tier_repeat.jsonl 2>&1)
(timeout 1200 python scripts/ssd_tier_run.py 8 > $OUT/r02be_ssd_tier_8blocks.json 2> $OUT/r02be_ssd_tier.err)
(timeout 900 python bench.py > $OUT/r02be_bench.json 2> $OUT/r02be_bench.err; echo "bench rc=$?" >> $OUT/r02be_bench.err)
