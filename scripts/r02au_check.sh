# round 2, call au: file replay through the iteration's own buffers — executor /
# calibration / CLI / swap GPU tests, the swap file-leg probe, the default bench
OUT=gpurun_out; mkdir -p $OUT
(timeout 1500 python -m pytest tests/test_executor_gpu.py tests/test_calibration_gpu.py tests/test_cli_gpu.py tests/test_swap_gpu.py -q -p no:cacheprovider --timeout 900 > $OUT/r02au_pytest_exec.log 2>&1; echo "pytest rc=$?" >> $OUT/r02au_pytest_exec.log)
(timeout 600 python scripts/probes/swap_file_leg_probe.py default > $OUT/r02au_swap_file_leg.txt 2>&1; echo "rc=$?" >> $OUT/r02au_swap_file_leg.txt)
(timeout 900 python bench.py > $OUT/r02au_bench.json 2> $OUT/r02au_bench.err; echo "bench rc=$?" >> $OUT/r02au_bench.err)
