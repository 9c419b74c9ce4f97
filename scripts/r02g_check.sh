# round 2, call g: end-only instrumentation; calibration preset, traces,
# calibration / executor / CLI GPU tests
OUT=gpurun_out; mkdir -p $OUT
(timeout 900 python scripts/calibrate_b200.py > $OUT/r02g_calibrate.log 2>&1; echo "cal rc=$?" >> $OUT/r02g_calibrate.log; cp paper_2403_06504_b200/presets/b200_measured.json $OUT/b200_measured.json)
(timeout 900 python scripts/exec_trace_dump.py c1_b8 c1_b8_resident c1_b128 13b_4blk 13b_4blk_resident > $OUT/r02g_trace_dump.log 2>&1; echo "dump rc=$?" >> $OUT/r02g_trace_dump.log)
(timeout 1500 python -m pytest tests/test_calibration_gpu.py tests/test_executor_gpu.py tests/test_cli_gpu.py -q -s -m gpu -p no:cacheprovider --timeout 600 > $OUT/r02g_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02g_pytest_gpu.log)
