# round 2, call e: executor in CUDA-graph launch mode (traces for the
# calibration analysis, stream mode beside it), executor / CLI GPU tests,
# and the single-process world-W shard probe
OUT=gpurun_out; mkdir -p $OUT
(timeout 900 python scripts/exec_trace_dump.py c1_b8 c1_b8_resident c1_b128 13b_4blk 13b_4blk_resident > $OUT/r02e_trace_dump.log 2>&1; echo "dump rc=$?" >> $OUT/r02e_trace_dump.log)
(timeout 600 python scripts/exec_trace_dump.py c1_b8_resident c1_b128 --suffix _stream --opts '{"launch": "stream"}' > $OUT/r02e_trace_dump_stream.log 2>&1)
(timeout 1200 python -m pytest tests/test_executor_gpu.py tests/test_cli_gpu.py -q -m gpu -p no:cacheprovider --timeout 600 > $OUT/r02e_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02e_pytest_gpu.log)
(timeout 1500 python scripts/world_probe.py > $OUT/r02e_world_probe.jsonl 2>&1; echo "probe rc=$?" >> $OUT/r02e_world_probe.jsonl)
