#!/bin/bash
# compute-sanitizer over the round-2 code: the 16-consumer-warp TMA kernel
# (now the default) and its 512-consumer list kernel, the sharded step
# (fused peer-store epilogue + device barriers, streamed tier), the
# executor in CUDA-graph launch mode, and the step-counter trajectory.
TAG=${1:-r02}
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, log, pytest args...
  local tool=$1 log=$2; shift 2
  (timeout 1200 $CS --tool $tool --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider "$@" \
     > $OUT/${TAG}_${log}.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_${log}.log)
}
K16="tma_bulk_path_bit_exact and 14341 and (3-16 or 4-16) or bit_exact and 4099 or alias or nonfinite"
run memcheck memcheck_kernels16 tests/test_adamw_gpu.py -k "$K16"
run racecheck racecheck_kernels16 tests/test_adamw_gpu.py -k "tma_bulk_path_bit_exact and 14341 and (3-16 or 4-16)"
run synccheck synccheck_kernels16 tests/test_adamw_gpu.py -k "tma_bulk_path_bit_exact and 14341 and (3-16 or 4-16)"
run memcheck memcheck_list16 tests/test_adamw_gpu.py -k "multi_chunk_launch_bit_exact or batches_over_96"
run racecheck racecheck_list16 tests/test_adamw_gpu.py -k "multi_chunk_launch_bit_exact and tma"
run memcheck memcheck_shard tests/test_shard_gpu.py -k "world1 or single_process_peer and not world8"
run memcheck memcheck_executor_graph tests/test_executor_gpu.py -k "c1_overlapped_host_tier or resident_groups or gemm_dataflow"
run memcheck memcheck_trajectory tests/test_pipeline_gpu.py -k "trajectory or counter"
tail -n 2 $OUT/${TAG}_*.log
