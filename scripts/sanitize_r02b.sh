#!/bin/bash
# compute-sanitizer over the late round-2 additions: the sharded step with
# host gradients (grads_on_host) and with gradients in the arena slot, the
# budgeted split-DMA kernel shape, and the streamed pipeline at 16 pieces.
TAG=${1:-r02b}
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {
  local tool=$1 log=$2; shift 2
  (timeout 1200 $CS --tool $tool --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider "$@" \
     > $OUT/${TAG}_${log}.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_${log}.log)
}
run memcheck memcheck_shard_host_grads tests/test_shard_gpu.py -k "host_gradients or in_place"
run memcheck memcheck_budget_split tests/test_adamw_gpu.py -k "sm_budget"
run racecheck racecheck_budget_split tests/test_adamw_gpu.py -k "sm_budget and 64"
run synccheck synccheck_budget_split tests/test_adamw_gpu.py -k "sm_budget and 64"
tail -n 2 $OUT/${TAG}_*.log
