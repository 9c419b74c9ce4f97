#!/bin/bash
# One GPU session: smoke, GPU tests, bench, ncu launch list + full capture.
# Usage (under gpurun): bash scripts/gpu_check.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi -L > $OUT/${TAG}_gpu.txt 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/${TAG}_smoke.log)
(timeout 900 python -m pytest tests -x -q -m gpu > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log)
if [ "${SWEEP:-0}" = "1" ]; then
  (timeout 600 python scripts/kernel_sweep.py > $OUT/${TAG}_sweep.log 2>&1; echo "sweep rc=$?" >> $OUT/${TAG}_sweep.log)
fi
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  (timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?" >> $OUT/${TAG}_bench.err)
fi
if [ "${SKIP_NCU:-0}" != "1" ]; then
  (timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'adamw|reduce_partials|grad_stats' -c 400 --csv \
     --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e \
     --no-streamed --no-cpu-baseline --no-swap-sweep > $OUT/${TAG}_ncu_launch_run.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/${TAG}_ncu_launch_run.log)
  # hardware-counter sections only: the SASS-patching sections (SourceCounters,
  # InstructionStats) instrument the TMA kernel's mbarrier spin-waits and
  # inflate both its duration and its DRAM traffic
  (timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables \
     --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats \
     --section ComputeWorkloadAnalysis --clock-control none -k regex:adamw_bulk -s 4 -c 1 \
     -o $OUT/${TAG}_adamw_hw python bench.py --steps 1 --warmup 1 --layers 6 --no-e2e --no-streamed \
     --no-cpu-baseline --no-swap-sweep > $OUT/${TAG}_ncu_hw_run.log 2>&1; echo "ncu-hw rc=$?" >> $OUT/${TAG}_ncu_hw_run.log)
  (timeout 900 ncu --set full --clock-control none --import-source on -k regex:adamw_bulk -s 4 -c 1 --target-processes all \
     -o $OUT/${TAG}_adamw python bench.py --steps 1 --warmup 1 --layers 6 --no-e2e --no-streamed \
     --no-cpu-baseline --no-swap-sweep > $OUT/${TAG}_ncu_full_run.log 2>&1; echo "ncu-full rc=$?" >> $OUT/${TAG}_ncu_full_run.log)
fi
ls -la $OUT
