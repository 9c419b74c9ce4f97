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
     --no-streamed --no-cpu-baseline --no-swap-sweep --no-configs > $OUT/${TAG}_ncu_launch_run.log 2>&1; echo "ncu-launch rc=$?" >> $OUT/${TAG}_ncu_launch_run.log)
  # single-pass DRAM traffic of the fused kernel (no replay)
  (timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
     --clock-control none -k regex:adamw_ -c 6 --csv --log-file $OUT/${TAG}_traffic.csv \
     python scripts/ncu_target.py > $OUT/${TAG}_ncu_traffic_run.log 2>&1; echo "ncu-traffic rc=$?" >> $OUT/${TAG}_ncu_traffic_run.log)
  # full section set; application replay (kernel replay perturbs the TMA kernel)
  (timeout 1200 ncu --set full --replay-mode application --clock-control none --import-source on \
     -k regex:adamw_ -s 2 -c 1 -o $OUT/${TAG}_adamw python scripts/ncu_target.py \
     > $OUT/${TAG}_ncu_full_run.log 2>&1; echo "ncu-full rc=$?" >> $OUT/${TAG}_ncu_full_run.log)
fi
ls -la $OUT
