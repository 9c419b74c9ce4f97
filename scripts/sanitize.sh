#!/bin/bash
# compute-sanitizer passes over the fused kernels, the chunk pipeline and the
# executor (race detection / memory checking of K1).
# Usage (under gpurun): bash scripts/sanitize.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="bit_exact and (4099 or 1048579) or tma_bulk_path_bit_exact and 14341 or alias or nonfinite or unaligned"
(timeout 900 $CS --tool memcheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "$SEL" > $OUT/${TAG}_memcheck_kernels.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_memcheck_kernels.log)
(timeout 900 $CS --tool memcheck --error-exitcode 9 \
   python -m pytest tests/test_pipeline_gpu.py -q -x > $OUT/${TAG}_memcheck_pipeline.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_memcheck_pipeline.log)
(timeout 900 $CS --tool racecheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "tma_bulk_path_bit_exact and 14341 or bit_exact and 4099" > $OUT/${TAG}_racecheck.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_racecheck.log)
(timeout 900 $CS --tool synccheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "tma_bulk_path_bit_exact and 14341" > $OUT/${TAG}_synccheck.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_synccheck.log)
(timeout 1200 $CS --tool memcheck --error-exitcode 9 \
   python -m pytest tests/test_executor_gpu.py -q -x -k "c1_overlapped_host_tier or swap_only" > $OUT/${TAG}_memcheck_executor.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_memcheck_executor.log)
# round-1 session-2 additions: multi-chunk list kernel, device-side clip /
# skip controls, TMA sweep variants (split DMA warps, tiles, L2 hints)
NEW="multi_chunk_launch_bit_exact or batches_over_96 or device_side_clipping or sweep_variants and 22541"
(timeout 900 $CS --tool memcheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "$NEW" > $OUT/${TAG}_memcheck_new_kernels.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_memcheck_new_kernels.log)
(timeout 900 $CS --tool racecheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "multi_chunk_launch_bit_exact and tma or sweep_variants and 22541" > $OUT/${TAG}_racecheck_new_kernels.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_racecheck_new_kernels.log)
(timeout 900 $CS --tool synccheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "multi_chunk_launch_bit_exact and tma or sweep_variants and 22541" > $OUT/${TAG}_synccheck_new_kernels.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_synccheck_new_kernels.log)
(timeout 900 $CS --tool memcheck --error-exitcode 9 \
   python -m pytest tests/test_swap_gpu.py -q -x > $OUT/${TAG}_memcheck_swap.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_memcheck_swap.log)
# fp32 gradients on the TMA path (18 B/element stages)
FP32="tma_bulk_path_bit_exact and 14341 and 2- or multi_chunk_launch_bit_exact and tma and 2-"
(timeout 900 $CS --tool memcheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "$FP32" > $OUT/${TAG}_memcheck_fp32.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_memcheck_fp32.log)
(timeout 900 $CS --tool racecheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "$FP32" > $OUT/${TAG}_racecheck_fp32.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_racecheck_fp32.log)
(timeout 900 $CS --tool synccheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "$FP32" > $OUT/${TAG}_synccheck_fp32.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_synccheck_fp32.log)
# the vectorised grad-stats pass (16-B loads, unaligned / ragged fallbacks)
(timeout 900 $CS --tool memcheck --error-exitcode 9 \
   python -m pytest tests/test_adamw_gpu.py -q -x -k "grad_stats or device_side_clipping" > $OUT/${TAG}_memcheck_grad_stats.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_memcheck_grad_stats.log)
tail -n 3 $OUT/${TAG}_*check*.log
