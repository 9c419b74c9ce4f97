#!/bin/bash
# The bench's N>1 path with 2 ranks on the one GPU of a gpurun box (gloo group,
# CUDA IPC through torch symmetric memory): the fused update + all-gather
# epilogue across processes, the per-step device barrier and max-over-ranks.
# NOT a multi-GPU measurement (both ranks share one GPU's HBM bandwidth).
OUT=gpurun_out; mkdir -p $OUT
FY_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --gather auto --layers 8 --steps 5 \
  --warmup 3 --no-e2e --shard-blocks 0 > $OUT/same_gpu_ranks.json 2> $OUT/same_gpu_ranks.err
echo "rc=$?" >> $OUT/same_gpu_ranks.err
tail -5 $OUT/same_gpu_ranks.err; cat $OUT/same_gpu_ranks.json | tail -1 | cut -c1-600
# the streamed-shard phase and the e2e path at N=2 (gloo stages the CUDA
# all-gathers through host memory: plumbing only)
FY_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --layers 4 --steps 3 --warmup 3 \
  --shard-blocks 1 > $OUT/same_gpu_ranks_full.json 2> $OUT/same_gpu_ranks_full.err
echo "rc=$?" >> $OUT/same_gpu_ranks_full.err
