#!/bin/bash
# Exercises the bench's distributed plumbing on one GPU: torchrun with one
# rank, the fused-gather path (symmetric-memory rendezvous, peer-pointer
# epilogue, device barrier) and the reference arm under torchrun.
OUT=gpurun_out; TAG=${1:-r01}
mkdir -p $OUT
(timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
   --master-port 29517 bench.py --gpus 1 --gather fused --layers 20 --steps 5 --warmup 3 \
   --no-streamed --no-cpu-baseline --no-swap-sweep > $OUT/${TAG}_fused_gather.json 2> $OUT/${TAG}_fused_gather.err; \
   echo "rc=$?" >> $OUT/${TAG}_fused_gather.err)
(timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
   --master-port 29518 bench.py --gpus 1 --impl reference --steps 5 --warmup 3 \
   > $OUT/${TAG}_reference_arm.json 2> $OUT/${TAG}_reference_arm.err; echo "rc=$?" >> $OUT/${TAG}_reference_arm.err)
tail -n 3 $OUT/${TAG}_fused_gather.err $OUT/${TAG}_reference_arm.err
