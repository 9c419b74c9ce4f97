# round 2, call ah: e2e through fy_shard (host grads) — default bench and
# the N=2 same-GPU plumbing run
OUT=gpurun_out; mkdir -p $OUT
(timeout 900 python bench.py > $OUT/r02ah_bench.json 2> $OUT/r02ah_bench.err; echo "bench rc=$?" >> $OUT/r02ah_bench.err)
FY_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --layers 4 --steps 3 --warmup 3 \
  --shard-blocks 1 > $OUT/r02ah_same_gpu_n2_full.json 2> $OUT/r02ah_same_gpu_n2_full.err
echo "rc=$?" >> $OUT/r02ah_same_gpu_n2_full.err
