# round 2, call o: the bench's N>1 path through fy_shard with 2 ranks on
# the one GPU (plumbing only), then the full default bench (C5 legs)
OUT=gpurun_out; mkdir -p $OUT
FY_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --gather auto --layers 8 --steps 5 \
  --warmup 3 --no-e2e --shard-blocks 0 > $OUT/r02o_same_gpu_n2.json 2> $OUT/r02o_same_gpu_n2.err
echo "rc=$?" >> $OUT/r02o_same_gpu_n2.err
FY_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --layers 4 --steps 3 --warmup 3 \
  --shard-blocks 1 > $OUT/r02o_same_gpu_n2_full.json 2> $OUT/r02o_same_gpu_n2_full.err
echo "rc=$?" >> $OUT/r02o_same_gpu_n2_full.err
FY_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 \
  > $OUT/r02o_ref_n2.json 2> $OUT/r02o_ref_n2.err
echo "rc=$?" >> $OUT/r02o_ref_n2.err
(timeout 900 python bench.py > $OUT/r02o_bench.json 2> $OUT/r02o_bench.err; echo "bench rc=$?" >> $OUT/r02o_bench.err)
