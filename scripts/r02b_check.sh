OUT=gpurun_out; mkdir -p $OUT
(timeout 1500 python -m pytest tests/test_shard_gpu.py tests/test_pipeline_gpu.py tests/test_cli_gpu.py tests/test_adamw_gpu.py -q -m gpu -p no:cacheprovider --timeout 600 -x > $OUT/r02b_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02b_pytest_gpu.log)
(timeout 600 python scripts/budget_overlap_probe.py 6 stages > $OUT/r02b_budget_stages.jsonl 2>&1; echo "probe rc=$?" >> $OUT/r02b_budget_stages.jsonl)
(timeout 900 python bench.py --steps 5 --warmup 3 --no-swap-sweep --no-configs --shard-blocks 1 > $OUT/r02b_bench.json 2> $OUT/r02b_bench.err; echo "bench rc=$?" >> $OUT/r02b_bench.err)
(FY_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --layers 8 --steps 5 \
  --warmup 3 --no-e2e --shard-blocks 1 > $OUT/r02b_same_gpu_n2.json 2> $OUT/r02b_same_gpu_n2.err; echo "rc=$?" >> $OUT/r02b_same_gpu_n2.err)
