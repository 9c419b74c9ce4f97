# round 2, call bp: adam_quad gated to the budgeted split shape (<= 80 CTAs): new uniform-math
# tests + all kernel tests, interleaved A/B vs the previous build, a default bench line
OUT=gpurun_out; mkdir -p $OUT
(timeout 1500 python -m pytest tests/test_adamw_gpu.py tests/test_fullsize_gpu.py -q -p no:cacheprovider --timeout 900 > $OUT/r02bp_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/r02bp_pytest.log)
: > $OUT/r02bp_ab.jsonl
LIBF=paper_2403_06504_b200/lib/liboffsim.so.0
for rep in 1 2; do for v in prev new; do
  cp build/ab/liboffsim_$v.so.0 $LIBF
  timeout 300 python scripts/budget_default_probe.py 6 2>/dev/null | sed "s/^{/{\"build\": \"$v\", \"rep\": $rep, /" >> $OUT/r02bp_ab.jsonl
done; done
cp build/ab/liboffsim_new.so.0 $LIBF
(timeout 900 python bench.py --no-e2e --no-streamed --no-cpu-baseline --no-swap-sweep --no-configs --no-iteration --shard-blocks 0 > $OUT/r02bp_bench.json 2> $OUT/r02bp_bench.err; echo "bench rc=$?" >> $OUT/r02bp_bench.err)
