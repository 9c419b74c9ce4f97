# round 2, call bq: full check on the current tree — smoke, every GPU test,
# the default bench and the reference arm, plus an ncu launch list
OUT=gpurun_out; mkdir -p $OUT
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02bq_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r02bq_smoke.log)
(timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 900 > $OUT/r02bq_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02bq_pytest_gpu.log)
(timeout 900 python bench.py > $OUT/r02bq_bench.json 2> $OUT/r02bq_bench.err; echo "bench rc=$?" >> $OUT/r02bq_bench.err)
(timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/r02bq_ref.json 2> $OUT/r02bq_ref.err; echo "ref rc=$?" >> $OUT/r02bq_ref.err)
(timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r02bq_launch_list.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-streamed --no-cpu-baseline --no-swap-sweep --no-configs --no-iteration --shard-blocks 0 > $OUT/r02bq_ncu_bench.log 2>&1; echo "ncu rc=$?" >> $OUT/r02bq_ncu_bench.log)
