# round 2, call h: kernel preloading (lazy-loading deadlock fix) — world
# probe, then the full GPU suite, smoke and the default bench
OUT=gpurun_out; mkdir -p $OUT
(FY_BARRIER_TIMEOUT_S=60 timeout 900 python scripts/world_probe.py 2:8 4:32 8:8 8:32 > $OUT/r02h_world_probe.jsonl 2>&1; echo "probe rc=$?" >> $OUT/r02h_world_probe.jsonl)
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02h_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r02h_smoke.log)
(timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 900 > $OUT/r02h_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02h_pytest_gpu.log)
(timeout 900 python bench.py > $OUT/r02h_bench.json 2> $OUT/r02h_bench.err; echo "bench rc=$?" >> $OUT/r02h_bench.err)
