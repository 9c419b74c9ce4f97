OUT=gpurun_out; mkdir -p $OUT
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02a_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r02a_smoke.log)
(timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 > $OUT/r02a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02a_pytest_gpu.log)
(timeout 600 python scripts/budget_overlap_probe.py 6 stages > $OUT/r02a_budget_stages.jsonl 2>&1; echo "probe rc=$?" >> $OUT/r02a_budget_stages.jsonl)
