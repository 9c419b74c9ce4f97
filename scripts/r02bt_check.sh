# round 2, call bt: final tree — smoke + every GPU test (after the SM-budget changes)
OUT=gpurun_out; mkdir -p $OUT
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02bt_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r02bt_smoke.log)
(timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 900 > $OUT/r02bt_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02bt_pytest_gpu.log)
