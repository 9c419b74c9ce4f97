OUT=gpurun_out; mkdir -p $OUT
nvidia-smi > $OUT/r02c_nvsmi.txt 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02c_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r02c_smoke.log)
(timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 > $OUT/r02c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/r02c_pytest_gpu.log)
(timeout 900 python bench.py > $OUT/r02c_bench.json 2> $OUT/r02c_bench.err; echo "bench rc=$?" >> $OUT/r02c_bench.err)
(timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/r02c_ref.json 2> $OUT/r02c_ref.err; echo "ref rc=$?" >> $OUT/r02c_ref.err)
