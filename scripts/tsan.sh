#!/bin/bash
# ThreadSanitizer pass over the host-side C++ ("TSAN on the host
# pipeline"): the offsim core + C ABI built with -fsanitize=thread (CPU only;
# the CUDA executor is stubbed by tests/parity/tsan_exec_stub.cpp), running the
# reference's own unit suites, its C ABI suite (thread-local last error,
# sweep worker pool) and its acceptance binary (220-scenario matrix, sweeps
# with 4 workers, CLI-free reruns). Needs /root/reference (build container).
# Usage: bash scripts/tsan.sh [outdir]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=${1:-$ROOT/gpurun_out}
B=$(mktemp -d)
R=/root/reference/proj
JSON=$(python3 -c "import os,sysconfig;print(os.path.join(sysconfig.get_paths()['purelib'],'include','cudnn_frontend','thirdparty','nlohmann'))")
SH=$ROOT/tests/parity/doctest_shim
CXX="g++ -std=c++20 -O1 -g -fsanitize=thread -fPIC -I$ROOT/include -I$JSON"
for f in $ROOT/paper_2403_06504_b200/csrc/core/*.cpp $ROOT/tests/parity/tsan_exec_stub.cpp; do
  $CXX -c $f -o $B/$(basename $f .cpp).o &
done
wait
CORE="$B/cost_model.o $B/des.o $B/geometry.o $B/orchestration.o $B/schedule.o"
$CXX -I$SH $R/tests/main.cpp $R/tests/test_{workload,hardware,cost_model,planner,sim,capacity,scenario}.cpp $CORE -pthread -o $B/unit
$CXX -I$SH $R/tests/test_capi.cpp $B/capi.o $B/capi_exec.o $B/tier_map.o $B/io_engine.o $B/tsan_exec_stub.o $CORE -pthread -o $B/capi
$CXX $R/tests/acceptance/acceptance_main.cpp $CORE -pthread -o $B/acc
mkdir -p $OUT
export TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0"
for t in unit capi acc; do
  (timeout 1800 $B/$t > $OUT/tsan_$t.log 2>&1; echo "rc=$?" >> $OUT/tsan_$t.log)
  echo "$t: $(grep -c 'WARNING: ThreadSanitizer' $OUT/tsan_$t.log) TSAN warnings; $(tail -2 $OUT/tsan_$t.log | head -1)"
done
rm -rf $B
