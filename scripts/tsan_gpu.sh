#!/bin/bash
# ThreadSanitizer over the GPU host pipeline: the whole
# library (C++ core + CUDA host code; -fsanitize=thread on the host side
# only) and tests/parity/host_pipeline_driver.cpp. `build` cross-compiles
# here (no GPU needed); `run` executes on a B200 box:
#   bash scripts/tsan_gpu.sh build
#   gpurun -- 'bash scripts/tsan_gpu.sh run'
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=$ROOT/build/tsan_gpu
if [ "$1" = "build" ]; then
  mkdir -p $B
  JSON=$(python3 -c "import os,sysconfig;print(os.path.join(sysconfig.get_paths()['purelib'],'include','cudnn_frontend','thirdparty','nlohmann'))")
  for f in $ROOT/paper_2403_06504_b200/csrc/core/*.cpp; do
    g++ -std=c++20 -O1 -g -fsanitize=thread -fPIC -I$ROOT/include -I$JSON -c $f -o $B/$(basename $f .cpp).o &
  done
  for f in $ROOT/paper_2403_06504_b200/csrc/cuda/*.cu; do
    /usr/local/cuda/bin/nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fsanitize=thread,-g \
      -I$ROOT/include -c $f -o $B/$(basename $f .cu).cu.o &
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fsanitize=thread \
    -o $B/liboffsim_tsan.so $B/*.o -lpthread -L/usr/local/cuda/lib64 -lcublas -Xlinker -rpath=/usr/local/cuda/lib64
  g++ -std=c++17 -O1 -g -fsanitize=thread -I$ROOT/include -I/usr/local/cuda/include \
    $ROOT/tests/parity/host_pipeline_driver.cpp -L$B -l:liboffsim_tsan.so -Wl,-rpath,$B \
    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,/usr/local/cuda/lib64 -pthread -o $B/host_pipeline_driver
  echo built $B/host_pipeline_driver
elif [ "$1" = "run" ]; then
  OUT=$ROOT/gpurun_out; mkdir -p $OUT
  D=$(mktemp -d)
  TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 second_deadlock_stack=1" \
    timeout 900 $B/host_pipeline_driver $D > $OUT/tsan_gpu.log 2>&1; echo "rc=$?" >> $OUT/tsan_gpu.log
  rm -rf $D
  echo "$(grep -c 'WARNING: ThreadSanitizer' $OUT/tsan_gpu.log) TSAN warnings; $(tail -2 $OUT/tsan_gpu.log | tr '\n' ' ')"
fi
