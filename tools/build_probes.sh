#!/bin/bash
# Rebuild libcosched_b200.so WITH the timing-probe instances (-DCS_TIMING_PROBES;
# they return wrong results by design -- GPU-box experiments only, never commit
# the resulting .so).  Usage: bash tools/build_probes.sh
ROOT=$(cd "$(dirname "$0")/.." && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCS_TIMING_PROBES \
  -Xcompiler -fPIC,-O3 -shared -cudart static -I$ROOT/include $ROOT/paper_2405_03831_b200/csrc/sweep.cu \
  -o $ROOT/paper_2405_03831_b200/libcosched_b200.so
