#!/bin/bash
# Debug build of libhaarshift with per-phase clock64 instrumentation of the shift tile kernel.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/dbg
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
  --expt-relaxed-constexpr -Iinclude -Ipaper_1705_07272_b200/csrc -DHS_PHASE_TIMING \
  -c paper_1705_07272_b200/csrc/shift2d.cu -o build/dbg/shift2d.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC \
  -o paper_1705_07272_b200/lib/libhaarshift_dbg.so build/dbg/shift2d.o $(ls build/obj/*.o | grep -v shift2d)
