#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root).
#   1) bench (plain) -> gpurun_out/bench.log
#   2) launch list of the same short bench command under ncu (cold-cache, serialised)
#   3) ncu --set full of the relight and shift kernels (one launch each)
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo "bench exit=$?" >> gpurun_out/bench_${TAG}.log
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch-list exit=$?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"relight_tc_kernel|shift2d_tile_kernel|relight_tc_prep" \
    -c 3 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full exit=$?" >> gpurun_out/ncu_full_${TAG}.log
