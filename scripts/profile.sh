#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root).
#   1) default bench (plain)                       -> gpurun_out/bench_${TAG}.log
#   2) launch list of a short bench under ncu     -> gpurun_out/launches_${TAG}.csv
#   3) ncu --set full of relight_tc / shift tile  -> gpurun_out/prof_${TAG}.ncu-rep
#   4) ncu --set full of the fused c4 residue-plane kernels -> gpurun_out/prof_c4_${TAG}.ncu-rep
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench exit=$?" >> gpurun_out/bench_${TAG}.log
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch-list exit=$?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"relight_tc_kernel|shift2d_tile_kernel" \
    -c 2 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full exit=$?" >> gpurun_out/ncu_full_${TAG}.log
timeout 300 python scripts/run_c4.py 20000 1 > gpurun_out/c4plain_${TAG}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"planes_(a|c)_kernel" -c 2 \
    -o gpurun_out/prof_c4_${TAG} python scripts/run_c4.py 20000 1 > gpurun_out/ncu_c4_${TAG}.log 2>&1
echo "c4 exit=$?" >> gpurun_out/ncu_c4_${TAG}.log
