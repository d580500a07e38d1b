#!/bin/bash
# End-of-round refresh on one B200 (run under gpurun from the repo root):
#   every bench config's JSON line, the c5 launch list, ncu --set full of the dominant kernels
#   (c5: relight_tc + shift tile; c4: residue-plane kernels; c5s: vectorised gather), parity margins.
set -u
TAG=${1:-r01g}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for c in c5 c2 c3 c4 c5s c5t c5x c6r; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c exit=$?" >> $OUT/status.txt
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file $OUT/launches_c5.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch-list exit=$?" >> $OUT/status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"relight_tc_kernel|shift2d_tile_kernel" \
    -c 2 -o $OUT/prof_c5 $CMD > $OUT/ncu_c5.log 2>&1
echo "ncu c5 exit=$?" >> $OUT/status.txt
timeout 300 python scripts/run_c4.py 20000 1 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"planes_(a|c)_kernel" -c 2 \
    -o $OUT/prof_c4 python scripts/run_c4.py 20000 1 > $OUT/ncu_c4.log 2>&1
echo "ncu c4 exit=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"relight_sparse64" -c 1 \
    -o $OUT/prof_c5s python bench.py --config c5s --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_c5s.log 2>&1
echo "ncu c5s exit=$?" >> $OUT/status.txt
timeout 900 python scripts/parity_margins.py > $OUT/parity_margins.txt 2>&1
echo "margins exit=$?" >> $OUT/status.txt
