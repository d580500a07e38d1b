#!/bin/bash
# End-of-round refresh on one B200 (run under gpurun from the repo root):
#   every bench config's JSON line, the c5 launch list, one ncu --set full capture per hot-path
#   kernel family (c5: relight_tc + the shift kernels; c4: residue planes; c3: GEMV; c2: small-face
#   shift + short-row GEMV; 1D shift; c6r: rotation; c5s: sparse gather; c5t: triple product; c7s:
#   the composed BRDF-rotated shading), and
#   the parity margins.  Each ncu capture runs only after its command exited 0 without ncu.
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
NCU="ncu --set full --clock-control none --import-source on"
for c in c5 c2 c3 c4 c5s c5t c5x c6r c7s; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c exit=$?" >> $OUT/status.txt
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file $OUT/launches_c5.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch-list exit=$?" >> $OUT/status.txt
timeout 1200 $NCU -k regex:"relight_tc_kernel|shift2d_band_kernel|band_finish_kernel" \
    -c 4 -o $OUT/prof_c5 $CMD > $OUT/ncu_c5.log 2>&1
echo "ncu c5 exit=$?" >> $OUT/status.txt
timeout 300 python scripts/run_c4.py 20000 1 > /dev/null 2>&1 && \
timeout 900 $NCU -k regex:"planes_(a|c|low)_kernel" -c 3 -o $OUT/prof_c4 python scripts/run_c4.py 20000 1 \
    > $OUT/ncu_c4.log 2>&1
echo "ncu c4 exit=$?" >> $OUT/status.txt
declare -A KRX=([c3]="shift2d_band|band_finish|relight_gemv" [c2]="shift2d_small|relight_gemv_short" [c6r]="rot_chainrule|rot_dc|rot_bottomup|rot_closure")
for c in c3 c2 c6r; do
  C2="python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 300 $C2 > /dev/null 2>&1 && \
  timeout 900 $NCU -k regex:"${KRX[$c]}" -c 6 -o $OUT/prof_$c $C2 > $OUT/ncu_$c.log 2>&1
  echo "ncu $c exit=$?" >> $OUT/status.txt
done
timeout 300 python scripts/run_shift1d.py 1 > /dev/null 2>&1 && \
timeout 900 $NCU -k regex:"shift1d_kernel" -c 1 -o $OUT/prof_shift1d python scripts/run_shift1d.py 1 \
    > $OUT/ncu_shift1d.log 2>&1
echo "ncu shift1d exit=$?" >> $OUT/status.txt
timeout 900 $NCU -k regex:"relight_sparse64" -c 1 \
    -o $OUT/prof_c5s python bench.py --config c5s --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_c5s.log 2>&1
echo "ncu c5s exit=$?" >> $OUT/status.txt
timeout 900 $NCU -k regex:"relight_triple_tc" -c 1 \
    -o $OUT/prof_c5t python bench.py --config c5t --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_c5t.log 2>&1
echo "ncu c5t exit=$?" >> $OUT/status.txt
timeout 900 $NCU -k regex:"relight_triple_tc|pack_qtree" -c 2 \
    -o $OUT/prof_c7s python bench.py --config c7s --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_c7s.log 2>&1
echo "ncu c7s exit=$?" >> $OUT/status.txt
timeout 900 python scripts/parity_margins.py > $OUT/parity_margins.txt 2>&1
echo "margins exit=$?" >> $OUT/status.txt
