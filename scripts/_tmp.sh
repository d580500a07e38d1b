cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01e
python bench.py > gpurun_out/r01e/bench_c5.json 2>/dev/null; echo c5 $?
for c in c5x c4 c3 c2 c5s c5t c6r; do python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/r01e/bench_$c.json 2>/dev/null; echo $c $?; done
