cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; echo "bench rc=$?"; cat gpurun_out/bench_r01c.json | head -c 2500
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 192 -c 40 --csv --log-file gpurun_out/c5t_launches2.csv python bench.py --config c5t --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c5t_ncu3.log 2>&1; echo "ncu rc=$?"
