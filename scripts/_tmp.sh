cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_relight.py -q -x -k "shifted" 2>&1 | tail -2
python scripts/run_c4.py 20000 3
python bench.py --config c4 --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | head -c 300
