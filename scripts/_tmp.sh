cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shift.py tests/test_gpu_coarse.py tests/test_gpu_relight.py -x -q 2>&1 | tail -4
python scripts/run_shift_c5.py c5 20
python scripts/run_shift_c5.py c5 20
