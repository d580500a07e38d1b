cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shift.py tests/test_gpu_coarse.py -x -q 2>&1 | tail -2
python scripts/run_shift_c5.py c5 20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"shift2d_tile|coarse_" -c 3 --csv python scripts/run_shift_c5.py c5 1 2>/dev/null | grep -E "coarse|tile" | cut -c1-200
