cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2o}
timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | cut -c1-1500
( timeout 200 python scripts/split_dev.py ) 2>&1 | grep -v Warn | tail -3
timeout 1500 python -m pytest tests/test_parity_r2_gpu.py tests/test_head_gpu.py tests/test_step_gpu.py -x -q 2>&1 | tail -4
