cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2f}
( timeout 200 python scripts/split_dev.py --trace ) 2>&1 | grep -v Warn | tee gpurun_out/${T}_split.log
timeout 900 python -m pytest tests/test_head_gpu.py tests/test_step_gpu.py tests/test_full_vocab_gpu.py -x -q 2>&1 | tail -5
