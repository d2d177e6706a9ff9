cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2m}
( timeout 200 python scripts/split_dev.py --trace ) 2>&1 | grep -v Warn | tee gpurun_out/${T}_split.log
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
