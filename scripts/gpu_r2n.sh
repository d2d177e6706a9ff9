cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2n}
( timeout 200 python scripts/split_dev.py --trace ) 2>&1 | grep -v Warn | tail -22 | tee gpurun_out/${T}_split.log
timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | cut -c1-1500
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
