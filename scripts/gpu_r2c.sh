cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2c}
( timeout 200 python scripts/split_dev.py --trace
  NANOSPEC_SPLIT_FLAGS=1 timeout 200 python scripts/split_dev.py
  NANOSPEC_SPLIT_FLAGS=2 timeout 200 python scripts/split_dev.py
  timeout 200 python scripts/split_dev.py --mode 2 ) 2>&1 | grep -v Warn | tee gpurun_out/${T}_split.log
