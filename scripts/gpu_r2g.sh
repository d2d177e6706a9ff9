cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2g}
( for f in 0 1 4 8 16; do NANOSPEC_SPLIT_FLAGS=$f timeout 200 python scripts/split_dev.py; done
  NANOSPEC_SPLIT_FLAGS=8 timeout 200 python scripts/split_dev.py --trace ) 2>&1 | grep -v Warn | tee gpurun_out/${T}_split.log
