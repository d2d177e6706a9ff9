# round-2 iteration: pair kernel check + timing vs the cluster head, then GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 300 python scripts/pair_dev.py 2>&1 | tail -40 > gpurun_out/${T}_pair_dev.log; tail -40 gpurun_out/${T}_pair_dev.log
for m in -1 2 6; do MODE=$m timeout 120 python scripts/pair_time.py 2>&1 | tail -1; done | tee gpurun_out/${T}_pair_time.log
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/${T}_pytest.log; tail -8 gpurun_out/${T}_pytest.log
