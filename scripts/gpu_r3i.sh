cd $GRAFT_REPO_ROOT
python scripts/e2e_dev.py 2>&1 | tail -2
for f in 0 1024; do NANOSPEC_SPLIT_FLAGS=$f timeout 300 python scripts/split_dev.py 2>&1 | grep -v Warn | tail -2; done
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | grep -A16 "trace fused step" | grep "A drained\|A loads\|B done\|B dep"
timeout 900 python -m pytest -q -x tests/test_step_gpu.py 2>&1 | tail -2
