cd $GRAFT_REPO_ROOT
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | grep -B3 -A30 "trace fused step" | head -34
for f in 0 512; do NANOSPEC_SPLIT_FLAGS=$f timeout 300 python scripts/split_dev.py 2>&1 | grep -v Warn | tail -2; done
timeout 900 python -m pytest -q -x tests/test_step_gpu.py tests/test_head_gpu.py tests/test_parity_r2_gpu.py 2>&1 | tail -3
