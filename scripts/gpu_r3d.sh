cd $GRAFT_REPO_ROOT
python scripts/list_dev.py 2>&1 | grep -v "busy"; python scripts/list_dev.py --B 8 2>&1 | grep -v busy
timeout 600 python -m pytest -q -x tests/test_parity_r2_gpu.py tests/test_full_vocab_gpu.py 2>&1 | tail -3
bash scripts/gpu_r3c.sh
