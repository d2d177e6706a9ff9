cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | grep -A14 "trace fused step" | head -14
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | tail -4
timeout 900 python bench.py --steps 100 --warmup 10 --no-cpu --no-dense 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'])"
timeout 1500 python -m pytest tests/test_step_gpu.py tests/test_parity_r2_gpu.py tests/test_state_gpu.py -x -q 2>&1 | tail -3
