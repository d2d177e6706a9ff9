cd $GRAFT_REPO_ROOT
for f in 4096 0; do NANOSPEC_SPLIT_FLAGS=$f timeout 300 python scripts/split_dev.py 2>&1 | grep -v Warn | tail -2; done
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | grep -A30 "trace fused step" | grep "B \|A drained"
for f in 4096 0 4096 0; do
NANOSPEC_SPLIT_FLAGS=$f timeout 900 python bench.py --no-cpu --no-dense --steps 100 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('flags $f', j['value'], 'head', j['breakdown']['us_head_call'])"
done
timeout 900 python -m pytest -q -x tests/test_step_gpu.py tests/test_head_gpu.py tests/test_parity_r2_gpu.py 2>&1 | tail -2
