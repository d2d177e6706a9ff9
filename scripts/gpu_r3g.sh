cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | grep -A30 "trace fused step" | grep "B \|head\|fused"
timeout 900 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/r3g_bench.json
python -c "
import json; j=json.load(open('gpurun_out/r3g_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline']['frac'], j['roofline']['stream_kernel'], 'dense', j['dense'], 'e2e', j['e2e'], 'clocks', j['clocks'])"
