# re-entry baseline at HEAD: GPU tests, trace of the fused step, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | tail -40
timeout 900 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/r3a_bench.json
python -c "
import json; j=json.load(open('gpurun_out/r3a_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline'], 'dense', j['dense'], 'clocks', j['clocks'])"
