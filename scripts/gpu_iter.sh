# quick iteration: GPU parity (all), trace, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-it}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python scripts/trace_head.py --state 2>&1 | tail -24 | tee gpurun_out/${T}_trace.log
timeout 300 python bench.py --steps 200 --warmup 20 --head tc --no-cpu 2>&1 | tail -1 > gpurun_out/${T}_bench.log
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.log'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['value'], 'dense', j['dense'])"
