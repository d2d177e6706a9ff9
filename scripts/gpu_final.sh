# final check of the committed code: every GPU test, smoke, the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/final_pytest.log; cat gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/final_bench.json
python -c "
import json; j=json.load(open('gpurun_out/final_bench.json'))
print('value', j['value'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['value'], 'dense', j['dense'], 'clocks', j['clocks'], 'launches', j['gpu_launches'])"
