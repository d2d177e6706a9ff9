cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_step_gpu.py -k "host" 2>&1 | tail -3
timeout 900 python bench.py --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/r3h_bench.json
python -c "
import json; j=json.load(open('gpurun_out/r3h_bench.json'))
print('value', j['value'], 'e2e', j['e2e'], 'serial', j['breakdown'].get('us_e2e_serial_host_step'))"
