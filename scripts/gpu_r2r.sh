cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2r}
timeout 1500 python -m pytest tests/test_full_vocab_gpu.py tests/test_parity_r2_gpu.py tests/test_head_gpu.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown']['us_head_call'], 'dense', j['dense'])"
timeout 600 python bench.py --config vp32k --steps 20 --warmup 3 2>&1 | tail -1 | cut -c1-250
