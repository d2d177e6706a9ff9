cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2q}
for f in 0 32; do NANOSPEC_SPLIT_FLAGS=$f timeout 200 python scripts/split_dev.py 2>&1 | grep -v Warn | tail -2; done
timeout 900 python bench.py --steps 100 --warmup 10 --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown'])"
timeout 1500 python -m pytest tests/test_parity_r2_gpu.py tests/test_head_gpu.py tests/test_step_gpu.py -x -q 2>&1 | tail -3
