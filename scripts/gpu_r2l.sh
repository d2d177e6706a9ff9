cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2l}
timeout 900 python bench.py --steps 100 --warmup 10 --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline'], 'e2e', j['e2e']['value'], 'replays', j['replays'])"
