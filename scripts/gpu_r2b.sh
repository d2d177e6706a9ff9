# round-2: split head correctness + bench vs the cluster head
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2b}
timeout 300 python scripts/pair_dev.py --mode 7 2>&1 | tail -40 > gpurun_out/${T}_dev.log; tail -40 gpurun_out/${T}_dev.log
for m in 7 2; do MODE=$m timeout 120 python scripts/pair_time.py 2>&1 | tail -1; done
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['value'])"
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu --no-dense --head-mode 2 2>&1 | tail -1 > gpurun_out/${T}_bench_m2.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench_m2.json'))
print('MODE2 value', j['value'], j['breakdown'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['value'])"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/${T}_pytest.log; tail -30 gpurun_out/${T}_pytest.log
