# full round check: GPU parity tests, smoke, default bench, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-full}
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['value'], 'dense', j['dense'], 'cpu', j['cpu_baseline'], 'clocks', j['clocks'])"
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_ref.json
cat gpurun_out/${T}_bench_ref.json | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-dense > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_tc|state_update" -s 40 -c 2 -o gpurun_out/${T}_full python bench.py --steps 10 --warmup 5 --no-cpu --no-dense > gpurun_out/${T}_ncu_full.log 2>&1
tail -1 gpurun_out/${T}_ncu_full.log
