# Round evidence: GPU parity tests, smoke, default bench (+ reference arm),
# dp64 / vp32k / qwen512 lines, ncu launch list of the headline step (both
# head kernels) -> profiles/traffic.json, one ncu --set full capture of each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-round}
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"head_|state_" -s 60 -c 60 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 40 --warmup 5 --no-cpu --no-dense --replays 1 > gpurun_out/${T}_ncu_launch.log 2>&1
python scripts/traffic_from_ncu.py gpurun_out/${T}_launches.csv --out profiles/traffic.json | tail -5
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline'], 'e2e', j['e2e']['value'], 'dense', j['dense'], 'cpu', j['cpu_baseline'], 'clocks', j['clocks'])"
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_ref.json
cut -c1-300 gpurun_out/${T}_bench_ref.json
timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_dp64.json
cut -c1-400 gpurun_out/${T}_bench_dp64.json
timeout 600 python bench.py --config vp32k --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_vp32k.json
cut -c1-400 gpurun_out/${T}_bench_vp32k.json
timeout 600 python bench.py --config qwen512 2>&1 | tail -1 > gpurun_out/${T}_bench_qwen512.json
cut -c1-600 gpurun_out/${T}_bench_qwen512.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_stream_kernel" -s 20 -c 1 -o gpurun_out/${T}_stream_full python bench.py --steps 10 --warmup 5 --no-cpu --no-dense --replays 1 > gpurun_out/${T}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_select" -s 20 -c 1 -o gpurun_out/${T}_select_full python bench.py --steps 10 --warmup 5 --no-cpu --no-dense --replays 1 > gpurun_out/${T}_ncu_full2.log 2>&1
tail -n 1 gpurun_out/${T}_ncu_full.log gpurun_out/${T}_ncu_full2.log
cp profiles/traffic.json gpurun_out/${T}_traffic.json
