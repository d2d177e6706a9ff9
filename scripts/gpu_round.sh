# Round-end evidence: GPU parity tests, smoke, default bench (+ reference arm),
# ncu launch list of the headline step and one full capture each of the fused
# step kernel and the head-only kernel; dp64 / vp32k single-GPU lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-round}
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['value'], 'dense', j['dense'], 'cpu', j['cpu_baseline']['value'], 'clocks', j['clocks'])"
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_ref.json
cut -c1-300 gpurun_out/${T}_bench_ref.json
timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_dp64.json
cut -c1-400 gpurun_out/${T}_bench_dp64.json
timeout 600 python bench.py --config vp32k --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${T}_bench_vp32k.json
cut -c1-400 gpurun_out/${T}_bench_vp32k.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"head_tc|state_" -s 24 -c 45 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 40 --warmup 5 --no-cpu --no-dense > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"head_tc_kernel<.int.64, .int.3>" -s 10 -c 1 -o gpurun_out/${T}_fused_full python bench.py --steps 10 --warmup 12 --no-cpu --no-dense > gpurun_out/${T}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"head_tc_kernel<.int.64, .int.2>" -s 30 -c 1 -o gpurun_out/${T}_head_full python bench.py --steps 10 --warmup 5 --no-cpu --no-dense --no-fuse > gpurun_out/${T}_ncu_full2.log 2>&1
tail -n 1 gpurun_out/${T}_ncu_full.log gpurun_out/${T}_ncu_full2.log
