cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2k}
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_parity_r2_gpu.py tests/test_parallel_nccl_gpu.py -q 2>&1 | tail -8
timeout 300 python scripts/sanitize.py 2>&1 | tail -2
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/${T}_sanitizer_${tool}.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/${T}_sanitizer_${tool}.log
done
timeout 900 python bench.py --steps 100 --warmup 10 --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/${T}_bench.json
python -c "
import json; j=json.load(open('gpurun_out/${T}_bench.json'))
print('value', j['value'], j['breakdown'], 'frac', j['roofline'], 'e2e', j['e2e']['value'], 'replays', j['replays'])"
