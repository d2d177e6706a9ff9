# parity + head-mode comparison (auto/cluster vs poll vs finish) on the headline bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-cmp}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
for M in -1 1 0; do
  NANOSPEC_HEAD_MODE=$M timeout 300 python bench.py --steps 200 --warmup 20 --head tc --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/${T}_bench_m$M.log
  python -c "
import json; j=json.load(open('gpurun_out/${T}_bench_m$M.log'))
print('mode $M', j['breakdown'], 'frac', j['roofline']['frac'])"
done
timeout 300 python scripts/trace_head.py 2>&1 | tail -14
