cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/r3r_bench_dp64.json
python -c "import json; j=json.load(open('gpurun_out/r3r_bench_dp64.json')); print('dp64', j['value'], j['breakdown'], j['roofline']['frac'])"
timeout 900 python bench.py --no-cpu --no-dense 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown']; print('step', j['value'], 'head', b['us_head_call'], 'two-launch', b['us_step_two_launches'], 'round', b['us_draft_round_tree_and_step'], 'e2e', j['e2e']['value'])"
