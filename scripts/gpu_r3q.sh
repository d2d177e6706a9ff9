# the stream kernel's deferred grid-dependency wait (overlap with the previous select): A/B vs flag 16384, tests
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | grep -A4 "graph of 3 step"
for f in 16384 0 16384 0; do
NANOSPEC_SPLIT_FLAGS=$f timeout 900 python bench.py --no-cpu --no-dense --steps 100 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown']; print('flags $f', j['value'], 'head', b['us_head_call'], 'two-launch', b['us_step_two_launches'], 'round', b['us_draft_round_tree_and_step'], 'e2e', j['e2e']['value'])"
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
