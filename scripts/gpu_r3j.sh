cd $GRAFT_REPO_ROOT
for f in 1024 0 1024 0; do
NANOSPEC_SPLIT_FLAGS=$f timeout 900 python bench.py --no-cpu --no-dense --steps 100 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('flags $f', j['value'], 'head', j['breakdown']['us_head_call'], 'e2e', j['e2e']['value'], 'serial', j['breakdown'].get('us_e2e_serial_host_step'), j['clocks'])"
done
python scripts/e2e_dev.py 2>&1 | tail -2
