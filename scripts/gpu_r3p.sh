cd $GRAFT_REPO_ROOT
for f in 0 16384 32768 0 16384 32768; do
NANOSPEC_SPLIT_FLAGS=$f timeout 900 python bench.py --no-cpu --no-dense --steps 100 2>&1 | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown']; print('flags $f', j['value'], 'head', b['us_head_call'], 'stream', b['us_stream_kernel_alone'], 'n1', b['us_head_n1'], 'warm', b['us_head_warm_l2'])"
done
