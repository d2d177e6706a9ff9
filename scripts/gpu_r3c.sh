# list-mode timing: dp64 / vp32k / dense lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for f in 0; do
  echo "flags $f"
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'])"
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config vp32k --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'])"
done
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu --replays 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['dense'])"
