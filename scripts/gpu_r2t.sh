cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for f in 0 64 128 96; do
  echo "flags $f"
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | cut -c150-200
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --replays 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['dense'])"
done
