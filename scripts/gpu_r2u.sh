cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for f in 0 128; do
  echo "flags $f"; NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'])"
done
timeout 300 python scripts/split_dev.py --trace 2>&1 | grep -v Warn | tail -32
