# list mode (persistent split-K 1): parity of the S = 1 shapes + dp64 / dense timings, list vs partials (flag 256)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_r2_gpu.py tests/test_full_vocab_gpu.py tests/test_head_gpu.py -x -q 2>&1 | tail -15
for f in 0 256; do
  echo "flags $f"
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'])"
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config vp32k --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'])"
done
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu --replays 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['dense'])"
