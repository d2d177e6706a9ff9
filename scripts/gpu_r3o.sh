cd $GRAFT_REPO_ROOT
for f in 0 8192; do
  echo "flags $f"
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config vp32k --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'])"
  NANOSPEC_SPLIT_FLAGS=$f timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --replays 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['dense'])"
done
timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('dp64', j['value'], j['breakdown'])"
timeout 900 python -m pytest -q -x tests/test_parity_r2_gpu.py tests/test_full_vocab_gpu.py tests/test_head_gpu.py tests/test_tree_gpu.py 2>&1 | tail -2
