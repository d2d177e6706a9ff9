# mixed tile-pair / single-tile units in the persistent mode: timing A/B (flag 2048 = pairs only), parity, sanitizers
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for f in 2048 0; do
  echo "flags $f"
  NANOSPEC_SPLIT_FLAGS=$f timeout 600 python bench.py --config dp64 --steps 20 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['breakdown'], j['roofline']['frac'])"
  NANOSPEC_SPLIT_FLAGS=$f timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --replays 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['dense'])"
done
timeout 900 python -m pytest -q -x tests/test_parity_r2_gpu.py tests/test_full_vocab_gpu.py tests/test_head_gpu.py 2>&1 | tail -2
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py > gpurun_out/r3k_sanitizer_$tool.log 2>&1; tail -2 gpurun_out/r3k_sanitizer_$tool.log
done
