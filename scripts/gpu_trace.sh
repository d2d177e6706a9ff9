cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/trace_head.py --state 2>&1 | tail -40 | tee gpurun_out/trace_head.log
timeout 300 python scripts/trace_head.py --n 1 --k 10 2>&1 | tail -12 | tee -a gpurun_out/trace_head.log
timeout 600 python -m pytest tests/test_head_gpu.py tests/test_full_vocab_gpu.py -x -q -k "tc" 2>&1 | tail -3
timeout 300 python bench.py --steps 200 --warmup 20 --head tc --no-cpu 2>&1 | tail -1 | cut -c 700-1300
