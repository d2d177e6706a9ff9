# round-1 GPU check: parity tests (CUDA-core path first, then tensor-core path), smoke, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "not tc" 2>&1 | tail -30 > gpurun_out/r1_pytest_simt.log
tail -3 gpurun_out/r1_pytest_simt.log
timeout 300 python bench.py --steps 100 --warmup 10 --head simt --no-cpu 2>&1 | tail -3 | tee gpurun_out/r1_bench_simt.log
timeout 300 python -m pytest tests/test_head_gpu.py -x -q -k "tiny and tc" 2>&1 | tail -30 > gpurun_out/r1_pytest_tc_tiny.log
tail -3 gpurun_out/r1_pytest_tc_tiny.log
timeout 600 python -m pytest tests -m gpu -x -q -k "tc" 2>&1 | tail -30 > gpurun_out/r1_pytest_tc.log
tail -3 gpurun_out/r1_pytest_tc.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 300 python bench.py --steps 100 --warmup 10 --head tc 2>&1 | tail -3 | tee gpurun_out/r1_bench_tc.log
