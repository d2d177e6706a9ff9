# GPU check: parity tests (CUDA-core path first, then tensor-core path), smoke, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r1}
timeout 900 python -m pytest tests -m gpu -x -q -k "not tc" 2>&1 | tail -30 > gpurun_out/${T}_pytest_simt.log
tail -3 gpurun_out/${T}_pytest_simt.log
timeout 300 python -m pytest tests/test_head_gpu.py -x -q -k "tiny and tc" 2>&1 | tail -30 > gpurun_out/${T}_pytest_tc_tiny.log
tail -3 gpurun_out/${T}_pytest_tc_tiny.log
timeout 600 python -m pytest tests -m gpu -x -q -k "tc" 2>&1 | tail -30 > gpurun_out/${T}_pytest_tc.log
tail -3 gpurun_out/${T}_pytest_tc.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python bench.py --steps 200 --warmup 20 --head tc 2>&1 | tail -3 | tee gpurun_out/${T}_bench_tc.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 5 --head tc --no-cpu --no-dense > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:head_tc -s 30 -c 1 -o gpurun_out/${T}_head_tc python bench.py --steps 10 --warmup 5 --head tc --no-cpu --no-dense > gpurun_out/${T}_ncu_full.log 2>&1
tail -2 gpurun_out/${T}_ncu_full.log
