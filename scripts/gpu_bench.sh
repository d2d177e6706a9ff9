# bench both heads + a launch list of the headline run (ncu, serialised, cold cache)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 200 --warmup 20 --head tc 2>&1 | tail -3 | tee gpurun_out/r1_bench_tc.log
timeout 300 python bench.py --steps 200 --warmup 20 --head simt --no-cpu 2>&1 | tail -3 | tee gpurun_out/r1_bench_simt.log
timeout 300 python bench.py --steps 100 --warmup 10 --head tc --n-nodes 1 --no-cpu --no-dense 2>&1 | tail -2 | tee gpurun_out/r1_bench_tc_n1.log
timeout 300 python bench.py --steps 100 --warmup 10 --head simt --n-nodes 1 --no-cpu --no-dense 2>&1 | tail -2 | tee gpurun_out/r1_bench_simt_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 20 --warmup 5 --head tc --no-cpu --no-dense > gpurun_out/r1_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:head_tc -s 30 -c 2 -o gpurun_out/r1_head_tc python bench.py --steps 10 --warmup 5 --head tc --no-cpu --no-dense > gpurun_out/r1_ncu_full.log 2>&1
tail -3 gpurun_out/r1_ncu_full.log
