# Profiles of the headline step: ncu launch list of the first fused steps and
# one full capture of the fused step kernel (head_tc_kernel<64, 3>).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-prof}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"head_tc|state_" -s 24 -c 45 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 40 --warmup 5 --no-cpu --no-dense > gpurun_out/${T}_ncu_launch.log 2>&1
tail -1 gpurun_out/${T}_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"head_tc_kernel<.int.64, .int.3>" -s 10 -c 1 -o gpurun_out/${T}_fused_full python bench.py --steps 10 --warmup 12 --no-cpu --no-dense > gpurun_out/${T}_ncu_full.log 2>&1
tail -1 gpurun_out/${T}_ncu_full.log
