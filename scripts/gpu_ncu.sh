cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-nc}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_tc|state_update" -s 40 -c 2 -o gpurun_out/${T}_full python bench.py --steps 10 --warmup 5 --head tc --no-cpu --no-dense > gpurun_out/${T}_ncu_full.log 2>&1
tail -2 gpurun_out/${T}_ncu_full.log
