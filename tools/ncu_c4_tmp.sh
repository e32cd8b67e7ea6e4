cd $GRAFT_REPO_ROOT
B="python bench.py --steps 8 --warmup 6 --no-e2e --no-cpu --tsteps 4"
$B > gpurun_out/plain_c4t4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_t4.csv $B > gpurun_out/ncu_launch_c4t4.log 2>&1
$B > gpurun_out/plain_c4t4b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_two_step_tb -s 1 -c 1 -o gpurun_out/prof_c4_t4 $B > gpurun_out/ncu_full_c4t4.log 2>&1
B1="python bench.py --steps 8 --warmup 6 --no-e2e --no-cpu --tsteps 1"
$B1 > gpurun_out/plain_c4t1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_two_step_stream -s 8 -c 1 -o gpurun_out/prof_c4_t1 $B1 > gpurun_out/ncu_full_c4t1.log 2>&1
