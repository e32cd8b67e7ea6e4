cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "temporal" > gpurun_out/pytest_tb.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_tb.log
for c in C5 C4 C3f32 C3; do for t in 1 2 4; do timeout 200 python bench.py --config $c --tsteps $t --no-e2e --no-cpu > gpurun_out/tb_${c}_T$t.log 2>&1; done; done
B="python bench.py --steps 6 --warmup 6 --no-e2e --no-cpu"
$B > gpurun_out/plain_c4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_v2.csv $B > gpurun_out/ncu_launch_c4.log 2>&1
$B > gpurun_out/plain_c4b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_two_step -s 8 -c 1 -o gpurun_out/prof_c4_v2 $B > gpurun_out/ncu_full_c4.log 2>&1
B5="python bench.py --config C5 --steps 8 --warmup 6 --no-e2e --no-cpu --tsteps 2"
$B5 > gpurun_out/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_two_step_tb -s 4 -c 1 -o gpurun_out/prof_c5_tb2 $B5 > gpurun_out/ncu_full_c5.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_default2.log 2>&1
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1
