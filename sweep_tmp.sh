cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_gpu5.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke5.log 2>&1
for c in C5 C3f32; do for t in 1 2 4; do timeout 200 python bench.py --config $c --tsteps $t --no-e2e --no-cpu > gpurun_out/tb3_${c}_T$t.log 2>&1; done; done
B5="python bench.py --config C5 --steps 8 --warmup 6 --no-e2e --no-cpu --tsteps 2"
$B5 > gpurun_out/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_two_step_tb -s 4 -c 1 -o gpurun_out/prof_c5_tb2c $B5 > gpurun_out/ncu_full_c5.log 2>&1
