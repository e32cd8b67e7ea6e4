cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 400 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1
for c in C1 C2 C3 C3f32; do timeout 300 python bench.py --config "$c" --no-e2e --no-cpu > "gpurun_out/bench_$c.log" 2>&1; done
timeout 400 python bench.py --config C5 --no-cpu > gpurun_out/bench_C5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_two_step_tb -s 3 -c 1 -o gpurun_out/prof_c4_r01final python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --tsteps 4 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_two_step_tb -s 3 -c 1 -o gpurun_out/prof_c5_r01final python bench.py --config C5 --steps 4 --warmup 3 --no-e2e --no-cpu --tsteps 4 > gpurun_out/ncu_full_c5.log 2>&1
