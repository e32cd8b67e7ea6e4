cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu11.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_gpu11.log
for c in C1 C2 C3 C3f32 C4 C5; do timeout 300 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/r11_$c.log 2>&1; done
timeout 400 python bench.py > gpurun_out/bench_default5.log 2>&1
