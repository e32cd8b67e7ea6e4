cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu6.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_gpu6.log
for c in C5 C4 C3 C3f32; do for t in 1 2 4; do timeout 200 python bench.py --config $c --tsteps $t --no-e2e --no-cpu > gpurun_out/r6_${c}_T$t.log 2>&1; done; done
for c in C1 C2; do timeout 200 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/r6_${c}_T1.log 2>&1; done
