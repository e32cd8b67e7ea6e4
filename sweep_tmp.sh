cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_gpu3.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1
for v in default f g h k a; do
  if [ $v = default ]; then L=""; else L="PS_LIBRARY=build/tune/libps_$v.so"; fi
  for c in C4 C3 C3f32 C2 C1 C5; do
    env $L timeout 150 python bench.py --config $c --warmup 6 --no-e2e --no-cpu > gpurun_out/sw2_${v}_$c.log 2>&1
  done
done
