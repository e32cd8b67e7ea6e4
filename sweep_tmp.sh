cd $GRAFT_REPO_ROOT
for v in default t43 t42 t82 t83 t24; do
  if [ $v = default ]; then L=""; else L="PS_LIBRARY=build/tune/libps_$v.so"; fi
  for c in C5 C4; do for t in 2 4; do
    env $L timeout 200 python bench.py --config $c --tsteps $t --no-e2e --no-cpu > gpurun_out/tbs_${v}_${c}_T$t.log 2>&1
  done; done
done
