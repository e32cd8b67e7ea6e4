cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "temporal_blocking or virtual_slabs or config5" -p no:cacheprovider > gpurun_out/vm_pytest_cur.log 2>&1; echo "exit=$?" >> gpurun_out/vm_pytest_cur.log
REPS="1 2" STEPS=40 CONFIGS="C4:4 C5:4 C3:2 C2:4 C3f32:4" MODE=run bash tools/tb_variants.sh
