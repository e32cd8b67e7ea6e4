#!/usr/bin/env bash
# Round verification on a B200 (run via gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_check.sh'
# GPU parity tests, smoke, the default bench line, the reference arm, and one bench line
# per BASELINE config; logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider \
  > gpurun_out/pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1
for c in C1 C2 C3 C3f32; do
  timeout 300 python bench.py --config "$c" --no-e2e --no-cpu > "gpurun_out/bench_$c.log" 2>&1
done
timeout 400 python bench.py --config C5 --no-cpu > gpurun_out/bench_C5.log 2>&1
