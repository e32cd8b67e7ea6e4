#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_cases.py — ONE tool per gpurun call
# (B200_PROFILING.md: several tools in one call have wedged the GPU):
#   gpurun --timeout 1500 -- 'bash tools/sanitize.sh memcheck'
#   gpurun --timeout 1500 -- 'bash tools/sanitize.sh racecheck'
#   gpurun --timeout 1500 -- 'bash tools/sanitize.sh synccheck'
# The case script first runs plain (it must exit 0 on its own), then under the tool; the
# tool's report lands in gpurun_out/sanitize_<tool>.log (summary copied to profiles/).
tool="${1:-memcheck}"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python tools/sanitize_cases.py > "gpurun_out/sanitize_plain_${tool}.log" 2>&1 || { echo "plain run failed"; tail -20 "gpurun_out/sanitize_plain_${tool}.log"; exit 1; }
timeout 1300 compute-sanitizer --tool "$tool" --print-limit 30 \
  --log-file "gpurun_out/sanitize_${tool}.log" python tools/sanitize_cases.py \
  > "gpurun_out/sanitize_${tool}.out" 2>&1
echo "rc=$?"; tail -3 "gpurun_out/sanitize_${tool}.out"; tail -15 "gpurun_out/sanitize_${tool}.log"
