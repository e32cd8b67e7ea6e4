#!/usr/bin/env bash
# One ncu --set full capture of a config's dominant kernel plus its launch list (run on a
# B200 via gpurun from the repo root; all ncu runs in ONE gpurun call):
#   gpurun --timeout 1500 -- 'bash tools/ncu_capture.sh C2:4 C3:2 C3f32:4'
# Each argument is CONFIG:TSTEPS.  The same bench command first runs plain (its line is the
# measured number, kept as gpurun_out/bench_<cfg>_T<t>.json); numbers printed under ncu
# are never bench values.  Summaries are made here with profiles/summarize.py.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for spec in "$@"; do
  cfg="${spec%%:*}"; T="${spec##*:}"
  tag="${cfg}_T${T}"
  # whole passes only: 4 passes per timed region, one pass of warm-up, one repetition
  cmd="python bench.py --config $cfg --tsteps $T --steps $((4 * T)) --warmup $T --reps 1 --no-e2e --no-cpu"
  pat="k_two_step_tb"; [ "$T" = 1 ] && pat="k_two_step_stream"
  $cmd > "gpurun_out/bench_${tag}.json" 2> "gpurun_out/bench_${tag}.err" &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file "gpurun_out/launches_${tag}.csv" $cmd > "gpurun_out/ncu_list_${tag}.log" 2>&1
  $cmd > /dev/null 2>&1 &&
  ncu --set full --clock-control none --import-source on -k "regex:$pat" -s 2 -c 1 -f \
      -o "gpurun_out/prof_${tag}" $cmd > "gpurun_out/ncu_full_${tag}.log" 2>&1
  echo "$tag done rc=$?"
done
